# k_moe2 at EP=1: persisting L2 window over h or the heap (DRAM bytes via ncu + bench time)
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 3 --block-steps 300 --variant-steps 0"
for cfg in "none 0" "h 32" "h 48" "heap 32" "heap 64"; do
  set -- $cfg
  if [ $1 = none ]; then unset PERSEUS_L2_WIN; else export PERSEUS_L2_WIN=$1 PERSEUS_L2_MB=$2; fi
  timeout 300 $B > gpurun_out/l2_$1_$2.log 2>&1
  grep '^{' gpurun_out/l2_$1_$2.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('$1 $2 median_us', round(d['timing_blocks']['median_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'kmoe2_tl', d['timeline_us']['fused'], 'mhz', d['clocks']['sm_mhz'])"
done
for cfg in "none 0" "h 48" "heap 64"; do
  set -- $cfg
  if [ $1 = none ]; then unset PERSEUS_L2_WIN; else export PERSEUS_L2_WIN=$1 PERSEUS_L2_MB=$2; fi
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_moe2 -s 5 -c 1 --csv $B 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v c="$1/$2" '{print c, $(NF-2), $(NF-1), $NF}'
done
