# k_moe2 at EP=1: self-copy window x discard of dead heap / h lines.
# Per setting: bench repeat-block median + k_moe2 event time, and ncu DRAM bytes of one launch.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 3 --block-steps 300 --variant-steps 0"
for cfg in "160 0" "160 3" "48 3" "24 3" "12 3" "24 0"; do
  set -- $cfg
  PERSEUS_SELF_WINDOW=$1 PERSEUS_DISCARD=$2 timeout 300 $B > gpurun_out/sw_$1_$2.log 2>&1
  python - $1 $2 <<PY
import json,sys
d=[json.loads(l) for l in open(f"gpurun_out/sw_{sys.argv[1]}_{sys.argv[2]}.log") if l.startswith("{")][-1]
print("window", sys.argv[1], "discard", sys.argv[2], "median_us", round(d["timing_blocks"]["median_ms"]*1e3,1),
      "kmoe2_us", round(d["roofline"]["launch_ms"]*1e3,1), "sm_mhz", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
done
for cfg in "160 0" "160 3" "24 3" "12 3"; do
  set -- $cfg
  PERSEUS_SELF_WINDOW=$1 PERSEUS_DISCARD=$2 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:k_moe2 -s 5 -c 1 --csv $B 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' -v c="$1/$2" '{print c, $(NF-2), $(NF-1), $NF}'
done
