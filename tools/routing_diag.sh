cd $GRAFT_REPO_ROOT
for r in "balanced 0" "zipf 1.5" "gate 0"; do set -- $r
  timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --blocks 3 --block-steps 300 --routing $1 --skew $2 > gpurun_out/rt_$1.log 2>&1
  grep '^{' gpurun_out/rt_$1.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('$1', round(d['timing_blocks']['median_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), d['cta_pairs'], 'mhz', d['clocks']['sm_mhz'], json.dumps(d['timeline_us']), 'recv_tiles', d['per_step_counters']['recv_tiles'])"
done
