# producer look-ahead beyond 6 and the weights' TMA L2 promotion (same box, alternating)
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 5 --block-steps 400 --variant-steps 0"
run() { env $1 timeout 300 $B > gpurun_out/misc.log 2>&1; grep '^{' gpurun_out/misc.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); pc=d['per_step_counters']
print('$1', 'median_us', round(d['timing_blocks']['median_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'fused', d['timeline_us']['fused'], 'mhz', d['clocks']['sm_mhz'], 'mma_data', round(pc['frac_mma_data_wait'],3))"; }
for rep in 1 2; do
  run PERSEUS_AHEAD=6; run PERSEUS_AHEAD=12; run PERSEUS_AHEAD=20
  run PERSEUS_WPROMO=0; run PERSEUS_WPROMO=128
done
