# producer look-ahead (take + poll the next item's flag N k-blocks early), same box, alternating
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 5 --block-steps 400 --variant-steps 0"
for rep in 1 2; do for ah in 1 3 6; do
  PERSEUS_AHEAD=$ah timeout 300 $B > gpurun_out/ah_$ah.log 2>&1
  grep '^{' gpurun_out/ah_$ah.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); pc=d['per_step_counters']
print('ahead $ah median_us', round(d['timing_blocks']['median_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'fused_tl', d['timeline_us']['fused'], 'mhz', d['clocks']['sm_mhz'], 'wait_d', round(pc['frac_wait_dispatch'],3), 'wait_g1', round(pc['frac_wait_g1'],3), 'mma_data', round(pc['frac_mma_data_wait'],3))"
done; done
