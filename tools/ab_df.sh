# A/B: dataflow combine inside the fused kernel (EP=1) vs the combine kernel after it, same box, alternating
cd $GRAFT_REPO_ROOT
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 5 --block-steps 400 --variant-steps 0"
for rep in 1 2 3; do for df in 1 0; do
  PERSEUS_DF_COMBINE=$df timeout 300 $B > gpurun_out/df_$df.log 2>&1
  grep '^{' gpurun_out/df_$df.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); pc=d['per_step_counters']
print('df $df median_us', round(d['timing_blocks']['median_ms']*1e3,1), 'min', round(d['timing_blocks']['min_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'fused', d['timeline_us'].get('fused'), 'combine', d['timeline_us'].get('combine'), 'mhz', d['clocks']['sm_mhz'], 'e2e', int(d['e2e']['value']), 'ok', d['e2e']['output_matches_device_forward'])"
done; done
