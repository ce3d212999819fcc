cd $GRAFT_REPO_ROOT
for rep in 1 2; do for v in 1 2; do
  PERSEUS_GATE_V=$v timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --blocks 3 --block-steps 300 --routing gate > gpurun_out/gv_$v.log 2>&1
  grep '^{' gpurun_out/gv_$v.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print('gate v$v', round(d['timing_blocks']['median_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'mhz', d['clocks']['sm_mhz'], 'route', d['timeline_us']['route'], 'fused', d['timeline_us']['fused'])"
done; done
