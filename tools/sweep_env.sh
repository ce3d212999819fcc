# generic same-box A/B of environment switches, alternating:  SETS="PERSEUS_X=0 PERSEUS_X=1" REPS=2 bash tools/sweep_env.sh
# (a set may hold several assignments joined by ','); extra bench flags in BENCH_ARGS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --blocks 5 --block-steps 400 --variant-steps 0 $BENCH_ARGS"
for rep in $(seq ${REPS:-2}); do for s in $SETS; do
  tag=$(echo $s | tr ',=' '__')
  env $(echo $s | tr ',' ' ') timeout 300 $B > gpurun_out/sw_$tag.log 2>&1
  grep '^{' gpurun_out/sw_$tag.log | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); tl=d['timeline_us']
print('$s median_us', round(d['timing_blocks']['median_ms']*1e3,1), 'min', round(d['timing_blocks']['min_ms']*1e3,1), 'K', round(d['ms_per_step']*1e3,1), 'mhz', d['clocks']['sm_mhz'],
      'plan', tl.get('plan'), 'entry', tl.get('fused_cta_entry'), 'fused', tl.get('fused'), 'combine', tl.get('combine'))" || tail -5 gpurun_out/sw_$tag.log
done; done
