# end-of-schedule lag at EP=1: PERSEUS_LAG_END=0 (off: the round-1 schedule) vs the default rule, alternated
for CFG in ${CFGS:-qwen3}; do for r in 1 2 3; do for L in 0 -1; do
  if [ $L = -1 ]; then unset PERSEUS_LAG_END; else export PERSEUS_LAG_END=$L; fi
  timeout 300 python bench.py --config $CFG --steps ${STEPS:-500} --warmup 5 --no-cpu-baseline $A 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); t=d['timeline_us']
print('$CFG lag_end=$L', round(d['ms_per_step']*1e3,1), {k: t[k] for k in ('fused','mma_out_of_work') if k in t}, d['clocks']['sm_mhz'])"
done; done; done
