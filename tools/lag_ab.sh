# new lag rule (PERSEUS_LAG_PAIRS unset) vs the round-1 rule (one wave of GEMM1 items), per shape, alternated
declare -A OLD=([qwen3]=13 [llama4]=8 [dsv3]=5)
declare -A ST=([qwen3]=400 [llama4]=100 [dsv3]=40)
for CFG in ${CFGS:-qwen3 dsv3 llama4}; do for r in 1 2; do for L in ${OLD[$CFG]} 0; do
  PERSEUS_LAG_PAIRS=$L timeout 300 python bench.py --config $CFG --steps ${ST[$CFG]} --warmup 5 --no-cpu-baseline $A 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); t=d['timeline_us']
print('$CFG lag=$L', round(d['ms_per_step']*1e3,1), {k: t[k] for k in ('fused','mma_out_of_work') if k in t}, d['clocks']['sm_mhz'])"
done; done; done
