# GEMM1 -> GEMM2 lag of the fused kernel (PERSEUS_LAG_PAIRS; 0 = the default rule), with the MMA tail spread
for r in 1 2; do
for L in 0 ${LAGS:-20 26 40}; do
  PERSEUS_LAG_PAIRS=$L timeout 300 python bench.py --steps 400 --warmup 5 --no-cpu-baseline $A 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); t=d['timeline_us']
print('lag=$L', round(d['ms_per_step']*1e3,1), {k: t[k] for k in ('fused','mma_out_of_work','combine') if k in t}, d['clocks']['sm_mhz'])"
done
done
