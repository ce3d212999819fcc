# EP=1 fused-kernel issue-side stall breakdown at a few token counts
for S in ${SLIST:-4096 8192}; do
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --tokens $S 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); c=d['per_step_counters']
print('S=$S', round(d['ms_per_step']*1e3,1), int(d['value']), 'clk', d['clocks'].get('sm_mhz'), {k: round(c[k],3) for k in c if k.startswith('frac')})"
done
