# A/B of an env switch with the per-kernel timeline: ABVAR unset vs ABVAR=ABVAL, alternated
for r in 1 2 3; do
  for v in "" "$ABVAL"; do
    if [ -z "$v" ]; then unset $ABVAR; else export $ABVAR=$v; fi
    timeout 300 python bench.py --steps 300 --warmup 5 --no-cpu-baseline $A 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); t=d['timeline_us']
print('$ABVAR=$v', round(d['ms_per_step']*1e3,1), 'e2e', round(d['e2e']['ms_per_step']*1e3,1), {k: t[k] for k in ('plan','fused_cta_entry','fused','combine') if k in t})"
  done
done
