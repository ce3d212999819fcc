# per-kernel device timeline of one forward (EP=1 fused; router on/off the side stream)
for SG in 1 0; do
PERSEUS_SIDE_GATE=$SG timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline $A 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('side=$SG', round(d['ms_per_step']*1e3,1), json.dumps(d['timeline_us']))"
done
