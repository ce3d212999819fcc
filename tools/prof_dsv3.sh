mkdir -p gpurun_out
B="python bench.py --config dsv3 --experts 64 --steps 5 --warmup 3 --no-cpu-baseline --variant-steps 0"
timeout 600 $B 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); c=d['per_step_counters']; print(round(d['ms_per_step']*1e3,1), json.dumps(d['timeline_us']), {k: round(v,3) for k,v in c.items() if k.startswith('frac')}, d['clocks'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_moe2" -s 2 -c 1 -o gpurun_out/prof_dsv3e64 $B > gpurun_out/ncu_dsv3e64.log 2>&1
tail -1 gpurun_out/ncu_dsv3e64.log
