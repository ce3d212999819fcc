N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for args in "--group-size 0" "--signaling vanilla"; do
  timeout 300 $R --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 300 --warmup 5 --no-cpu-baseline $args 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); c=d['per_step_counters']; print('$args', round(d['ms_per_step']*1e3,1), int(d['value']), {k:round(v*1e3,1) for k,v in d['stage_ms'].items()}, {k: round(c[k],3) for k in ('frac_wait_dispatch','frac_wait_g1','frac_copy_busy')}, round(c['cta_ns']/148/1e3,1))"
done
