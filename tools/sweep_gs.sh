N=${N:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for args in "--group-size 0" "--group-size 32" "--group-size 8" "--group-size 2" "--signaling vanilla" "--group-size 0 --unfused"; do
  timeout 300 $R --master-port $((29600 + RANDOM % 300)) bench.py --gpus $N --steps 300 --warmup 5 --no-cpu-baseline $args 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('$args', round(d['ms_per_step']*1e3,1), int(d['value']), {k:round(v*1e3,1) for k,v in d['stage_ms'].items()}, d['per_step_counters']['dispatch_fences'], d['per_step_counters']['combine_fences'])"
done
