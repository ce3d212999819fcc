# bench under the reference's skewed routing and the learned gate (N = 1 and 4)
for R in "--routing zipf --skew 1.5" "--routing zipf --skew 0.5" "--routing gate"; do for N in 1 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29970+N)) bench.py --gpus $N --steps 200 --warmup 5 --no-cpu-baseline --variant-steps 0 $R 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); c=d['per_step_counters']
print('$R N=$N', round(d['ms_per_step']*1e3,1), int(d['value']), 'timeouts', c['wait_timeouts'], 'errors', c['errors'], 'pairs', d['cta_pairs'], d['timeline_us'].get('fused'))"
done; done
