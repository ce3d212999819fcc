# long multi-GPU runs: 20000 forwards back to back (ranks coupled only through device flags)
for R in "--routing balanced" "--routing zipf --skew 1.2" "--routing gate --signaling vanilla"; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${N:-4} --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus ${N:-4} --steps 20000 --warmup 5 --no-cpu-baseline --variant-steps 0 $R 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); c=d['per_step_counters']
print('$R', 'steps', d['steps'], 'us', round(d['ms_per_step']*1e3,1), 'timeouts', c['wait_timeouts'], 'errors', c['errors'], 'e2e_ok', d['e2e']['output_matches_device_forward'])"
done
