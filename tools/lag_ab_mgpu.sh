# new lag rule vs the round-1 rule (13 pairs) at N GPUs (qwen3), alternated; exposed comm too
N=${N:-4}
for r in 1 2; do for L in 13 0; do
  PERSEUS_LAG_PAIRS=$L timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700+r*10+L%7)) bench.py --gpus $N --steps 400 --warmup 5 --no-cpu-baseline --variant-steps 0 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); t=d['timeline_us']; c=d['comm'] or {}
print('N=$N lag=$L', round(d['ms_per_step']*1e3,1), {k: t[k] for k in ('fused','mma_out_of_work','combine') if k in t}, 'exposed', c.get('exposed_frac'), d['clocks']['sm_mhz'])"
done; done
