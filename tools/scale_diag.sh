# N = 1, 2, 4 bench lines with the producer / MMA stall split (run under gpurun --gpus 4)
for N in ${NLIST:-1 2 4}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29800+N)) bench.py --gpus $N --steps 300 --warmup 5 --no-cpu-baseline --variant-steps 0 2>&1 | grep '^{' | python -c "
import sys,json
d=json.loads(sys.stdin.read()); c=d['per_step_counters']
print('N=$N', round(d['ms_per_step']*1e3,1), int(d['value']), {k: round(c[k],3) for k in c if k.startswith('frac')}, 'exp', None if not d['comm'] else (round(d['comm']['exposed_dispatch_us'],1), round(d['comm']['exposed_combine_us'],1), round(d['comm']['dispatch_nvlink_gbs'])), d['timeline_us'].get('fused'))"
done
