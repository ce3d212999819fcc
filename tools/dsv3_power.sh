timeout 600 python bench.py --config dsv3 --experts 64 --steps 300 --warmup 5 --no-cpu-baseline --variant-steps 0 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('E64 EP1', round(d['ms_per_step']*1e3,1), d['clocks'], d['timeline_us'].get('fused'))"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus 4 --config dsv3 --steps 300 --warmup 5 --no-cpu-baseline --variant-steps 0 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('DSV3 EP4', round(d['ms_per_step']*1e3,1), d['clocks'], d['timeline_us'].get('fused'), d['comm']['exposed_frac'])"
