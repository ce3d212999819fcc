timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_check.py > gpurun_out/mgpu_pairs.log 2>&1; grep -o '"mgpu_check": "[A-Z]*[a-z]*"' gpurun_out/mgpu_pairs.log
for CFG in dsv3 qwen3; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29881 bench.py --gpus 4 --config $CFG --steps 200 --warmup 5 --no-cpu-baseline --variant-steps 0 2>&1 | grep '^{' | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$CFG EP4', round(d['ms_per_step']*1e3,1), int(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), round(d['comm']['exposed_frac'],3))"
done
