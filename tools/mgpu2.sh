# GPU tests + multi-GPU parity + bench with comm evidence (run under gpurun --gpus N)
N=${N:-2}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_check.py 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 500 --warmup 5 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/bench_n$N.json
python - <<PY
import json
d=json.load(open("gpurun_out/bench_n$N.json"))
print("us", round(d["ms_per_step"]*1e3,1), "tok/s", int(d["value"]), "e2e", int(d["e2e"]["value"]))
print("comm", json.dumps(d["comm"]))
print("variant", json.dumps(d["per_tile_fence_variant"]))
PY
