# N-GPU: parity + device-trace checks, then the bench line (comm evidence + per-tile variant)
N=${N:-4}
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_check.py > gpurun_out/mgpu_n$N.log 2>&1
grep mgpu_check gpurun_out/mgpu_n$N.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['mgpu_check']); [print(json.dumps({k: t[k] for k in ('protocol','violations','conservation')}), t['dispatch']['fence_count'], t['dispatch']['flagged_signal_count']) for t in d['device_trace']]"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --steps 500 --warmup 5 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/bench_n$N.json
python - <<PY
import json
d=json.load(open("gpurun_out/bench_n$N.json"))
print("us", round(d["ms_per_step"]*1e3,1), "tok/s", int(d["value"]), "e2e", int(d["e2e"]["value"]))
print("comm", json.dumps(d["comm"]))
print("variant", json.dumps(d["per_tile_fence_variant"]))
print("timeline", json.dumps(d["timeline_us"]))
PY
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 tools/nccl_baseline.py 2>&1 | grep '^{' | tee gpurun_out/nccl_n$N.json
