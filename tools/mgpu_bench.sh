# multi-GPU bench lines (+ parity check) on the GPUs of this box: N = 2 and, if present, 4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r02}
for N in ${NS:-2 4}; do
  [ $N -le $NG ] || continue
  PYTHONFAULTHANDLER=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2951$N \
    bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ep$N.log 2>&1
  grep '^{' gpurun_out/${TAG}_bench_ep$N.log | tail -1 > gpurun_out/${TAG}_bench_ep$N.json
  python - $N $TAG <<'PY'
import json, sys
N, tag = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/{tag}_bench_ep{N}.json"))
c = d["comm"]
print("EP", N, "K-step us", round(d["ms_per_step"] * 1e3, 1), "median us", round(d["timing_blocks"]["median_ms"] * 1e3, 1),
      "tok/s", int(d["value"]), "e2e", int(d["e2e"]["value"]), "clocks", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
print(" exposed", json.dumps(c["exposed"]), "ep1 twin", round(c["compute_only_twin_ep1"]["median_ms"] * 1e3, 1) if c["compute_only_twin_ep1"] else None)
print(" nvlink alg", json.dumps(c["nvlink_algorithmic_bytes_per_forward"]), "twins", json.dumps({k: v["median_ms"] for k, v in c["same_schedule_twins"].items() if isinstance(v, dict)}))
print(" per-tile", json.dumps({k: d["per_tile_fence_variant"][k] for k in ("ms_per_step", "fences_per_forward")}))
print(" auto-gs", json.dumps({k: d["auto_group_variant"][k] for k in ("ms_per_step", "group_size", "fences_per_forward")}) if d["auto_group_variant"] else None)
dv = d.get("dedup_variant")
print(" dedup", json.dumps({k: dv.get(k) for k in ("ms_per_step", "speedup_vs_this_run", "wire_bytes_ratio_vs_this_run", "fences_per_forward", "unavailable")}) if dv else None)
print(" roofline", json.dumps({k: d["roofline"].get(k) for k in ("bound", "frac", "launch_ms")}), json.dumps(d["layer_roofline"]["frac_of_max_compute_nvlink"]))
PY
done
# NCCL all-to-all baseline (bulk synchronous, precomputed splits, CUDA graph) at the same N
[ -n "$SKIP_NCCL" ] && exit 0
for N in ${NS:-2 4}; do
  [ $N -le $NG ] || continue
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N \
    tools/nccl_baseline.py > gpurun_out/${TAG}_nccl_ep$N.log 2>&1
  grep '^{' gpurun_out/${TAG}_nccl_ep$N.log | tail -1
done
