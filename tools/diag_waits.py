"""Where does the fused kernel's producer wait for dispatch data?  One traced
forward per rank (trace mode), then per-item GEMM1 waits split self/remote over
time.  torchrun --nproc-per-node N tools/diag_waits.py"""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch, torch.distributed as dist
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2605_00686_b200 as pb
    m = pb.ModelConfig("qwen3", 2048, 768, 128, 8)
    l = pb.MoELayer(m, 4096, rank=rank, world=world, device=local)
    if world > 1:
        l.connect_dist()
    x = torch.empty(4096, 2048, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(x)
    l.fill_synthetic_x(x, 1)
    for _ in range(5):
        l.forward(x, out)
    l.set_trace(True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l.forward(x, out)
    torch.cuda.synchronize()
    ev = l.trace()
    w = ev[ev["kind"] == 21]
    t0 = int(w["t"].min())
    selfw = w[w["peer"] == rank]
    remw = w[w["peer"] != rank]
    sr = ev[ev["kind"] == 20]
    res = {"rank": rank, "items_gemm1": int(len(w)),
           "self_wait_us_total": float(selfw["bytes"].sum()) / 1e3, "remote_wait_us_total": float(remw["bytes"].sum()) / 1e3,
           "self_ready_us": [round((int(t) - t0) / 1e3, 1) for t in np.percentile(sr["t"].astype(np.int64), [0, 25, 50, 75, 100])] if len(sr) else None,
           "waits_by_20us": {}}
    for arr, name in ((selfw, "self"), (remw, "remote")):
        b = ((arr["t"].astype(np.int64) - t0) // 20000).astype(int)
        for bi in np.unique(b):
            res["waits_by_20us"].setdefault(int(bi) * 20, {})[name] = round(float(arr["bytes"][b == bi].sum()) / 1e3, 1)
    allr = [None] * world
    if world > 1:
        dist.all_gather_object(allr, res)
    else:
        allr = [res]
    if rank == 0:
        for r in allr:
            print(json.dumps(r))
    l.set_trace(False)
    l.close()


if __name__ == "__main__":
    main()
