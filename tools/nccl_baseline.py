"""NCCL all-to-all baseline of the same MoE layer forward (what Perseus removes
from the path): route (balanced, as bench.py) -> sort rows by destination ->
NCCL all_to_all_single (counts, then rows) -> per-expert SwiGLU FFN as cuBLAS
bf16 batched GEMMs -> NCCL all_to_all_single back -> weighted combine.  Same
shape, synthetic data and timing rules as bench.py (CUDA events, K forwards,
max over ranks); prints one JSON line on rank 0.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/nccl_baseline.py
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import torch.nn.functional as F

    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--H", type=int, default=2048)
    ap.add_argument("--I", type=int, default=768)
    ap.add_argument("--E", type=int, default=128)
    ap.add_argument("--k", type=int, default=8)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    S, H, I, E, k, P = args.tokens, args.H, args.I, args.E, args.k, world
    El = E // P
    g = torch.Generator(device="cuda").manual_seed(1 + rank)
    x = torch.randn(S, H, device="cuda", dtype=torch.bfloat16, generator=g)
    w1 = (torch.randn(El, H, 2 * I, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(El, I, H, device="cuda", generator=g) / I ** 0.5).to(torch.bfloat16)
    logits = torch.randn(S, E, device="cuda", generator=g)
    flat = torch.arange(S * k, device="cuda")
    ids = (flat % E).view(S, k)                       # balanced routing (workload.cpp:180-195)
    wts = torch.softmax(logits.gather(1, ids), dim=1)  # combine weights

    def forward():
        e = ids.reshape(-1)
        dst = e % P
        order = torch.argsort(dst * E + e, stable=True)  # by destination, then expert
        send = x[order // k]
        cnt = torch.bincount(dst, minlength=P)
        rcnt = torch.empty_like(cnt)
        dist.all_to_all_single(rcnt, cnt)               # count exchange
        sc, rc = cnt.tolist(), rcnt.tolist()
        recv = torch.empty(sum(rc), H, device="cuda", dtype=torch.bfloat16)
        dist.all_to_all_single(recv, send, rc, sc)      # dispatch
        # received rows are (src, expert)-ordered; balanced routing => equal rows per
        # local expert per source: regroup to [El, rows, H] and run the FFN as bmm
        per = recv.shape[0] // (P * El)
        r = recv.view(P, El, per, H).transpose(0, 1).reshape(El, P * per, H)
        h = torch.bmm(r, w1)
        h = F.silu(h[..., :I]) * h[..., I:]
        y = torch.bmm(h, w2)
        y = y.view(El, P, per, H).transpose(0, 1).reshape(-1, H).contiguous()
        back = torch.empty_like(send)
        dist.all_to_all_single(back, y, sc, rc)        # combine
        out_rows = torch.empty_like(back)
        out_rows[order] = back
        return (out_rows.view(S, k, H).float() * wts.unsqueeze(-1)).sum(1).to(torch.bfloat16)

    for _ in range(args.warmup):
        forward()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.steps):
        forward()
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / args.steps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t.item())
        print(json.dumps({"impl": "nccl_all_to_all + cuBLAS bmm (PyTorch)", "n_gpus": P, "tokens_per_gpu": S,
                          "shape": {"H": H, "I": I, "E": E, "k": k}, "ms_per_step": ms,
                          "value": P * S / (ms / 1e3), "unit": "tokens/s", "steps": args.steps}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
