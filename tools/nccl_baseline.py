"""NCCL all-to-all baseline of the same MoE-layer forward — the bulk-synchronous
design Perseus removes from the path, made fair:

  * routing is the bench's (balanced, workload.cpp:180-195), so the permutation
    and the all-to-all split sizes are computed ONCE on the host before timing —
    nothing in the timed forward synchronises with the host;
  * dispatch = one index_select + ncclAllToAllv (all_to_all_single with fixed
    splits), expert FFN = cuBLAS bf16 batched GEMMs (gate+up, SwiGLU, down) over
    the [local experts][rows][H] block, combine = ncclAllToAllv back + one
    index_copy + a batched weighted reduce;
  * the whole forward is captured in a CUDA graph (--no-graph to disable), so
    launch overhead is not what is measured;
  * identical bytes on NVLink to the fused kernel (2 * S*k*(P-1)/P * H * 2 per
    GPU per forward), same shape, CUDA-event timing, max over ranks.

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
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--H", type=int, default=2048)
    ap.add_argument("--I", type=int, default=768)
    ap.add_argument("--E", type=int, default=128)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--no-graph", action="store_true")
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
    ids = (torch.arange(S * k, device="cuda") % E).view(S, k)  # balanced routing
    wts = torch.softmax(logits.gather(1, ids), dim=1).to(torch.bfloat16).unsqueeze(1)  # [S, 1, k]

    # host-side plan, once (static routing): rows by (destination, expert)
    e = ids.reshape(-1)
    dst = e % P
    order = torch.argsort(dst * E + e, stable=True)
    src_tok = (order // k).contiguous()
    cnt = torch.bincount(dst, minlength=P)
    rcnt = torch.empty_like(cnt)
    dist.all_to_all_single(rcnt, cnt)
    sc, rc = cnt.tolist(), rcnt.tolist()
    per = sum(rc) // (P * El)  # balanced: equal rows per (source, local expert)
    send = torch.empty(S * k, H, device="cuda", dtype=torch.bfloat16)
    recv = torch.empty(sum(rc), H, device="cuda", dtype=torch.bfloat16)
    back = torch.empty_like(send)
    rows = torch.empty_like(send)
    out = torch.empty(S, H, device="cuda", dtype=torch.bfloat16)

    def forward():
        torch.index_select(x, 0, src_tok, out=send)
        dist.all_to_all_single(recv, send, rc, sc)                      # dispatch
        r = recv.view(P, El, per, H).transpose(0, 1).reshape(El, P * per, H)
        h = torch.bmm(r, w1)                                             # gate + up
        h = F.silu(h[..., :I]) * h[..., I:]
        y = torch.bmm(h, w2)                                             # down
        y = y.view(El, P, per, H).transpose(0, 1).reshape(-1, H)
        dist.all_to_all_single(back, y, sc, rc)                         # combine
        rows.index_copy_(0, order, back)
        torch.bmm(wts, rows.view(S, k, H), out=out.view(S, 1, H))       # weighted reduce

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            forward()
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            forward()
        torch.cuda.synchronize()
    run = graph.replay if graph is not None else forward
    with torch.cuda.stream(stream):
        for _ in range(3):
            run()
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record()
        for _ in range(args.steps):
            run()
        b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / args.steps], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ms = float(t.item())
        nvl = 2 * S * k * (P - 1) / P * H * 2
        print(json.dumps({"impl": "NCCL all_to_all_single x2 + cuBLAS bf16 bmm (PyTorch), precomputed splits, "
                                  + ("CUDA graph" if graph is not None else "eager"),
                          "n_gpus": P, "tokens_per_gpu": S, "shape": {"H": H, "I": I, "E": E, "k": k},
                          "ms_per_step": ms, "us_per_step": ms * 1e3, "value": P * S / (ms / 1e3),
                          "unit": "tokens/s", "steps": args.steps, "nvlink_bytes_per_gpu": nvl}), flush=True)
    # a captured graph holding NCCL work can hang process-group teardown: drop it
    # first, and leave without the interpreter's atexit teardown
    del graph
    torch.cuda.synchronize()
    dist.barrier()
    sys.stdout.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
