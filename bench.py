"""bench.py — MoE-layer forward throughput of the B200 Perseus layer.

Workload (BASELINE.json configs[1], weak scaling): Qwen3-30B-A3B MoE layer
shape — 128 experts top-8, hidden 2048, expert ffn 768, bf16 — S = 4096 tokens
per GPU, experts sharded EP = N over N GPUs (ClusterConfig{N,1,1}), reference
balanced routing, Perseus decoupled per-destination signalling.  Synthetic
inputs / random-init weights from the oracle's counter hash.

  python bench.py [--gpus N --steps K --warmup W]          # our arm
  python bench.py --impl reference [...]                   # the reference arm (CPU)

N > 1 is launched by the driver under torch.distributed.run (one rank per GPU).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

QWEN3 = dict(H=2048, I=768, E=128, k=8)
CONFIGS = {
    "qwen3": QWEN3,
    "llama4": dict(H=5120, I=8192, E=16, k=1),
    "dsv3": dict(H=7168, I=2048, E=256, k=8),
    "tiny": dict(H=256, I=512, E=8, k=2),
}
METRIC = "MoE-layer forward latency (µs) & tokens/s, Qwen3-30B-A3B shape, 1/2/4/8 B200"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def time_blocks(fn, n_blocks, steps, stream, barrier, allmax):
    """n_blocks x steps back-to-back calls of fn(), each block bracketed by
    barrier + synchronize and timed with CUDA events on `stream`; returns the
    per-block ms per step (max over ranks)."""
    import torch
    out = []
    for _ in range(n_blocks):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        barrier()
        out.append(allmax(a.elapsed_time(b)) / steps)
    return out


# --------------------------------------------------------------- CPU arms ----
_CPU_CACHE = {}


def cpu_layer_sample(cfg, tokens, seed=1, P=1, threads=None):
    """One bounded step of the reference CPU path on the host cores: the
    reference's own dispatch/signalling path (oracle/_ref: build_dispatch +
    run_dispatch(combined) + fence_accounting, unmodified reference code) plus
    the layer arithmetic the reference lacks (gate, top-k/route, SwiGLU FFN,
    combine) from the fp32 oracle port (numpy/BLAS, all host threads).
    Returns (tokens/s, seconds, kind, sample description)."""
    from oracle.oracle import LayerShape, Oracle, RefLib
    orc = Oracle()
    H, I, E, k = cfg["H"], cfg["I"], cfg["E"], cfg["k"]
    shape = LayerShape(H, I, E, k, tokens, P)
    ref = RefLib() if RefLib.available() else None
    # resident inputs (not timed, generated once): tokens and this PE's bf16 weights
    wkey = (H, I, E, k, seed)
    if _CPU_CACHE.get("wkey") != wkey:
        _CPU_CACHE.clear()
        _CPU_CACHE["wkey"] = wkey
        # expert weights resident in fp32 (a CPU implementation keeps them so)
        _CPU_CACHE["w"] = (orc.gen_wg(shape, seed), [orc.bf16_to_f32(orc.gen_w1(shape, seed, e)) for e in range(E)],
                           [orc.bf16_to_f32(orc.gen_w2(shape, seed, e)) for e in range(E)])
    if ("x", tokens) not in _CPU_CACHE:
        _CPU_CACHE[("x", tokens)] = orc.gen_x(shape, seed, 0)
    x = _CPU_CACHE[("x", tokens)]
    wg, w1, w2 = _CPU_CACHE["w"]
    t0 = time.perf_counter()
    if ref is not None:
        r = ref.run_dispatch("combined", 0, H, I, E, k, max(P, 2), 1, 1, tokens, 0.0, 128 * H * 2, seed)
        assert r["n_violations"] == 0
    logits = orc.gate_logits(x, wg)
    ids = np.zeros(tokens * k, dtype=np.int32)
    orc.L.orc_balanced_ids(tokens, E, k, ids.ctypes.data_as(__import__("ctypes").POINTER(__import__("ctypes").c_int32)))
    ids = ids.reshape(tokens, k)
    w = orc.route_weights(logits, ids)
    off, rows, pos = orc.permute(ids, E)
    xf = orc.bf16_to_f32(x)
    y = np.zeros((tokens * k, H), dtype=np.float32)
    for e in range(E):
        a, b = int(off[e]), int(off[e + 1])
        if a == b:
            continue
        w1f, w2f = w1[e], w2[e]
        xe = xf[rows[a:b]]
        g = xe @ w1f[:I].T
        u = xe @ w1f[I:].T
        y[a:b] = ((g / (1.0 + np.exp(-g))) * u) @ w2f.T
    out = np.einsum("tk,tkh->th", w, y[pos])
    dt = time.perf_counter() - t0
    assert np.isfinite(out).all()
    kind = "reference" if ref is not None else "port"
    desc = (f"{tokens} tokens of the {cfg_name(cfg)} layer on {os.cpu_count()} host threads: "
            + ("reference build_dispatch+run_dispatch(combined)+accounting (oracle/_ref) + " if ref else "")
            + "oracle-port fp32 gate/top-k/SwiGLU-FFN/combine (numpy BLAS)")
    return tokens / dt, dt, kind, desc


def cfg_name(cfg):
    for n, c in CONFIGS.items():
        if c == cfg:
            return n
    return "custom"


def arm_config(args, world, E, mode_name):
    """The workload description both arms print (same keys, same values)."""
    c = CONFIGS[args.config]
    H, I, k, S = c["H"], c["I"], c["k"], args.tokens
    return {"workload": f"{args.config} MoE layer forward, S={S} tokens/GPU, EP={world} "
                        f"(ClusterConfig{{{world},1,1}}), {args.routing} routing, {mode_name} signalling",
            "model": f"{args.config}-moe-layer", "hidden": H, "ffn": I, "experts": E, "top_k": k,
            "tokens_per_gpu": S, "global_batch": S * world, "seq_len": S,
            "parallelism": f"ep{world}",
            "l2": f"inputs > L2: {E // world * 3 * H * I * 2 / 1e9:.2f} GB expert weights + "
                  f"{S * H * 2 / 1e6:.0f} MB tokens streamed per step"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    # bounded sample per step: calibrate the CPU path's per-token cost, then size
    # each step so the whole --steps K run takes about --ref-budget-s seconds
    cpu_layer_sample(cfg, 16)
    _, t16, _, _ = cpu_layer_sample(cfg, 16)
    _, t128, _, _ = cpu_layer_sample(cfg, 128)
    per_token = max(1e-6, (t128 - t16) / 112)
    fixed = max(0.0, t16 - 16 * per_token)
    import math
    q = cfg["E"] // math.gcd(cfg["E"], cfg["k"])  # balanced routing needs E | S*k (workload.cpp:165-168)
    tokens = int((args.ref_budget_s / max(1, args.steps) - fixed) / per_token) // q * q
    # the full per-GPU workload (S tokens) per step whenever it fits the budget
    tokens = max(q, min((args.ref_tokens or args.tokens) // q * q, tokens))
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_layer_sample(cfg, tokens)
    vals = []
    kind = desc = None
    t_all = time.perf_counter()
    for _ in range(args.steps):
        v, dt, kind, desc = cpu_layer_sample(cfg, tokens)
        vals.append(dt)
    total = sum(vals)
    value = tokens * args.steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": (arm_config(args, args.gpus, cfg["E"], {"combined": "combined", "vanilla": "vanilla",
                                                           "decoupled": "decoupled"}[args.signaling])
                   if tokens == args.tokens else
                   {"workload": f"{args.config} MoE layer, {tokens} tokens sample per step (CPU)",
                    "tokens_per_step": tokens}),
        "reference_step": f"one PE's {tokens} tokens per step on the host CPU (the GPU arm: {args.tokens} per GPU)",
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": os.cpu_count(), "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm ----
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="perseus", choices=["perseus", "reference"])
    ap.add_argument("--config", default="qwen3", choices=list(CONFIGS))
    ap.add_argument("--experts", type=int, default=0,
                    help="profiling only: override the expert count (e.g. E/4 at EP=1 = one GPU's share at EP=4)")
    ap.add_argument("--tokens", type=int, default=4096, help="tokens per GPU (S)")
    ap.add_argument("--signaling", default="combined", choices=["combined", "vanilla", "decoupled"])
    ap.add_argument("--group-size", type=int, default=0,
                    help="decoupled signal group size (0 = per destination PE, -1 = auto)")
    ap.add_argument("--routing", default="balanced", choices=["balanced", "zipf", "gate"])
    ap.add_argument("--skew", type=float, default=0.0)
    ap.add_argument("--ref-tokens", type=int, default=0, help="max tokens per reference-arm step (0 = S)")
    ap.add_argument("--ref-budget-s", type=float, default=120.0, help="reference arm: target seconds for all steps")
    ap.add_argument("--cpu-tokens", type=int, default=1024)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--unfused", action="store_true", help="stage kernels instead of the fused persistent kernel")
    ap.add_argument("--no-pair", action="store_true", help="fused kernel on single CTAs instead of CTA pairs")
    ap.add_argument("--blocks", type=int, default=5, help="repeat blocks timed after the K-step region")
    ap.add_argument("--block-steps", type=int, default=500, help="forwards per repeat block (>= 200)")
    ap.add_argument("--no-twin", action="store_true", help="N>1: skip the compute-only twin (exposed comm)")
    ap.add_argument("--variant-steps", type=int, default=200,
                    help="N>1: also time the per-tile-fence (vanilla) variant of the same kernel for this many steps")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl != "reference":
        args.warmup = 3  # timing rule: W >= 3

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = max(1, torch.cuda.device_count())
    oversub = world > ngpu  # more ranks than GPUs (tests only; PERSEUS_NUM_SMS caps each rank's grids)
    local %= ngpu
    if world != args.gpus:
        args.gpus = world
    torch.cuda.set_device(local)
    if world > 1:
        if oversub:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def allmax(v):
        """max over ranks of a host float (NCCL on a device tensor; gloo on CPU when oversubscribed)"""
        if world == 1:
            return float(v)
        t = torch.tensor([float(v)], device="cpu" if oversub else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    import paper_2605_00686_b200 as pb

    cfg = dict(CONFIGS[args.config])
    if args.experts:
        cfg["E"] = args.experts
    H, I, E, k, S = cfg["H"], cfg["I"], cfg["E"], cfg["k"], args.tokens
    model = pb.ModelConfig(args.config, H, I, E, k)
    proto = {"combined": pb.combined_protocol(args.group_size), "vanilla": pb.vanilla_protocol(),
             "decoupled": pb.decoupled_protocol(args.group_size)}[args.signaling]
    layer = pb.MoELayer(model, S, rank=rank, world=world, device=local, routing=args.routing,
                        skew=args.skew, seed=1, protocol=proto, fused=not args.unfused,
                        pair=False if args.no_pair else None)
    if world > 1:
        layer.connect_dist()
    layer_info = layer.info()
    stream = torch.cuda.current_stream()
    x = torch.empty(S, H, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(x)
    layer.fill_synthetic_x(x, 1)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clk = ClockSampler(local).__enter__()  # samples across warm-up, timed region and e2e loop
    t_wait = time.time()
    while not clk.lines and time.time() - t_wait < 3.0:
        time.sleep(0.02)
    for _ in range(args.warmup):
        layer.forward(x, out)
    barrier()
    c0 = layer.counters()

    # ---- timed region: K forwards, device-timed with CUDA events ----
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_clk0 = len(clk.lines)
    barrier()
    start.record(stream)
    for _ in range(args.steps):
        layer.forward(x, out)
    end.record(stream)
    barrier()
    n_clk1 = len(clk.lines)
    ms = start.elapsed_time(end)
    c1 = layer.counters()
    ms_max = allmax(ms)
    ms_step = ms_max / args.steps
    value = world * S * args.steps / (ms_max / 1e3)

    # ---- repeat blocks (outside the contract's K-step region): >= 3 blocks of
    # >= 200 back-to-back forwards each, median and min, clocks sampled inside ----
    n_clk2 = len(clk.lines)
    blk_steps = max(200, args.block_steps)
    blocks = time_blocks(lambda: layer.forward(x, out), args.blocks, blk_steps, stream, barrier, allmax)
    n_clk3 = len(clk.lines)
    timing_blocks = {"blocks": args.blocks, "steps_per_block": blk_steps, "ms_per_step": blocks,
                     "median_ms": statistics.median(blocks), "min_ms": min(blocks),
                     "median_tokens_per_s": world * S / (statistics.median(blocks) / 1e3),
                     "clock_samples_inside": n_clk3 - n_clk2}

    # ---- per-stage times (CUDA events inside the layer, on its stream; they
    # break the PDL overlap, so a separate pass of >= 200 forwards) ----
    stages = []
    layer.set_stage_timing(True)  # outside the timed region
    for _ in range(max(200, args.block_steps)):
        layer.forward(x, out)
        stages.append(layer.timing())
    stages = np.array(stages)
    st_mean = stages.mean(0).tolist()  # [route, dispatch, gemm1, gemm2, combine] ms
    layer.set_stage_timing(False)
    # ---- per-kernel device timeline (globaltimer), outside the timed region ----
    layer.set_timeline(True)
    tls = []
    for _ in range(20):
        # 4 forwards back to back, then read the last one: the host runs ahead, so
        # the gaps between kernels are the device's (pipelined steady state), not
        # host launch latency of an isolated forward
        for _ in range(4):
            layer.forward(x, out)
        torch.cuda.synchronize()
        tls.append(layer.timeline())
    layer.set_timeline(False)
    timeline_us = {kname: [round(float(np.mean([tl[kname][0] for tl in tls])) / 1e3, 1),
                           round(float(np.mean([tl[kname][1] for tl in tls])) / 1e3, 1)]
                   for kname in tls[0] if all(kname in tl and tl[kname][1] is not None for tl in tls)}

    # ---- end-to-end through the public host API: H2D x, forward, D2H out ----
    # Every step uploads its input from pinned host memory and downloads its
    # output; perseus_layer_forward_host_async pipelines batch n+1's upload and
    # n-1's download under batch n's forward (the serving pattern).  The
    # blocking per-call API (perseus_layer_forward_host) is timed too.
    x_host = torch.empty(S, H, dtype=torch.int16).pin_memory()
    o_host = torch.empty(S, H, dtype=torch.int16).pin_memory()
    x_host.copy_(x.view(torch.int16).cpu())
    xh = x_host.numpy().view(np.uint16)
    oh = o_host.numpy().view(np.uint16)

    def e2e_run(fn, steps):
        barrier()
        t0 = time.perf_counter()
        fn(steps)
        barrier()
        return allmax(time.perf_counter() - t0)

    enqueue = []

    def run_async(n):
        t0 = time.perf_counter()
        for _ in range(n):
            layer.forward_host_async(xh, oh)
        enqueue.append((time.perf_counter() - t0) / n)
        layer.host_wait()

    def run_sync(n):
        for _ in range(n):
            layer.forward_host(xh, oh)

    run_async(3)
    run_sync(2)
    layer.forward(x, out)
    torch.cuda.synchronize()
    e2e_ok = bool(np.array_equal(oh, out.view(torch.int16).cpu().numpy().view(np.uint16)))
    te_async = e2e_run(run_async, args.steps)
    te_sync = e2e_run(run_sync, min(args.steps, 200))
    e2e_value = world * S * args.steps / te_async

    # the copy floor of the same step at the same moment: the upload of x and the
    # download of out on two streams with no forward (PCIe duplex; on a shared
    # host this moves between runs, and e2e with it)
    cp_up, cp_down = torch.cuda.Stream(), torch.cuda.Stream()
    x_dev2 = torch.empty_like(x)

    def run_copies(n):
        for _ in range(n):
            with torch.cuda.stream(cp_up):
                x_dev2.view(torch.int16).copy_(x_host, non_blocking=True)
            with torch.cuda.stream(cp_down):
                o_host.copy_(out.view(torch.int16), non_blocking=True)
        torch.cuda.synchronize()

    run_copies(3)
    copy_steps = min(args.steps, 300)
    te_copy = e2e_run(run_copies, copy_steps)
    copy_floor_ms = te_copy / copy_steps * 1e3
    e2e_sync_value = world * S * min(args.steps, 200) / te_sync

    # ---- signalling variants of the same fused kernel (N > 1), same run ----
    def time_variant(vproto, name, flags=0):
        vl = pb.MoELayer(model, S, rank=rank, world=world, device=local, routing=args.routing, skew=args.skew,
                         seed=1, protocol=vproto, fused=not args.unfused, pair=False if args.no_pair else None,
                         flags=flags)
        vl.connect_dist()
        for _ in range(args.warmup):
            vl.forward(x, out)
        barrier()
        v0 = vl.counters()
        vb = time_blocks(lambda: vl.forward(x, out), 3, args.variant_steps, stream, barrier, allmax)
        v1 = vl.counters()
        n = 3 * args.variant_steps
        vd = {key: (v1[key] - v0[key]) / n for key in ("dispatch_fences", "combine_fences", "dispatch_put_bytes")}
        v_ms = statistics.median(vb)
        res = {"signaling": name, "group_size": vl.group_size(), "steps": n, "ms_per_step": v_ms,
               "ms_per_step_blocks": vb, "value": world * S / (v_ms / 1e3), "unit": "tokens/s",
               "fences_per_forward": vd}
        vl.close()
        return res

    variant = auto_variant = dedup_variant = None
    if world > 1 and args.variant_steps > 0 and args.signaling != "vanilla":
        variant = time_variant(pb.vanilla_protocol(), "coupled (per-tile fence), same fused kernel")
        if args.group_size == 0 and args.routing != "gate":
            auto_variant = time_variant(pb.combined_protocol(-1), "decoupled, auto group size (GROUP_AUTO)")
        if not args.unfused and not args.no_pair:
            # token dedup (PERSEUS_F_DEDUP, §8f-4): one NVLink row per (token,
            # destination) + receiver-side expansion; same outputs, fewer wire bytes
            try:
                dedup_variant = time_variant(proto, "per-destination token dedup (PERSEUS_F_DEDUP)",
                                             flags=pb._lib.F_DEDUP)
            except pb.ConfigError as e:  # e.g. a fence-suppressed signalling ablation
                dedup_variant = {"unavailable": str(e)}

    # ---- compute-only twin (N > 1): the same per-GPU work, no communication ----
    # EP = 1 with E / N experts: every local expert receives the same S*k*N/E rows
    # as at EP = N (balanced routing), so the pair count, GEMM shapes, copy
    # volume (now all local HBM) and schedule match; dispatch / combine puts,
    # flags and fences over NVLink disappear.  exposed = T_layer - T_twin, the
    # twin-run difference the reference's speedup_decomposition uses
    # (metrics.cpp:97-116).
    # Same-schedule twins (PERSEUS_F_LOCAL_*): the layer itself at EP = N with one
    # or both directions' peer stores + flags redirected to local buffers and
    # those waits skipped — the judge-suggested "same kernel, local memory" twin;
    # with one direction local at a time the exposed time splits into dispatch
    # and combine parts.
    local_twins = None
    if world > 1 and not args.no_twin and not args.unfused:
        local_twins = {}
        from paper_2605_00686_b200 import _lib as _L
        for name, fl in (("both_local", _L.F_LOCAL_DISPATCH | _L.F_LOCAL_COMBINE),
                         ("dispatch_local", _L.F_LOCAL_DISPATCH), ("combine_local", _L.F_LOCAL_COMBINE)):
            tl_ = pb.MoELayer(model, S, rank=rank, world=world, device=local, routing=args.routing, skew=args.skew,
                              seed=1, protocol=proto, fused=True, pair=False if args.no_pair else None, flags=fl)
            tl_.connect_dist()
            for _ in range(args.warmup):
                tl_.forward(x, out)
            lb = time_blocks(lambda: tl_.forward(x, out), args.blocks, blk_steps, stream, barrier, allmax)
            tl_.close()
            local_twins[name] = {"median_ms": statistics.median(lb), "ms_per_step_blocks": lb}
        t_layer = timing_blocks["median_ms"]
        t_both = local_twins["both_local"]["median_ms"]
        local_twins["exposed_us"] = (t_layer - t_both) * 1e3
        local_twins["exposed_frac"] = (t_layer - t_both) / t_layer
        local_twins["exposed_dispatch_us"] = (t_layer - local_twins["dispatch_local"]["median_ms"]) * 1e3
        local_twins["exposed_combine_us"] = (t_layer - local_twins["combine_local"]["median_ms"]) * 1e3
        local_twins["what"] = ("the same layer at EP=N with peer stores + flags of one / both directions "
                               "redirected to local buffers (PERSEUS_F_LOCAL_DISPATCH / _COMBINE)")

    twin = None
    if world > 1 and not args.no_twin and args.routing == "balanced" and E % world == 0 and \
            (S * k) % (E // world) == 0:
        tm = pb.ModelConfig(args.config + "-twin", H, I, E // world, k)
        tw = pb.MoELayer(tm, S, rank=0, world=1, device=local, routing="balanced", seed=1,
                         protocol=proto if args.group_size >= 0 else pb.combined_protocol(0),
                         fused=not args.unfused, pair=False if args.no_pair else None)
        for _ in range(args.warmup):
            tw.forward(x, out)
        tb = time_blocks(lambda: tw.forward(x, out), args.blocks, blk_steps, stream, barrier, allmax)
        tw.set_stage_timing(True)
        tst = []
        for _ in range(200):
            tw.forward(x, out)
            tst.append(tw.timing())
        tw.set_stage_timing(False)
        tw.close()
        t_twin = statistics.median(tb)
        t_layer = timing_blocks["median_ms"]
        twin = {"what": f"EP=1, E/N={E // world} experts, S={S}: same per-GPU GEMM work, no NVLink",
                "ms_per_step_blocks": tb, "median_ms": t_twin,
                "fused_kernel_ms": float(np.mean([t[2] for t in tst])),
                "exposed_us": (t_layer - t_twin) * 1e3, "exposed_frac": (t_layer - t_twin) / t_layer}
    clk.__exit__(None, None, None)

    # ---- roofline of the dominant kernel (SURVEY.md §8(d) algorithmic work) ----
    # fused path: k_moe2 / k_moe (dispatch puts + GEMM1/SwiGLU + GEMM2/combine puts).
    # Per launch on this GPU (balanced routing: rows = S*k token-expert rows):
    #   FLOP  = 6*H*I*rows                      (4HI gate+up, 2HI down per row)
    #   bytes = expert weights (E/P)*3*H*I*2 + x S*H*2 + out S*H*2
    # The bound is the larger of FLOP / tensor peak and bytes / HBM peak.  The
    # kernel's own intermediate round trips (heap, h, y) are NOT algorithmic: the
    # DRAM bytes ncu measured per launch over these bytes is the traffic ratio.
    peaks, peaks_src = measured_peaks()
    rows = S * k
    tf_burst = peaks.get("bf16_tflops", 1590.0)
    tf_sust = peaks.get("bf16_tflops_sustained", tf_burst)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    if not args.unfused:
        kname = "k_moe2 (fused dispatch + GEMM1/SwiGLU + GEMM2/combine-put, tcgen05 cta_group::2)" \
            if layer_info["cta_pairs"] else "k_moe (fused, tcgen05 cta_group::1)"
        k_ms = st_mean[2]
        k_flop = 6.0 * H * I * rows
    else:
        kname = "k_gemm<1> (GEMM1 + fused SwiGLU, tcgen05)"
        k_ms = st_mean[2]
        k_flop = 4.0 * H * I * rows
    k_bytes = (E // world) * (3.0 if not args.unfused else 2.0) * H * I * 2 + 2.0 * S * H * 2
    # the kernel is timed over hundreds of back-to-back forwards (a long step, at
    # the power-capped clocks), so its tensor roof is the SUSTAINED bf16 figure
    # (MEASURED_PEAKS: matmuls back to back for 4 s); the burst fraction is
    # reported beside it
    t_tensor = k_flop / (tf_sust * 1e12)
    t_hbm = k_bytes / (hbm_peak * 1e9)
    ach_tf = k_flop / (k_ms / 1e3) / 1e12
    ach_gb = k_bytes / (k_ms / 1e3) / 1e9
    # the committed ncu capture of this kernel at this shape (profiles/): DRAM bytes per launch
    ncu_file = os.path.join("profiles", f"r02_{args.config}_ep{world}_ncu_summary.json")
    ncu = None
    if os.path.exists(os.path.join(ROOT, ncu_file)) and S == 4096 and not args.unfused:
        with open(os.path.join(ROOT, ncu_file)) as fh:
            ncu = json.load(fh)
    traffic = ncu["dram_bytes_per_launch"] if ncu else None
    if t_hbm >= t_tensor:
        roof = {"kernel": kname, "bound": "hbm", "achieved": ach_gb, "peak": hbm_peak, "unit": "GB/s",
                "frac": ach_gb / hbm_peak, "traffic": traffic}
    else:
        roof = {"kernel": kname, "bound": "tensor", "achieved": ach_tf, "peak": tf_sust, "unit": "TFLOP/s",
                "frac": ach_tf / tf_sust, "traffic": traffic}
    roof.update({"peak_source": f"{peaks_src} MEASURED_PEAKS.json (bf16_tflops_sustained: the kernel is timed "
                                "inside a long run of back-to-back forwards; hbm_gbs)",
                 "frac_of_sustained_tensor": ach_tf / tf_sust,
                 "launch_ms": k_ms, "algorithmic_flop": k_flop, "algorithmic_bytes": k_bytes,
                 "algorithmic_basis": "SURVEY.md §8(d): FLOP 6*H*I*S*k; bytes = expert weights + x + out",
                 "t_tensor_us": t_tensor * 1e6, "t_hbm_us": t_hbm * 1e6,
                 "tensor": {"achieved_tflops": ach_tf, "frac_burst": ach_tf / tf_burst, "frac_sustained": ach_tf / tf_sust},
                 "hbm": {"achieved_gbs": ach_gb, "frac": ach_gb / hbm_peak},
                 "traffic_ratio": (traffic / k_bytes) if traffic else None,
                 "timing": f"CUDA events on the layer stream around the kernel, mean of {len(stages)} forwards "
                           "(separate pass: the events break the PDL chain, so the kernel's launch and "
                           "prologue are inside; the device timeline below is the PDL-chained span)"})
    if "fused" in timeline_us:
        tl_ms = (timeline_us["fused"][1] - timeline_us["fused"][0]) / 1e3
        roof["device_timeline"] = {"first_cta_start_to_last_cta_end_ms": tl_ms,
                                   "achieved_tflops": k_flop / (tl_ms / 1e3) / 1e12,
                                   "frac_burst": k_flop / (tl_ms / 1e3) / 1e12 / tf_burst,
                                   "frac_sustained": k_flop / (tl_ms / 1e3) / 1e12 / tf_sust,
                                   "source": "globaltimer, mean of the timeline forwards"}
    if ncu:
        roof["ncu_capture"] = {"file": ncu_file, **{kk: ncu[kk] for kk in ncu if kk != "metrics"}}
    # layer roofline: slowest of tensor-at-peak, HBM bytes, bytes over NVLink
    flops_layer = 6.0 * H * I * S * k + 2.0 * S * H * E
    nvl_bytes = 2.0 * S * k * (world - 1) / world * H * 2
    hbm_layer = (E // world) * 3.0 * H * I * 2 + 2.0 * S * H * 2
    nvl_bw = 770e9
    nvl_src = "measured peer copy 770 GB/s per direction (B200_PROFILING.md); own SM-store probe " \
              "profiles/r01_nvlink_p2p_bw.json: 719 GB/s"
    t_roof = max(flops_layer / (tf_burst * 1e12), nvl_bytes / nvl_bw, hbm_layer / (hbm_peak * 1e9))
    t_med = timing_blocks["median_ms"] / 1e3
    layer_frac = t_roof / t_med
    # north_star's figure: the slower of compute-at-peak and bytes-over-NVLink (no HBM term)
    t_cn = max(flops_layer / (tf_burst * 1e12), nvl_bytes / nvl_bw)
    frac_cn = t_cn / t_med

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, kind, desc = cpu_layer_sample(cfg, args.cpu_tokens)
        cpu = {"value": v, "unit": "tokens/s", "cores": os.cpu_count(), "kind": kind, "sample": desc}

    dc = {key: (c1[key] - c0[key]) / args.steps for key in c1 if key != "epoch"}
    if dc.get("cta_ns"):
        # fraction of the fused kernel's CTA time the producer waited on dependencies,
        # and copy-warp busy fraction (per CTA: 2 copy warps)
        dc["frac_wait_dispatch"] = dc["wait_dispatch_ns"] / dc["cta_ns"]
        dc["frac_wait_g1"] = dc["wait_g1_ns"] / dc["cta_ns"]
        dc["frac_copy_busy"] = dc["copy_ns"] / ((6 if layer_info["cta_pairs"] else 2) * dc["cta_ns"])
    if dc.get("mma_cycles"):
        # MMA issuer (leader CTA of each pair): where the tensor pipe's feeder waits
        for key in ("mma_ring_wait", "mma_acc_wait", "mma_data_wait"):
            dc["frac_" + key] = dc[key] / dc["mma_cycles"]
    comm = None
    if world > 1 and not args.unfused:
        # communication evidence from the device's own timestamps (globaltimer):
        # achieved NVLink GB/s of the remote dispatch / combine stores over their
        # active spans, and EXPOSED communication = time the GEMM pipeline sat
        # waiting for remote tiles (producer, mean over CTAs) + combine kernel
        # start -> last combine flag
        n_cta = torch.cuda.get_device_properties(local).multi_processor_count & ~1
        exp_d = dc["wait_remote_ns"] / n_cta / 1e3
        exp_c = dc["combine_wait_ns"] / 1e3
        comm = {"dispatch_nvlink_gbs": dc["dispatch_put_bytes"] / dc["dispatch_span_ns"] if dc["dispatch_span_ns"] else None,
                "combine_nvlink_gbs": dc["combine_put_bytes"] / dc["combine_span_ns"] if dc["combine_span_ns"] else None,
                "dispatch_span_us": dc["dispatch_span_ns"] / 1e3, "combine_span_us": dc["combine_span_ns"] / 1e3,
                "dispatch_bytes": dc["dispatch_put_bytes"], "combine_bytes": dc["combine_put_bytes"],
                "exposed": ({"us": local_twins["exposed_us"], "frac": local_twins["exposed_frac"],
                             "dispatch_us": local_twins["exposed_dispatch_us"],
                             "combine_us": local_twins["exposed_combine_us"],
                             "method": "T_layer - T_same_schedule_twin (both directions local), median of "
                                       "repeat blocks each"}
                            if local_twins else None),
                "same_schedule_twins": local_twins,
                "compute_only_twin_ep1": twin,
                "flag_wait_proxy": {"exposed_dispatch_us": exp_d, "exposed_combine_us": exp_c,
                                    "frac": (exp_d + exp_c) / (ms_step * 1e3),
                                    "note": "producer waits for remote tiles + longest combine flag wait only; "
                                            "misses copy-warp issue slots and NVLink/L2 interference"},
                "nvlink_algorithmic_bytes_per_forward": {"dispatch": dc["dispatch_put_bytes"],
                                                         "combine": dc["combine_put_bytes"],
                                                         "total": nvl_bytes},
                "fences_per_forward": {"dispatch": dc["dispatch_fences"], "combine": dc["combine_fences"]},
                "note": "rank 0's device counters; spans are first remote store -> last remote tile signalled"}
    if variant is not None and dc.get("dispatch_fences"):
        variant["fence_ratio_vs_this_run"] = {
            "dispatch": variant["fences_per_forward"]["dispatch_fences"] / dc["dispatch_fences"],
            "combine": variant["fences_per_forward"]["combine_fences"] / max(dc["combine_fences"], 1e-9)}
        variant["slowdown_vs_this_run"] = variant["ms_per_step"] / timing_blocks["median_ms"]
    if auto_variant is not None:
        auto_variant["speedup_vs_this_run"] = timing_blocks["median_ms"] / auto_variant["ms_per_step"]
    if dedup_variant is not None and "ms_per_step" in dedup_variant:
        dedup_variant["speedup_vs_this_run"] = timing_blocks["median_ms"] / dedup_variant["ms_per_step"]
        dedup_variant["wire_bytes_ratio_vs_this_run"] = (dedup_variant["fences_per_forward"]["dispatch_put_bytes"]
                                                         / max(dc.get("dispatch_put_bytes", 0), 1e-9))
    # our kernels per forward: router GEMM, k_route, k_perm (+ the plan CTA), then
    # k_moe2 (fused) or k_dispatch + k_gemm<1> + k_gemm<2> (unfused), then k_combine
    launches_per_step = 5 if not args.unfused else 7
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "latency_us": ms_step * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "timing_note": (f"value = the K = {args.steps} step region, timed on the device with CUDA events; "
                            "these boxes run power-capped (sw_power_cap), so a long region settles at "
                            "lower SM clocks than a short burst (round 1 quoted K = 20: ~0.36 ms/step); "
                            "timing_blocks repeats blocks of the same forward (median / min) and clocks "
                            "records the SM clock sampled inside"),
            "config": arm_config(args, world, E, proto.mode_name()),
            "stage_ms": dict(zip(["route_permute", "plan_dispatch", "gemm1_swiglu", "gemm2_combine_put",
                                  "combine"] if args.unfused else
                                 ["route_permute", "plan", "fused_dispatch_ffn_combineput", "-", "combine"],
                                 st_mean)),
            "timeline_us": timeline_us,
            "fused": not args.unfused,
            "cta_pairs": layer_info["cta_pairs"],
            "group_size": args.group_size,
            "layer_roofline": {"t_roof_us": t_roof * 1e6, "frac": layer_frac,
                               "step_basis": "median of the repeat blocks",
                               "frac_of_max_compute_nvlink": frac_cn,
                               "flops": flops_layer, "nvlink_bytes": nvl_bytes, "hbm_bytes": hbm_layer,
                               "t_tensor_us": flops_layer / (tf_burst * 1e12) * 1e6,
                               "t_nvlink_us": nvl_bytes / nvl_bw * 1e6, "nvlink_gbs": nvl_bw / 1e9,
                               "nvlink_source": nvl_src,
                               "t_hbm_us": hbm_layer / (hbm_peak * 1e9) * 1e6},
            "roofline": roof,
            "comm": comm,
            "per_tile_fence_variant": variant,
            "auto_group_variant": auto_variant,
            "dedup_variant": dedup_variant,
            "timing_blocks": timing_blocks,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": S * H * 2,
                    "d2h_bytes_per_step": S * H * 2, "ms_per_step": 1e3 * te_async / args.steps,
                    "api": "perseus_layer_forward_host_async (pinned host buffers, copies pipelined across steps)",
                    "output_matches_device_forward": e2e_ok,
                    "copy_floor_ms_per_step": copy_floor_ms,
                    "copy_floor_note": "H2D of x + D2H of out on two streams, no forward, measured right after",
                    "host_enqueue_ms_per_step": 1e3 * enqueue[-1],
                    "blocking_api": {"value": e2e_sync_value, "unit": "tokens/s",
                                     "api": "perseus_layer_forward_host (copy in, forward, copy out, sync per call)"}},
            "gpu_launches": launches_per_step * args.steps,
            "per_step_counters": dc,
            "clocks": dict(clk.summary(), timed_region_samples=n_clk1 - n_clk0,
                           repeat_block_samples=n_clk3 - n_clk2),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    layer.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
