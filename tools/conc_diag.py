"""Diagnostics: P ranks concurrently on one GPU, per-rank counters + kernel
timelines, for a few grid caps.  Launched WITH programmatic dependent launch
(unlike tests/gpu_util.run_concurrent, which passes pdl=False) unless
DIAG_NO_PDL=1: with PDL a rank's grid waiting for its primary holds up the work
distributor and another rank's fused kernel stays unscheduled until the signal
waits time out (timeouts per rank in the output).
    python tools/conc_diag.py P CAP[,CAP...] ITERS TIMELINE(0|1|2)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
import torch  # noqa: E402

import paper_2605_00686_b200 as pb  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 4
caps = [int(c) for c in sys.argv[2].split(",")] if len(sys.argv) > 2 else [36, 32]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
use_tl = int(sys.argv[4]) if len(sys.argv) > 4 else 1
S = 1536 if P == 3 else 1024
m = pb.ModelConfig("qwen3", 2048, 768, 96 if P == 3 else 128, 8)
for cap in caps:
    os.environ["PERSEUS_NUM_SMS"] = str(cap)
    layers = [pb.MoELayer(m, S, rank=r, world=P, device=0, routing="balanced", seed=3,
                          protocol=(pb.decoupled_protocol(0) if os.environ.get("DIAG_PROTO") == "decoupled" else pb.combined_protocol(0)), pair=os.environ.get("DIAG_PAIR", "1") == "1",
                          pdl=os.environ.get("DIAG_NO_PDL", "0") != "1")
              for r in range(P)]
    pb.MoELayer.connect_local(layers)
    xs = [torch.empty(S, 2048, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    outs = [torch.zeros_like(x) for x in xs]
    for r, l in enumerate(layers):
        l.fill_synthetic_x(xs[r], 3)
        if use_tl:
            l.set_timeline(True)
        if os.environ.get("DIAG_TRACE") == "1":
            l.set_trace(True)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(P)]
    for it in range(iters):
        for r, l in enumerate(layers):
            l.forward(xs[r], outs[r], stream=streams[r])
        torch.cuda.synchronize()
        res = []
        t_all = None
        for r, l in enumerate(layers):
            c = l.counters()
            tl = l.timeline() if use_tl else {}
            if use_tl == 2:  # absolute globaltimer (PERSEUS_TL_KEEP=1: no per-forward reset)
                import ctypes as C
                n = len(l.TIMELINE_KERNELS)
                buf = (C.c_uint64 * (2 * n))()
                pb._lib.check(pb._lib.lib.perseus_layer_read_timeline(l._h, buf, n))
                tl = {name: (buf[2 * i], buf[2 * i + 1]) for i, name in enumerate(l.TIMELINE_KERNELS) if buf[2 * i]}
            if use_tl == 2:
                if t_all is None:
                    t_all = min(v[0] for ll in layers for v in [] ) if False else None
            res.append({"rank": r, "timeouts": c["wait_timeouts"], "errors": c["errors"],
                        "tl": tl if use_tl == 2 else {k: [round(v[0] / 1e3, 1), round(v[1] / 1e3, 1) if v[1] else None] for k, v in tl.items()}})
        if use_tl == 2:
            t0 = min(v[0] for rr in res for v in rr["tl"].values() if v[0])
            for rr in res:
                rr["tl"] = {k: [round((v[0] - t0) / 1e3, 1) if v[0] else None, round((v[1] - t0) / 1e3, 1) if v[1] else None]
                            for k, v in rr["tl"].items()}
        print(json.dumps({"cap": cap, "iter": it, "ranks": res}), flush=True)
    for l in layers:
        l.close()
