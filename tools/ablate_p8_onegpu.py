"""Signalling ablation at P = 8 (BASELINE configs[4]) without an 8-GPU box: the
8 EP ranks run CONCURRENTLY on one B200 (tests/gpu_util.run_concurrent: the
production fused CTA-pair kernel, 18 SMs per rank, no PDL).  What this
measures is the FENCE / SIGNAL accounting of the real device path at P = 8 —
per-PE dispatch and combine fences per forward vs the reference's accounting
of the same layout (ClusterConfig{8,1,1}, 128-row tiles).  The times are 8
ranks sharing one GPU's SMs and HBM, no NVLink: reported, not comparable.

    python tools/ablate_p8_onegpu.py [--out CSV]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"


def main():
    import torch
    import paper_2605_00686_b200 as pb
    from tests.gpu_util import run_concurrent

    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="256,1024,4096")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ablation_p8_onegpu.csv"))
    args = ap.parse_args()
    P = 8
    model = pb.model_preset("qwen3-30b")
    H = model.hidden_dim
    rows = []
    for S in [int(s) for s in args.tokens.split(",")]:
        wl = pb.build_dispatch(model, pb.ClusterConfig(P, 1, 1), S, 0.0, 128 * H * 2, 1)
        gs_auto = pb.resolve_group_size(model, S, P, protocol=pb.combined_protocol(-1))
        for name, proto in (("vanilla", pb.vanilla_protocol()), ("perseus", pb.combined_protocol(0)),
                            (f"auto_gs{gs_auto}", pb.combined_protocol(gs_auto))):
            layers, xs, outs = run_concurrent(pb, model, S, P, routing="balanced", seed=1, protocol=proto, reps=3)
            # time 10 more concurrent forwards (all ranks; one GPU)
            streams = [torch.cuda.Stream() for _ in range(P)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            for _ in range(10):
                for r, l in enumerate(layers):
                    l.forward(xs[r], outs[r], stream=streams[r])
                torch.cuda.synchronize()
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / 10 * 1e3
            for r, l in enumerate(layers):
                c = l.counters()
                assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
                ref = pb.expected_fences(proto, wl, r)
                own_bytes = sum(t.bytes for t in wl.remote_transfers if t.src_pe == r)
                rows.append((P, S, name, r, own_bytes, c["dispatch_fences"] / 13, c["combine_fences"] / 13, ref,
                             int(c["dispatch_fences"] == 13 * ref), us))
                l.close()
            r0 = [x for x in rows if x[1] == S and x[2] == name]
            print(f"P=8 S={S:6d} {name:12s} fences/PE dispatch {r0[0][5]:6.1f} (reference {r0[0][7]}) "
                  f"combine {r0[0][6]:6.1f}  match={all(x[8] for x in r0)}  {us:8.1f} us (8 ranks on one GPU)",
                  flush=True)
    with open(args.out, "w") as f:
        f.write("# schema=2 perseus-b200 signalling ablation at P=8, 8 ranks concurrently on ONE B200 (fence "
                "accounting; times are not NVLink timings)\n")
        f.write("P,S,mode,rank,bytes,dispatch_fences,combine_fences,reference_fences,match,us_per_forward_shared_gpu\n")
        for x in rows:
            f.write(",".join(str(v) for v in x) + "\n")
    print("wrote", args.out)


if __name__ == "__main__":
    main()
