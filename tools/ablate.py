"""Signalling ablation on the Qwen3-30B-A3B shape (BASELINE.json configs[4]):
per-tile fences (vanilla / Coupled) vs Perseus per-destination batched fences
(Decoupled, group_size 0), plus fixed group sizes, for S in {256, 1K, 4K, 16K}
tokens per GPU at P GPUs — the B200 analogue of the reference's `cmd_ablate`
(proj/src/runner.cpp:301-344) with real device fences instead of simulated ones.

    python -m torch.distributed.run --nproc-per-node P tools/ablate.py [--out CSV]

For every point the device's fence / signal counters per forward are checked
against the reference's fence accounting of the same layout (ClusterConfig
{P,1,1}, 128-row tiles), and the forward time is measured with CUDA events
(max over ranks).  Rank 0 writes a versioned CSV (runner.cpp:29-58 style).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="256,1024,4096,16384")
    ap.add_argument("--modes", default="vanilla,perseus,auto,gsdiv",
                    help="vanilla | perseus (per destination) | auto (GROUP_AUTO) | gsN | gsdiv (every power-of-two divisor)")
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "ablation.csv"))
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2605_00686_b200 as pb

    model = pb.model_preset("qwen3-30b")
    H = model.hidden_dim
    rows = []
    for S in [int(s) for s in args.tokens.split(",")]:
        # the reference's layout and fence accounting for this point
        wl = pb.build_dispatch(model, pb.ClusterConfig(world, 1, 1), S, 0.0, 128 * H * 2, 1)
        n_own0 = sum(1 for t in wl.remote_transfers if t.src_pe == rank)
        modes = []
        for mode in args.modes.split(","):
            if mode == "gsdiv":  # group-size sweep over the divisors (assign_groups gs > 0)
                g = 2
                while g < n_own0:
                    if n_own0 % g == 0:
                        modes.append(f"gs{g}")
                    g *= 2
            else:
                modes.append(mode)
        for mode in modes:
            if mode == "vanilla":
                proto = pb.vanilla_protocol()
            elif mode == "perseus":
                proto = pb.combined_protocol(0)
            elif mode == "auto":  # PERSEUS_GROUP_AUTO, resolved on the host like the layer does
                proto = pb.combined_protocol(pb.resolve_group_size(model, S, world, protocol=pb.combined_protocol(-1)))
            else:
                proto = pb.combined_protocol(int(mode[2:]))
            n_own = sum(1 for t in wl.remote_transfers if t.src_pe == rank)
            if proto.signaling == "decoupled" and proto.group_size and n_own % proto.group_size:
                continue
            ref_f = pb.expected_fences(proto, wl, rank)
            layer = pb.MoELayer(model, S, rank=rank, world=world, device=local, protocol=proto)
            layer.connect_dist()
            x = torch.empty(S, H, dtype=torch.bfloat16, device="cuda")
            out = torch.empty_like(x)
            layer.fill_synthetic_x(x, 1)
            for _ in range(3):
                layer.forward(x, out)
            torch.cuda.synchronize()
            dist.barrier()
            c0 = layer.counters()
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            st.record()
            for _ in range(args.steps):
                layer.forward(x, out)
            en.record()
            torch.cuda.synchronize()
            ms = torch.tensor([st.elapsed_time(en) / args.steps], device="cuda")
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            c1 = layer.counters()
            d = {k: (c1[k] - c0[k]) / args.steps for k in c1}
            assert d["wait_timeouts"] == 0 and d["errors"] == 0, d
            own_bytes = sum(t.bytes for t in wl.remote_transfers if t.src_pe == rank)
            row = dict(P=world, S=S, mode=proto.mode_name() + (f"_gs{proto.group_size}" if proto.group_size else "")
                       + ("_auto" if mode == "auto" else ""),
                       bytes=own_bytes,
                       dispatch_fences=d["dispatch_fences"], combine_fences=d["combine_fences"],
                       ref_fences=ref_f, signals=d["dispatch_signals"], us=float(ms.item()) * 1e3,
                       tokens_per_s=world * S / (float(ms.item()) / 1e3),
                       match=int(d["dispatch_fences"] == ref_f))
            allrows = [None] * world
            dist.all_gather_object(allrows, row)
            if rank == 0:
                rows.append(allrows)
                r0 = allrows[0]
                print(f"P={world} S={S:6d} {r0['mode']:16s} fences/PE dispatch {r0['dispatch_fences']:6.1f} "
                      f"(reference {r0['ref_fences']}) combine {r0['combine_fences']:6.1f}  "
                      f"{r0['us']:8.1f} us  {r0['tokens_per_s'] / 1e6:6.2f} Mtok/s  match={all(a['match'] for a in allrows)}",
                      flush=True)
            layer.close()
            dist.barrier()
    if rank == 0:
        # alpha-beta fit per mode: forward time vs this PE's dispatch bytes over S
        # (fit_alpha_beta, metrics.cpp:69-95)
        fits = {}
        by_mode = {}
        for allrows in rows:
            r0 = allrows[0]
            by_mode.setdefault(r0["mode"], []).append((float(r0["bytes"]), r0["us"] * 1e3))
        for mode, pts in by_mode.items():
            if len({p[0] for p in pts}) >= 2:
                a, b, r2 = pb.fit_alpha_beta(pts)
                fits[mode] = {"alpha_us": a / 1e3, "beta_ns_per_byte": b, "GBps_equiv": (1.0 / b) if b > 0 else None,
                              "r_squared": r2, "points": len(pts)}
        fit_path = os.path.splitext(args.out)[0] + f"_fits_p{world}.json"
        with open(fit_path, "w") as fh:
            json.dump({"P": world, "fits": fits}, fh, indent=1)
        print("alpha-beta fits:", json.dumps(fits), flush=True)
        new = not os.path.exists(args.out)
        with open(args.out, "a") as f:
            if new:
                f.write("# schema=2 perseus-b200 signalling ablation (BASELINE configs[4]); per-PE fences per forward;"
                        " time = max over ranks, CUDA events; bytes = this PE's dispatch payload\n")
                f.write("P,S,mode,rank,bytes,dispatch_fences,combine_fences,reference_fences,match,us_per_forward,"
                        "tokens_per_s\n")
            for allrows in rows:
                for rk, a in enumerate(allrows):
                    f.write(f"{a['P']},{a['S']},{a['mode']},{rk},{a['bytes']},{a['dispatch_fences']:.0f},{a['combine_fences']:.0f},"
                            f"{a['ref_fences']},{a['match']},{a['us']:.1f},{a['tokens_per_s']:.0f}\n")
        print("wrote", args.out)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
