"""Generate tests/golden/reference_vectors.json from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libsigsim_ref.so, which
oracle/Makefile compiles from /root/reference/proj/src):

    python tests/golden/make_golden.py

Every value here is produced by the reference library itself (sigsim
build_dispatch / zipf_route / assign_groups / run_dispatch + fence_accounting,
verify_ordering, conservation_check).  The CPU tests pin the oracle
restatement (oracle/oracle.c) and the product planner to these vectors; the GPU
tests pin the device's layout / tile ids / fence counts to them.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import RefLib  # noqa: E402

# (name, H, I, E, k, P, S, skew, tile_rows)  — ClusterConfig{P,1,1} mapping
LAYOUTS = [
    ("tiny_p2", 256, 512, 8, 2, 2, 128, 0.0, 0),
    ("tiny_p2_tiles", 256, 512, 8, 2, 2, 128, 0.0, 16),
    ("tiny_p2_zipf1", 256, 512, 8, 2, 2, 128, 1.0, 0),
    ("tiny_p2_zipf1_tiles", 256, 512, 8, 2, 2, 128, 1.0, 16),
    ("tiny_p4_zipf15_tiles", 256, 512, 8, 2, 4, 256, 1.5, 32),
    ("small_p4_gs", 128, 128, 16, 4, 4, 64, 0.0, 8),
    ("qwen3_p2", 2048, 768, 128, 8, 2, 4096, 0.0, 128),
    ("qwen3_p4", 2048, 768, 128, 8, 4, 4096, 0.0, 128),
    ("qwen3_p8", 2048, 768, 128, 8, 8, 4096, 0.0, 0),
    ("qwen3_p8_tiles", 2048, 768, 128, 8, 8, 4096, 0.0, 128),
    ("qwen3_p8_zipf15", 2048, 768, 128, 8, 8, 4096, 1.5, 0),
    ("qwen3_p8_zipf15_tiles", 2048, 768, 128, 8, 8, 4096, 1.5, 128),
    ("llama4_p8", 5120, 8192, 16, 1, 8, 4096, 0.0, 0),
    ("llama4_p8_tiles", 5120, 8192, 16, 1, 8, 4096, 0.0, 128),
    ("dsv3_p8_tiles", 7168, 2048, 256, 8, 8, 4096, 0.0, 128),
]
# signalling ablation grid (BASELINE.json configs[4]): Qwen3, 128-row tiles
for P in (2, 4, 8):
    for S in (256, 1024, 4096, 16384):
        LAYOUTS.append((f"ablate_p{P}_s{S}", 2048, 768, 128, 8, P, S, 0.0, 128))

FULL_LIST_MAX = 64  # store the whole transfer list when it is this small


def main():
    ref = RefLib()
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj (sigsim)",
           "seed": 1, "kats": {}, "zipf": [], "layouts": []}
    k = out["kats"]
    k["remote_transfer_count"] = [[E, P, L, ref.remote_transfer_count(E, P, L)]
                                  for E, P, L in [(128, 16, 4), (128, 32, 4), (128, 16, 16),
                                                  (128, 8, 1), (128, 4, 1), (128, 2, 1),
                                                  (16, 8, 1), (256, 8, 1), (8, 2, 1)]]
    k["message_size"] = [[S, kk, E, H, ref.message_size(S, kk, E, H)]
                         for S, kk, E, H in [(1024, 8, 128, 2048), (1024, 4, 128, 2880),
                                             (0, 8, 128, 2048), (4096, 8, 128, 2048),
                                             (4096, 1, 16, 5120), (4096, 8, 256, 7168),
                                             (128, 2, 8, 256)]]
    for S, E, s, kk, seed in [(128, 8, 1.0, 2, 1), (1000, 64, 0.5, 4, 7), (1000, 64, 1.5, 4, 7),
                              (4096, 128, 1.5, 8, 12345), (5000, 32, 1.0, 4, 99),
                              (64, 8, 8.0, 1, 9), (100, 4, 0.0, 4, 3), (256, 16, 0.7, 3, 2)]:
        out["zipf"].append({"S": S, "E": E, "s": s, "k": kk, "seed": seed,
                            "counts": [int(c) for c in ref.zipf_route(S, E, s, kk, seed)]})
    for name, H, I, E, kk, P, S, skew, tile_rows in LAYOUTS:
        tb = tile_rows * H * 2
        rem, loc, dig = ref.build_dispatch(H, I, E, kk, P, 1, 1, S, skew, tb, 1)
        ent = {"name": name, "H": H, "I": I, "E": E, "k": kk, "P": P, "S": S, "skew": skew,
               "tile_rows": tile_rows, "tile_bytes": tb, "workload_digest": f"{dig:016x}",
               "n_remote": int(len(rem)), "n_local": int(len(loc)),
               "total_remote_bytes": int(rem[:, 3].sum()) if len(rem) else 0,
               "runs": {}}
        if len(rem) <= FULL_LIST_MAX:
            ent["remote"] = rem.tolist()
        # per-src tile ids / offsets checksum (cheap structural pin for big lists)
        ent["remote_checksum"] = f"{int((rem * [1, 3, 5, 7, 11, 13]).sum()) & ((1 << 64) - 1):016x}"
        modes = [("vanilla", 0), ("decoupled", 0), ("combined", 0), ("gpu_direct", 0)]
        n_src0 = int((rem[:, 0] == 0).sum()) if len(rem) else 0
        for gs in (2, 4, 8):
            if n_src0 and all(int((rem[:, 0] == p).sum()) % gs == 0 for p in range(P)):
                modes.append(("decoupled", gs))
        if S * P <= 4096 * 8 and not (S >= 16384):
            for mode, gs in modes:
                r = ref.run_dispatch(mode, gs, H, I, E, kk, P, 1, 1, S, skew, tb, 1, 1)
                ent["runs"][f"{mode}:{gs}"] = {
                    "heap_digest": f"{r['heap_digest']:016x}", "fence_count": r["fence_count"],
                    "fences_per_pe": r["fences_per_pe"],
                    "flagged_signal_count": r["flagged_signal_count"],
                    "n_violations": r["n_violations"],
                    "conservation_pass": r["conservation_pass"],
                    "n_signals_visible": r["n_signals_visible"]}
        out["layouts"].append(ent)
    path = os.path.join(HERE, "reference_vectors.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
