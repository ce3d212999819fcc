"""Multi-GPU parity check: one process per GPU, launched by
`python -m torch.distributed.run --nproc-per-node P tests/mgpu_check.py`.

Every rank runs the real concurrent forward (dispatch puts and combine puts
over NVLink into cudaIpc-mapped symmetric buffers, ranks synchronising only
through device flag words), then checks — against the oracle and the
reference layout restatement — its routing, the realised dispatch layout
(tile ids, heap offsets), its flag words, its fence counts and its output.
Rank 0 prints one JSON line with the verdict.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    # more ranks than GPUs (oversubscribed run with PERSEUS_NUM_SMS capping each rank's grids)
    local = int(os.environ.get("LOCAL_RANK", rank)) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    import paper_2605_00686_b200 as pb
    from oracle.oracle import LayerShape, Oracle, transfers_to_np
    from tests.gpu_util import assert_close, bf16_bits

    orc = Oracle()
    from paper_2605_00686_b200 import _lib
    cases = [
        ("balanced", 0.0, pb.combined_protocol(0), 2048, 768, 128, 8, 4096, 0),  # the bench configuration
        ("balanced", 0.0, pb.combined_protocol(0), 2048, 768, 128, 8, 512, 0),
        ("balanced", 0.0, pb.vanilla_protocol(), 2048, 768, 128, 8, 512, 0),
        ("zipf", 1.2, pb.combined_protocol(0), 1024, 512, 16 * world, 4, 768, 0),
        ("gate", 0.0, pb.decoupled_protocol(0), 512, 256, 8 * world, 2, 1024, 0),
        # token dedup dispatch (PERSEUS_F_DEDUP): same outputs, its own fence accounting
        ("balanced", 0.0, pb.combined_protocol(0), 2048, 768, 128, 8, 4096, _lib.F_DEDUP),
        ("zipf", 1.2, pb.combined_protocol(0), 2048, 768, 128, 8, 1024, _lib.F_DEDUP),
    ]
    results = []
    ok = True
    for routing, skew, proto, H, I, E, k, S, lflags in cases:
        m = pb.ModelConfig("m", H, I, E, k)
        layer = pb.MoELayer(m, S, rank=rank, world=world, device=local, routing=routing, skew=skew,
                            seed=7, protocol=proto, pair=True, flags=lflags)  # the CTA-pair kernel even at small S
        layer.connect_dist()
        x = torch.empty(S, H, dtype=torch.bfloat16, device="cuda")
        out = torch.empty_like(x)
        layer.fill_synthetic_x(x, 7)
        for _ in range(3):  # repeated forwards flip the symmetric double buffers
            layer.forward(x, out)
        torch.cuda.synchronize()
        dist.barrier()
        r = {"routing": routing, "protocol": proto.mode_name() + ("+dedup" if lflags else ""), "rank": rank}
        try:
            c = layer.counters()
            assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
            table = layer.count_table()
            R, nr, _, _ = orc.layout_from_counts(table.astype(np.uint64), H, E, world, 1, 128 * H * 2)
            want = transfers_to_np(R, nr)
            sent, flags = layer.layout()
            assert np.array_equal(sent, want[want[:, 0] == rank]), "sent layout != reference"
            assert np.array_equal(np.sort(flags), np.sort(want[want[:, 1] == rank, 4])), "flags"
            own = want[want[:, 0] == rank]
            exp = orc.fences_for_src(own, rank, 0 if proto.signaling == "coupled" else 1, proto.group_size)
            per_fwd = c["dispatch_fences"] / 3
            if lflags:  # dedup: one fence per remote destination this rank sends to
                exp = len({int(t[1]) for t in own})
            assert per_fwd == exp, (per_fwd, exp)
            shape = LayerShape(H, I, E, k, S, world)
            ids, w, counts, pos = layer.routing()
            ref, ids_o, w_o = orc.layer_forward(shape, routing, 7, rank, skew)
            assert np.array_equal(ids, ids_o), "ids"
            got = orc.bf16_to_f32(bf16_bits(out))
            rel = assert_close(got, ref, what=f"{routing}/{proto.mode_name()} rank {rank}")
            r.update(ok=True, fences_per_forward=per_fwd, signals=c["dispatch_signals"] / 3,
                     rel_err=[float(rel[0]), float(rel[1])], n_sent=int(len(sent)))
        except AssertionError as e:
            ok = False
            r.update(ok=False, error=str(e)[:300])
        all_r = [None] * world
        dist.all_gather_object(all_r, r)
        results.append(all_r)
        layer.close()
        dist.barrier()
    # ---- device event log of real concurrent forwards -> the reference's RunTrace checks ----
    # Safe protocols must show no signal seen before its data; the fault-injection
    # variants (flags without the fence, transport.cpp:104-106; flags at put issue)
    # are reported.
    traces = []
    H, I, E, k, S = 2048, 768, 16 * world, 8, 2048
    for proto in (pb.combined_protocol(0), pb.vanilla_protocol(),
                  pb.ProtocolConfig(signaling="decoupled", ordering="nic_fence", suppress_fences=True),
                  pb.ProtocolConfig(signaling="coupled", suppress_fences=True),
                  pb.ProtocolConfig(fault_early_signal=True)):
        m = pb.ModelConfig("m", H, I, E, k)
        layer = pb.MoELayer(m, S, rank=rank, world=world, device=local, routing="balanced", seed=3, protocol=proto,
                            pair=True)
        layer.connect_dist()
        x = torch.empty(S, H, dtype=torch.bfloat16, device="cuda")
        out = torch.empty_like(x)
        layer.fill_synthetic_x(x, 3)
        layer.forward(x, out)
        layer.set_trace(True)
        reps = []
        for _ in range(5):
            torch.cuda.synchronize()
            dist.barrier()
            layer.forward(x, out)
            torch.cuda.synchronize()
            ev = [None] * world
            tr = [None] * world
            dist.all_gather_object(ev, layer.trace())
            dist.all_gather_object(tr, layer.layout()[0])
            if rank == 0:
                reps.append(pb.analyze_trace(np.concatenate(ev), proto, np.concatenate(tr)))
                if len(reps) == 1 and not proto.suppress_fences:
                    # one real forward's device RunTrace in the reference's text format
                    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
                    name = f"device_trace_{proto.mode_name()}_p{world}"
                    for d, tag in ((0, "dispatch"), (1, "combine")):
                        with open(os.path.join(ROOT, "gpurun_out", f"{name}_{tag}.txt"), "w") as fh:
                            fh.write(pb.serialize_trace(np.concatenate(ev), proto, d))
        layer.set_trace(False)
        layer.close()
        dist.barrier()
        if rank == 0:
            safe = not proto.suppress_fences and not proto.fault_early_signal
            viol = [r["dispatch"]["ordering_violations"] + r["combine"]["ordering_violations"] for r in reps]
            cons = all(r["dispatch"]["conservation_ok"] and r["combine"]["conservation_ok"] for r in reps)
            entry = {"protocol": proto.mode_name() + ("+no_fence" if proto.suppress_fences else "")
                     + ("+fault_early_signal" if proto.fault_early_signal else ""),
                     "forwards": len(reps), "violations": viol, "conservation": cons,
                     "dispatch": reps[-1]["dispatch"], "combine": reps[-1]["combine"]}
            if safe and (any(viol) or not cons):
                ok = False
                entry["ok"] = False
            if proto.fault_early_signal:
                # the checker must catch the signal-before-data fault in every forward
                entry["caught_fraction"] = sum(1 for v in viol if v > 0) / len(viol)
                if entry["caught_fraction"] < 1.0:
                    ok = False
                    entry["ok"] = False
            traces.append(entry)
    if rank == 0:
        verdict = ok and all(rr["ok"] for res in results for rr in res)
        print(json.dumps({"mgpu_check": "pass" if verdict else "FAIL", "world": world, "results": results,
                          "device_trace": traces}))
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
