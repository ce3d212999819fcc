"""N>1 host logic on CPU (world_size 2, gloo): each rank synthesises the device
event log its kernels would record for its share of the reference layout
(puts, group fences, flag writes per assign_groups; receiver-side first
observations), the ranks all-gather events and realised transfers as
tests/mgpu_check.py does on GPUs, and rank 0 runs the C-ABI adapter
(perseus_trace_analyze -> sigsim::RunTrace -> the reference's
fence_accounting / verify_ordering / conservation_check).  Also the negative
cases: a tile seen before its data, a tile signalled twice."""
import os
import socket

import numpy as np
import pytest

import paper_2605_00686_b200 as pb
from paper_2605_00686_b200 import _lib

P = 2
MODEL = pb.ModelConfig("m", 256, 256, 8, 2)
S = 512


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _events_for_rank(rank, wl, proto, late_tile=None, dup_signal_tile=None):
    """The events rank `rank` records in one forward (device semantics of
    signal.cuh / moe2.cu): its remote puts, one fence per signal group, one flag
    write per member (the first after a fence carries it), and its first
    observation of every tile it receives."""
    ev = []
    t = 1000 * (rank + 1)
    own = [tr for tr in wl.remote_transfers if tr.src_pe == rank]
    gs = proto.group_size if proto.signaling == "decoupled" else 1
    groups = pb.assign_groups(own, gs) if proto.signaling == "decoupled" else \
        [pb.sigsim.SignalGroup(i, [i], i, 1) for i in range(len(own))]
    gof = {m: g.group_id for g in groups for m in g.members}
    for i, tr in enumerate(own):
        ev.append((t, _lib.EV_DISPATCH_PUT, rank, tr.dst_pe, tr.tile_id, gof[i], tr.bytes, 0))
        t += 10
    for g in groups:
        if not proto.suppress_fences:
            ev.append((t, _lib.EV_DISPATCH_FENCE, rank, own[g.members[0]].dst_pe, -1, g.group_id, 0, 0))
        for j, m in enumerate(g.members):
            ev.append((t + 1, _lib.EV_DISPATCH_SIGNAL, rank, own[m].dst_pe, own[m].tile_id, g.group_id, 0,
                       int(j == 0 and not proto.suppress_fences)))
        t += 10
    for tr in wl.remote_transfers:
        if tr.dst_pe == rank:
            late = tr.tile_id == late_tile
            ev.append((t, _lib.EV_DISPATCH_SEEN, rank, tr.src_pe, tr.tile_id, -1, 500 if late else 0, 0 if late else 1))
            if tr.tile_id == dup_signal_tile:  # the same tile's signal becomes visible a second time
                ev.append((t + 1, _lib.EV_DISPATCH_SEEN, rank, tr.src_pe, tr.tile_id, -1, 0, 1))
            t += 5
    arr = np.zeros(len(ev), dtype=[("t", np.uint64), ("kind", np.int32), ("pe", np.int32), ("peer", np.int32),
                                   ("tile", np.int32), ("group", np.int32), ("bytes", np.uint32),
                                   ("aux", np.uint32), ("pad", np.uint32)])
    for i, e in enumerate(ev):
        arr[i] = (*e, 0)
    return arr


CASES = ["vanilla", "combined", "decoupled_gs2", "late", "dup", "gpu_direct"]


def _worker(rank, port, q):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=P)
    try:
        out = {}
        for case in CASES:
            proto = {"vanilla": pb.vanilla_protocol(), "combined": pb.combined_protocol(0),
                     "decoupled_gs2": pb.decoupled_protocol(2), "late": pb.combined_protocol(0),
                     "dup": pb.vanilla_protocol(), "gpu_direct": pb.gpu_direct_protocol()}[case]
            skew = 0.0 if case == "decoupled_gs2" else 1.0  # balanced: gs=2 divides every PE's tile count
            wl = pb.build_dispatch(MODEL, pb.ClusterConfig(P, 1, 1), S, skew, 128 * MODEL.hidden_dim * 2, 5)
            late = wl.remote_transfers[0].tile_id if case == "late" else None
            dup = wl.remote_transfers[-1].tile_id if case == "dup" else None
            ev = _events_for_rank(rank, wl, proto, late_tile=late, dup_signal_tile=dup)
            own = np.array([(t.src_pe, t.dst_pe, t.expert, t.bytes, t.tile_id, t.heap_offset)
                            for t in wl.remote_transfers if t.src_pe == rank], dtype=np.int64).reshape(-1, 6)
            all_ev, all_tr = [None] * P, [None] * P
            dist.all_gather_object(all_ev, ev)
            dist.all_gather_object(all_tr, own)
            if rank == 0:
                rep = pb.analyze_trace(np.concatenate(all_ev), proto, np.concatenate(all_tr))
                want = sum(pb.expected_fences(proto, wl, s) for s in range(P))
                out[case] = (rep, want, int(np.concatenate(all_tr)[:, 3].sum()))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("case", ["vanilla", "combined", "decoupled_gs2", "gpu_direct"])
def test_two_rank_trace_adapter_matches_reference_accounting(results, case):
    rep, want, nbytes = results[case]
    d = rep["dispatch"]
    nic = case == "combined"
    if case == "gpu_direct":  # the reference records no fence markers and no flagged signals
        assert want == 0 and d["fence_count"] == 0 and d["flagged_signal_count"] == 0, d
    assert (d["flagged_signal_count"] if nic else d["fence_count"]) == want, (d, want)
    # NicFence: each group's fence marker arms its first signal's flag (both counted, as the reference)
    assert d["flagged_signal_count"] == (d["fence_count"] if nic else 0)
    assert d["ordering_violations"] == 0 and d["late_tiles"] == 0
    assert d["conservation_ok"], rep["conservation_error"]
    assert d["put_bytes"] == nbytes


def test_two_rank_trace_adapter_flags_a_signal_seen_before_its_data(results):
    d = results["late"][0]["dispatch"]
    assert d["late_tiles"] == 1 and d["ordering_violations"] == 1, d


def test_two_rank_trace_adapter_flags_a_tile_signalled_twice(results):
    rep = results["dup"][0]
    assert not rep["dispatch"]["conservation_ok"], rep
    err = rep["conservation_error"]
    assert "2 times" in err or "delivered bytes" in err, err


def test_device_trace_serializes_in_the_reference_format(results):
    """perseus_trace_serialize: the device RunTrace in sigsim::serialize_trace's text
    format (trace.cpp:33-51): header line, one record per line."""
    proto = pb.vanilla_protocol()
    wl = pb.build_dispatch(MODEL, pb.ClusterConfig(P, 1, 1), S, 1.0, 128 * MODEL.hidden_dim * 2, 5)
    ev = np.concatenate([_events_for_rank(r, wl, proto) for r in range(P)])
    text = pb.serialize_trace(ev, proto, 0)
    lines = text.strip().splitlines()
    assert lines[0].startswith("# trace v1 ")
    kinds = [ln.split()[2] for ln in lines[1:]]
    n_fence = sum(1 for ln in lines[1:] if ln.split()[3] == "fence")
    assert n_fence == results["vanilla"][1]
    assert len(lines) - 1 == len([e for e in ev if e["kind"] in (1, 2, 3)]) + 2 * len([e for e in ev if e["kind"] == 4])
    assert set(kinds) <= {"submit", "nic_service_start", "signal_visible", "completion"}, set(kinds)


@pytest.mark.parametrize("case", CASES + ["missing"])
def test_reference_checkers_agree_on_the_device_runtrace(case):
    """The RunTrace the adapter builds (perseus_trace_records) run through the
    UNMODIFIED reference checkers (oracle/_ref: fence_accounting,
    verify_ordering, conservation_check, metrics.cpp:10-59,118-190) gives the
    same fence markers, flagged signals, violations and conservation verdict
    (first failure message included) as libperseus' perseus_trace_analyze."""
    from oracle.oracle import RefLib
    from tests.trace_util import compare_checkers
    if not RefLib.available():
        pytest.skip("oracle/_ref not built")
    ref = RefLib()
    proto = {"vanilla": pb.vanilla_protocol(), "combined": pb.combined_protocol(0),
             "decoupled_gs2": pb.decoupled_protocol(2), "late": pb.combined_protocol(0),
             "dup": pb.vanilla_protocol(), "gpu_direct": pb.gpu_direct_protocol(),
             "missing": pb.vanilla_protocol()}[case]
    skew = 0.0 if case == "decoupled_gs2" else 1.0
    wl = pb.build_dispatch(MODEL, pb.ClusterConfig(P, 1, 1), S, skew, 128 * MODEL.hidden_dim * 2, 5)
    late = wl.remote_transfers[0].tile_id if case == "late" else None
    dup = wl.remote_transfers[-1].tile_id if case == "dup" else None
    ev = np.concatenate([_events_for_rank(r, wl, proto, late_tile=late, dup_signal_tile=dup) for r in range(P)])
    if case == "missing":  # one tile's put never observed at the receiver
        gone = wl.remote_transfers[1].tile_id
        ev = ev[~((ev["kind"] == _lib.EV_DISPATCH_SEEN) & (ev["tile"] == gone))]
    tr = np.array([(t.src_pe, t.dst_pe, t.expert, t.bytes, t.tile_id, t.heap_offset)
                   for t in wl.remote_transfers], dtype=np.int64).reshape(-1, 6)
    rep = compare_checkers(pb, ref, ev, proto, tr)
    if case == "late":
        assert rep["dispatch"]["ordering_violations"] == 1
    if case in ("dup", "missing"):
        assert not rep["dispatch"]["conservation_ok"]
    if case == "missing":
        assert "delivered bytes" in rep["conservation_error"], rep["conservation_error"]
        recs, n, sub, dlv = pb.trace_records(ev, proto, 0)
        assert f"put tile {gone} has no completion" in ref.analyze_records(recs, n, sub, dlv, tr)["failures"]
