"""The oracle (oracle/oracle.c) pinned against the reference's golden vectors
(tests/golden/reference_vectors.json, generated from the UNMODIFIED reference
by tests/golden/make_golden.py) and, where oracle/_ref is built, against the
reference library live.  CPU only."""
import numpy as np
import pytest

from oracle.oracle import RefLib


def test_kats(oracle, golden):
    for E, P, L, want in golden["kats"]["remote_transfer_count"]:
        assert oracle.remote_transfer_count(E, P, L) == want
    for S, k, E, H, want in golden["kats"]["message_size"]:
        assert oracle.message_size(S, k, E, H) == want
    # test_workload.cpp:9-20 literal KATs
    assert oracle.remote_transfer_count(128, 16, 4) == 96
    assert oracle.remote_transfer_count(128, 32, 4) == 112
    assert oracle.remote_transfer_count(128, 16, 16) == 0
    with pytest.raises(ValueError):
        oracle.remote_transfer_count(100, 16, 4)
    assert oracle.message_size(1024, 8, 128, 2048) == 262144


def test_zipf_counts_match_reference(oracle, golden):
    for z in golden["zipf"]:
        c, ids = oracle.zipf_route(z["S"], z["E"], z["s"], z["k"], z["seed"], want_ids=True)
        assert c.tolist() == z["counts"]
        # the per-token ids are the same draws: they re-count to the reference counts
        assert np.bincount(ids, minlength=z["E"]).tolist() == z["counts"]
        # k distinct experts per token
        per_tok = ids.reshape(z["S"], z["k"])
        assert all(len(set(r)) == z["k"] for r in per_tok[:200])


@pytest.mark.parametrize("idx", range(0, 27))
def test_layout_and_digests_match_reference(oracle, golden, idx):
    if idx >= len(golden["layouts"]):
        pytest.skip("no such layout")
    g = golden["layouts"][idx]
    rem, loc, dig = oracle.build_dispatch(g["H"], g["E"], g["k"], g["P"], 1, g["S"], g["skew"],
                                          g["tile_bytes"], 1)
    assert f"{dig:016x}" == g["workload_digest"]
    assert len(rem) == g["n_remote"] and len(loc) == g["n_local"]
    assert int(rem[:, 3].sum()) == g["total_remote_bytes"]
    assert f"{int((rem * [1, 3, 5, 7, 11, 13]).sum()) & ((1 << 64) - 1):016x}" == g["remote_checksum"]
    if "remote" in g:
        assert rem.tolist() == g["remote"]
    hd = oracle.heap_digest(rem[:, [1, 5, 3]], rem[:, 4])
    for key, run in g["runs"].items():
        mode, gs = key.split(":")
        gs = int(gs)
        assert f"{hd:016x}" == run["heap_digest"], key
        per_pe = [oracle.fences_for_src(rem, s, 0 if mode == "vanilla" else 1, gs,
                                        gpu_direct=mode.startswith("gpu_direct"))
                  for s in range(g["P"])]
        assert per_pe == run["fences_per_pe"], key
        assert run["n_violations"] == 0 and run["conservation_pass"] == 1


def test_assign_groups_reference_case(oracle):
    # test_protocols.cpp:64-88
    t = np.array([(0, 4 + e % 28, e, 64, e, 0) for e in range(112)], dtype=np.int64)
    for gs, n in [(1, 112), (28, 4), (112, 1)]:
        _, leaders = oracle.assign_groups(t, gs)
        assert len(leaders) == n
    gof, leaders = oracle.assign_groups(t, 0)
    assert len(leaders) == 28
    for g in range(28):
        members = np.nonzero(gof == g)[0]
        assert len(members) == 4 and len(set(t[members, 1])) == 1
        assert leaders[g] == members[np.lexsort((t[members, 4], t[members, 2], t[members, 1]))][0]
    with pytest.raises(ValueError):
        oracle.assign_groups(t, 5)


def test_synthetic_tensor_determinism(oracle):
    a = oracle.fill_bf16(1, 1, 0, 1000, 1.7320508)
    b = oracle.fill_bf16(1, 1, 0, 1000, 1.7320508)
    c = oracle.fill_bf16(2, 1, 0, 1000, 1.7320508)
    assert np.array_equal(a, b) and not np.array_equal(a, c)
    # sub-range addressing is consistent
    assert np.array_equal(oracle.fill_bf16(1, 1, 500, 500, 1.7320508), a[500:])
    f = oracle.bf16_to_f32(a)
    assert abs(f.mean()) < 0.15 and 0.8 < f.var() < 1.2


def test_permute_is_stable_counting_sort(oracle):
    rng = np.random.default_rng(0)
    ids = np.stack([rng.permutation(16)[:4] for _ in range(50)]).astype(np.int32)
    off, rows, pos = oracle.permute(ids, 16)
    for e in range(16):
        seg = rows[off[e]:off[e + 1]]
        assert np.all(np.diff(seg) > 0)
        assert sorted(seg.tolist()) == sorted(np.nonzero((ids == e).any(1))[0].tolist())
    for t in range(50):
        for j in range(4):
            assert rows[pos[t, j]] == t and off[ids[t, j]] <= pos[t, j] < off[ids[t, j] + 1]


def test_gate_topk_ties_to_lower_index(oracle):
    logits = np.array([[1.0, 3.0, 3.0, 2.0, 3.0]], dtype=np.float32)
    assert oracle.topk(logits, 3).tolist() == [[1, 2, 4]]


@pytest.mark.skipif(not RefLib.available(), reason="oracle/_ref not built")
def test_oracle_against_live_reference(oracle):
    ref = RefLib()
    for (H, I, E, k, P, S, skew, tb) in [(256, 512, 8, 2, 2, 128, 0.7, 256 * 32 * 2),
                                          (128, 128, 16, 4, 4, 96, 1.2, 0),
                                          (512, 256, 32, 2, 8, 512, 0.0, 512 * 64 * 2)]:
        rr, rl, rd = ref.build_dispatch(H, I, E, k, P, 1, 1, S, skew, tb, 3)
        orr, orl, od = oracle.build_dispatch(H, E, k, P, 1, S, skew, tb, 3)
        assert rd == od and np.array_equal(rr, orr) and np.array_equal(rl, orl)
        for s in range(P):
            gof_r, lead_r = ref.assign_groups(rr[rr[:, 0] == s], 0)
            gof_o, lead_o = oracle.assign_groups(rr[rr[:, 0] == s], 0)
            assert np.array_equal(gof_r, gof_o) and np.array_equal(lead_r, lead_o)
