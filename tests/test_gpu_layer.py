"""GPU parity of the CUDA layer against the oracle and the reference golden
vectors.  Every call goes through the C ABI (libperseus.so).

Bars (north_star): routing ids, token permutation, per-destination tile /
fence counts, tile ids and heap offsets bit-exact; layer output within bf16
tolerance (max-abs and normwise relative error <= 1e-2 vs the fp32 oracle).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TINY = dict(H=256, I=512, E=8, k=2)


def _pb():
    import paper_2605_00686_b200 as pb
    return pb


def _model(pb, H, I, E, k):
    return pb.ModelConfig("t", H, I, E, k)


def _check_rank(oracle, pb, shape, layer, x, out, routing, seed, skew, rank, subset=None):
    from tests.gpu_util import assert_close, bf16_bits
    ids, w, counts, pos = layer.routing()
    # x on device == oracle synthetic x, bit for bit
    xo = oracle.gen_x(shape, seed, rank)
    assert np.array_equal(bf16_bits(x), xo)
    ref_out, ids_o, w_o = oracle.layer_forward(shape, routing, seed, rank, skew, token_subset=subset)
    assert np.array_equal(ids, ids_o), "routing ids differ"
    assert np.abs(w - w_o).max() < 1e-5, "combine weights differ"
    off_o, rows_o, pos_o = oracle.permute(ids_o, shape.experts)
    assert np.array_equal(counts, np.diff(off_o).astype(np.int32)), "per-expert counts differ"
    assert np.array_equal(pos, pos_o), "token permutation differs"
    got = oracle.bf16_to_f32(bf16_bits(out))
    if subset is not None:
        got = got[subset]
    return assert_close(got, ref_out, what=f"rank {rank} {routing}")


@pytest.mark.parametrize("routing", ["balanced", "gate", "zipf"])
def test_tiny_single_rank(oracle, routing):
    from tests.gpu_util import run_emulated, shape_of
    pb = _pb()
    m = _model(pb, **TINY)
    S = 128
    layers, xs, outs = run_emulated(pb, m, S, 1, routing=routing, skew=1.0, seed=1)
    _check_rank(oracle, pb, shape_of(m, S, 1), layers[0], xs[0], outs[0], routing, 1, 1.0, 0)
    c = layers[0].counters()
    assert c["wait_timeouts"] == 0 and c["errors"] == 0
    assert c["dispatch_fences"] == 0  # one PE: nothing crosses NVLink


def test_forward_api_matches_phased(oracle):
    """perseus_layer_forward (all phases in one call) == phased path; repeated
    forwards (epoch parity flips) are stable."""
    import torch
    from tests.gpu_util import bf16_bits
    pb = _pb()
    m = _model(pb, **TINY)
    l = pb.MoELayer(m, 256, routing="gate", seed=3)
    x = torch.empty(256, 256, dtype=torch.bfloat16, device="cuda")
    l.fill_synthetic_x(x, 3)
    outs = []
    for _ in range(3):
        o = torch.empty_like(x)
        l.forward(x, o)
        torch.cuda.synchronize()
        outs.append(bf16_bits(o))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    host = l.forward_host(bf16_bits(x))
    assert np.array_equal(host, outs[0])


@pytest.mark.parametrize("P,routing,skew,proto", [
    (2, "balanced", 0.0, "vanilla"),
    (2, "balanced", 0.0, "combined"),
    (2, "zipf", 1.0, "combined"),
    (4, "gate", 0.0, "combined"),
    (4, "zipf", 1.5, "vanilla"),
    (8, "zipf", 0.7, "combined"),
])
def test_emulated_ranks_layout_fences_and_output(oracle, golden, P, routing, skew, proto):
    """P ranks emulated on one device: the realised dispatch layout (tile ids,
    heap offsets), flag words, fence counts and outputs vs the reference /
    oracle."""
    from tests.gpu_util import run_emulated, shape_of
    pb = _pb()
    E = 8 * P if P > 2 else 8
    m = _model(pb, 256, 256, E, 2)
    S = 256
    protocol = pb.vanilla_protocol() if proto == "vanilla" else pb.combined_protocol(0)
    layers, xs, outs = run_emulated(pb, m, S, P, routing=routing, skew=skew, seed=5, protocol=protocol)
    shape = shape_of(m, S, P)
    table = layers[0].count_table()
    for l in layers[1:]:
        assert np.array_equal(l.count_table(), table)
    # per-(src, expert) counts realised on the device == the reference routing
    if routing in ("balanced", "zipf"):
        ref_counts = oracle.route_counts(S, E, 2, skew, 5, P)
        assert np.array_equal(table.astype(np.uint64), ref_counts)
    tile_bytes = 128 * m.hidden_dim * 2
    R, nr, Lo, nl = oracle.layout_from_counts(table.astype(np.uint64), m.hidden_dim, E, P, 1, tile_bytes)
    from oracle.oracle import transfers_to_np
    want = transfers_to_np(R, nr)
    got = np.concatenate([l.layout()[0] for l in layers])
    got = got[np.lexsort((got[:, 4], got[:, 2], got[:, 1], got[:, 0]))]
    assert np.array_equal(got, want), "dispatch layout (tile ids / heap offsets) differs from the reference"
    flags = np.sort(np.concatenate([l.layout()[1] for l in layers]))
    assert np.array_equal(flags, np.sort(want[:, 4])), "flag words set != transfer tiles"
    hd_dev = pb.heap_digest(got[:, [1, 5, 3]], flags)
    assert hd_dev == oracle.heap_digest(want[:, [1, 5, 3]], want[:, 4])
    for r, l in enumerate(layers):
        c = l.counters()
        assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
        own = want[want[:, 0] == r]
        exp = oracle.fences_for_src(own, r, 0 if proto == "vanilla" else 1, 0)
        assert c["dispatch_fences"] == exp, (r, c, exp)
        assert c["dispatch_signals"] == len(own)
        assert c["combine_signals"] == int((want[:, 1] == r).sum())
        _check_rank(oracle, pb, shape, l, xs[r], outs[r], routing, 5, skew, r)


def test_reference_golden_fences_qwen3_p8_emulated(golden):
    """Qwen3-30B-A3B @ EP=8 (BASELINE configs[1]), 8 ranks emulated on one GPU:
    per-PE dispatch fences 224 (per tile, vanilla) vs 7 (per destination,
    Perseus) — the reference's own counts at ClusterConfig{8,1,1} with
    128-row tiles, and the digest of the realised heap."""
    from tests.gpu_util import run_emulated
    pb = _pb()
    g = next(l for l in golden["layouts"] if l["name"] == "qwen3_p8_tiles")
    m = pb.model_preset("qwen3-30b")
    for proto, key in ((pb.vanilla_protocol(), "vanilla:0"), (pb.combined_protocol(0), "combined:0")):
        layers, xs, outs = run_emulated(pb, m, 4096, 8, routing="balanced", seed=1, protocol=proto)
        got = np.concatenate([l.layout()[0] for l in layers])
        flags = np.concatenate([l.layout()[1] for l in layers])
        assert len(got) == g["n_remote"]
        assert f"{pb.heap_digest(got[:, [1, 5, 3]], flags):016x}" == g["runs"][key]["heap_digest"]
        fences = [l.counters()["dispatch_fences"] for l in layers]
        assert fences == g["runs"][key]["fences_per_pe"], (key, fences)
        for l in layers:
            c = l.counters()
            assert c["wait_timeouts"] == 0 and c["errors"] == 0
            l.close()


def test_qwen3_bench_config_every_token(oracle):
    """The bench workload exactly (Qwen3-30B-A3B shape, S=4096, EP=1, balanced
    routing, the fused CTA-pair kernel the bench times): routing bit-exact and
    ALL 4096 tokens' outputs vs the fp32 oracle, after repeated forwards."""
    import torch
    from tests.gpu_util import shape_of
    pb = _pb()
    m = pb.model_preset("qwen3-30b")
    S = 4096
    l = pb.MoELayer(m, S, routing="balanced", seed=1)
    assert l.info() == {"fused": True, "cta_pairs": True}
    x = torch.empty(S, m.hidden_dim, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(x)
    l.fill_synthetic_x(x, 1)
    for _ in range(3):
        l.forward(x, out)
    torch.cuda.synchronize()
    c = l.counters()
    assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
    _check_rank(oracle, pb, shape_of(m, S, 1), l, x, out, "balanced", 1, 0.0, 0)
    l.close()


@pytest.mark.parametrize("routing,pair", [("balanced", True), ("zipf", True), ("gate", True),
                                          ("balanced", False), ("zipf", False)])
def test_fused_kernel_bit_identical_to_stage_kernels(oracle, routing, pair):
    """The fused persistent kernel (dispatch + GEMM1 + GEMM2/combine-put, dynamic
    tile scheduler) computes exactly what the stage kernels compute."""
    import torch
    from tests.gpu_util import bf16_bits
    pb = _pb()
    m = pb.model_preset("qwen3-30b")
    S = 1024
    outs, cnts = [], []
    for fused in (True, False):
        l = pb.MoELayer(m, S, routing=routing, skew=1.1, seed=9, fused=fused, pair=pair)
        x = torch.empty(S, m.hidden_dim, dtype=torch.bfloat16, device="cuda")
        l.fill_synthetic_x(x, 9)
        o = torch.empty_like(x)
        for _ in range(3):
            l.forward(x, o)
        torch.cuda.synchronize()
        outs.append(bf16_bits(o))
        c = l.counters()
        assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
        cnts.append(c["recv_tiles"])
        l.close()
    assert np.array_equal(outs[0], outs[1])
    assert cnts[0] == cnts[1]


@pytest.mark.parametrize("preset,S,routing", [("llama4-scout", 2048, "balanced"),
                                               ("deepseek-v3", 1024, "balanced"),
                                               ("deepseek-v3", 512, "gate")])
def test_other_baseline_shapes_single_gpu(oracle, preset, S, routing):
    """BASELINE.json configs[2] (Llama4-Scout: 16 experts top-1, H 5120, ffn 8192)
    and configs[3] (DeepSeek-V3: 256 experts top-8, H 7168, ffn 2048) on the fused
    CTA-pair kernel: routing bit-exact, output vs the oracle on a token subset."""
    import torch
    from tests.gpu_util import shape_of
    pb = _pb()
    m = pb.model_preset(preset)
    l = pb.MoELayer(m, S, routing=routing, seed=4, pair=True)
    x = torch.empty(S, m.hidden_dim, dtype=torch.bfloat16, device="cuda")
    l.fill_synthetic_x(x, 4)
    out = torch.empty_like(x)
    for _ in range(2):
        l.forward(x, out)
    torch.cuda.synchronize()
    c = l.counters()
    assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
    subset = np.sort(np.random.default_rng(1).choice(S, 24, replace=False))
    _check_rank(oracle, pb, shape_of(m, S, 1), l, x, out, routing, 4, 0.0, 0, subset=subset)
    l.close()


@pytest.mark.gpu
def test_forward_host_async_pipeline_matches_blocking(oracle):
    """perseus_layer_forward_host_async: several batches in flight (two staging
    slots, upload/download streams) give exactly the blocking API's outputs."""
    import torch
    from tests.gpu_util import bf16_bits
    pb = _pb()
    m = _model(pb, **TINY)
    l = pb.MoELayer(m, 256, routing="gate", seed=5)
    xs, want = [], []
    for seed in range(4):
        x = torch.empty(256, 256, dtype=torch.bfloat16, device="cuda")
        l.fill_synthetic_x(x, 11 + seed)
        torch.cuda.synchronize()
        xb = np.ascontiguousarray(bf16_bits(x))
        xs.append(xb)
        want.append(l.forward_host(xb))
    outs = [np.zeros_like(xb) for xb in xs]
    for i in range(4):
        l.forward_host_async(xs[i], outs[i])
    l.host_wait()
    for i in range(4):
        assert np.array_equal(outs[i], want[i]), i
    l.close()


@pytest.mark.gpu
@pytest.mark.parametrize("P,proto", [(2, "vanilla"), (2, "combined"), (4, "decoupled"), (4, "combined")])
def test_device_trace_to_reference_runtrace(oracle, P, proto):
    """Device event log -> sigsim::RunTrace -> the reference's fence_accounting,
    verify_ordering and conservation_check (metrics.cpp:10-59,118-190): fence
    markers (ProxyFence) or flagged signals (NicFence) equal the reference's
    per-PE fence accounting of the realised layout, no signal is seen before
    its data, and every put tile is submitted, delivered and signalled once."""
    from tests.gpu_util import run_emulated
    pb = _pb()
    E = 8 * P if P > 2 else 8
    m = _model(pb, 256, 256, E, 2)
    protocol = {"vanilla": pb.vanilla_protocol(), "combined": pb.combined_protocol(0),
                "decoupled": pb.decoupled_protocol(0)}[proto]
    layers, xs, outs = run_emulated(pb, m, 256, P, routing="zipf", skew=1.0, seed=7, protocol=protocol,
                                    before=lambda ls: [l.set_trace(True) for l in ls])
    events = np.concatenate([l.trace() for l in layers])
    transfers = np.concatenate([l.layout()[0] for l in layers])
    rep = pb.analyze_trace(events, protocol, transfers)
    counters = [l.counters() for l in layers]
    nic = protocol.ordering == "nic_fence"
    for d, key in ((0, "dispatch"), (1, "combine")):
        dev_fences = sum(c[f"{key}_fences"] for c in counters)
        r = rep[key]
        assert (r["flagged_signal_count"] if nic else r["fence_count"]) == dev_fences, (key, r, dev_fences)
        # NicFence: each group's fence marker arms its first signal's flag (both counted, as the reference)
        assert r["flagged_signal_count"] == (r["fence_count"] if nic else 0), (key, r)
        assert r["ordering_violations"] == 0 and r["late_tiles"] == 0, (key, r)
        assert r["conservation_ok"], rep["conservation_error"]
        assert r["put_bytes"] == int(transfers[:, 3].sum())
    # dispatch fences vs the reference's accounting of the same layout
    tr = transfers[np.lexsort((transfers[:, 4], transfers[:, 2], transfers[:, 1], transfers[:, 0]))]
    mode = 0 if protocol.signaling == "coupled" else 1
    want = sum(oracle.fences_for_src(tr[tr[:, 0] == s], s, mode, 0) for s in range(P))
    got = rep["dispatch"]["flagged_signal_count" if nic else "fence_count"]
    assert got == want, (got, want)
    for l in layers:
        l.close()


@pytest.mark.gpu
@pytest.mark.parametrize("S,routing,pair", [(1000, "gate", True), (777, "zipf", None), (777, "gate", False)])
def test_fused_forward_ragged_token_counts(oracle, S, routing, pair):
    """Token counts that are not multiples of the 8-token route blocks, the 256-token
    permutation blocks or the combine's 2-token CTAs, through the fused forward
    (CTA-pair and 1-CTA kernels): routing bit-exact, output vs the oracle on a subset."""
    import torch
    from tests.gpu_util import shape_of
    pb = _pb()
    m = pb.model_preset("qwen3-30b")
    l = pb.MoELayer(m, S, routing=routing, skew=1.3, seed=6, pair=pair)
    x = torch.empty(S, m.hidden_dim, dtype=torch.bfloat16, device="cuda")
    out = torch.zeros_like(x)
    l.fill_synthetic_x(x, 6)
    for _ in range(2):
        l.forward(x, out)
    torch.cuda.synchronize()
    c = l.counters()
    assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
    subset = np.sort(np.concatenate([np.random.default_rng(1).choice(S - 8, 24, replace=False),
                                     np.arange(S - 8, S)]))  # incl. the ragged tail
    _check_rank(oracle, pb, shape_of(m, S, 1), l, x, out, routing, 6, 1.3, 0, subset=subset)
    l.close()


@pytest.mark.gpu
def test_c_abi_only_program(tmp_path):
    """A plain C program using only include/perseus.h (no Python, no torch) runs the
    layer end to end on the GPU: blocking and pipelined host APIs agree bit for bit."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "layer_c_abi")
    libdir = os.path.join(root, "paper_2605_00686_b200")
    subprocess.run(["gcc", "-std=c11", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "layer_c_abi.c"), "-L", libdir, "-lperseus",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "layer_c_abi: pass" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("routing", ["balanced", "zipf"])
def test_dataflow_combine_bit_identical(oracle, routing):
    """PERSEUS_F_DF_COMBINE (one PE): tokens combined inside the fused kernel as
    their rows complete give exactly the combine kernel's outputs and weights."""
    import torch
    from paper_2605_00686_b200 import _lib
    from tests.gpu_util import bf16_bits
    pb = _pb()
    m = pb.model_preset("qwen3-30b")
    S = 2048
    res = []
    for fl in (0, _lib.F_DF_COMBINE):
        l = pb.MoELayer(m, S, routing=routing, skew=1.1, seed=8, pair=True, flags=fl)
        x = torch.empty(S, m.hidden_dim, dtype=torch.bfloat16, device="cuda")
        o = torch.empty_like(x)
        l.fill_synthetic_x(x, 8)
        for _ in range(3):
            l.forward(x, o)
        torch.cuda.synchronize()
        c = l.counters()
        assert c["wait_timeouts"] == 0 and c["errors"] == 0, c
        res.append((bf16_bits(o), l.routing()[1]))
        l.close()
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])
