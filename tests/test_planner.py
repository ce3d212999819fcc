"""The product's host planner (libperseus.so C ABI, mirrored by
paper_2605_00686_b200.sigsim) against the reference golden vectors and the
reference's own doctest cases (proj/tests/test_workload.cpp,
test_protocols.cpp).  Also: the C-ABI library loads and exports every symbol
include/perseus.h declares.  CPU only — no compute is launched."""
import os
import re

import numpy as np
import pytest

import paper_2605_00686_b200 as pb
from paper_2605_00686_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "perseus.h")).read()
    decl = set(re.findall(r"\b(perseus_[a-z0-9_]+)\s*\(", hdr))
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(_lib.lib, name), name
    assert _lib.lib.perseus_abi_version() == 1


def test_workload_kats():
    # test_workload.cpp:9-20
    assert pb.remote_transfer_count(128, 16, 4) == 96
    assert pb.remote_transfer_count(128, 32, 4) == 112
    assert pb.remote_transfer_count(128, 16, 16) == 0
    with pytest.raises(pb.ConfigError):
        pb.remote_transfer_count(100, 16, 4)
    assert pb.message_size(1024, 8, 128, 2048) == 262144
    assert pb.message_size(1024, 4, 128, 2880) == 184320
    assert pb.message_size(0, 8, 128, 2048) == 0


def test_zipf_matches_reference_golden(golden):
    for z in golden["zipf"]:
        assert pb.zipf_route(z["S"], z["E"], z["s"], z["k"], z["seed"]).tolist() == z["counts"]


def test_zipf_properties():
    # test_workload.cpp:22-62
    for s in (0.0, 0.5, 1.0, 1.5):
        assert pb.zipf_route(1000, 64, s, 4, 7).sum() == 4000
    c = pb.zipf_route(100000, 4, 1.0, 1, 3)
    assert 0.47 < c.max() / 100000 < 0.49
    c = np.sort(pb.zipf_route(200000, 128, 1.5, 1, 5))[::-1]
    assert 0.79 < c[:10].sum() / 200000 < 0.85
    a, b = pb.zipf_route(5000, 32, 1.0, 4, 99), pb.zipf_route(5000, 32, 1.0, 4, 99)
    assert np.array_equal(a, b) and not np.array_equal(a, pb.zipf_route(5000, 32, 1.0, 4, 100))
    counts, ids = pb.zipf_route(300, 16, 1.2, 4, 11, want_ids=True)
    assert np.bincount(ids, minlength=16).tolist() == counts.tolist()


def test_build_dispatch_reference_cases():
    q = pb.model_preset("qwen3-30b")
    wl = pb.build_dispatch(q, pb.ClusterConfig(4, 4, 1), 1024, 0.0, 0, 1)
    pe0 = [t for t in wl.remote_transfers if t.src_pe == 0]
    assert len(pe0) == 96 and all(t.bytes == 262144 for t in pe0)
    assert sum(t.src_pe == 0 for t in wl.local_transfers) == 3 * (128 // 16)
    wl = pb.build_dispatch(q, pb.ClusterConfig(4, 4, 1), 1024, 0.0, 16384, 1)
    pe0 = [t for t in wl.remote_transfers if t.src_pe == 0]
    assert len(pe0) == 96 * 16 and all(t.bytes == 16384 for t in pe0)
    with pytest.raises(pb.ConfigError):
        pb.build_dispatch(q, pb.ClusterConfig(4, 4, 1), 1000, 0.0, 0, 1)
    pb.build_dispatch(q, pb.ClusterConfig(4, 4, 1), 1000, 0.5, 0, 1)
    tiny = pb.ModelConfig("tiny", 64, 64, 8, 1)
    wl = pb.build_dispatch(tiny, pb.ClusterConfig(2, 1, 1), 64, 8.0, 0, 9)
    assert all(t.bytes > 0 for t in wl.remote_transfers)
    # single node: no remote transfers at all (test_protocols.cpp:161-169)
    assert not pb.build_dispatch(q, pb.ClusterConfig(1, 4, 1), 1024, 0.0, 0, 1).remote_transfers


def test_build_dispatch_matches_golden(golden):
    for g in golden["layouts"]:
        m = pb.ModelConfig("g", g["H"], g["I"], g["E"], g["k"])
        wl = pb.build_dispatch(m, pb.ClusterConfig(g["P"], 1, 1), g["S"], g["skew"], g["tile_bytes"], 1)
        assert f"{wl.digest():016x}" == g["workload_digest"], g["name"]
        rem = wl.remote_array()
        assert len(rem) == g["n_remote"]
        assert f"{int((rem * [1, 3, 5, 7, 11, 13]).sum()) & ((1 << 64) - 1):016x}" == g["remote_checksum"]
        hd = pb.heap_digest(rem[:, [1, 5, 3]], rem[:, 4])
        for key, run in g["runs"].items():
            mode, gs = key.split(":")
            assert f"{hd:016x}" == run["heap_digest"]
            proto = {"vanilla": pb.vanilla_protocol(), "decoupled": pb.decoupled_protocol(int(gs)),
                     "combined": pb.combined_protocol(int(gs)),
                     "gpu_direct": pb.gpu_direct_protocol()}[mode]
            assert [pb.expected_fences(proto, wl, s) for s in range(g["P"])] == run["fences_per_pe"], (g["name"], key)


def test_assign_groups_reference_case():
    ts = [pb.TransferSpec(0, 4 + e % 28, e, 64, e, 0) for e in range(112)]
    assert len(pb.assign_groups(ts, 1)) == 112
    assert len(pb.assign_groups(ts, 28)) == 4
    assert len(pb.assign_groups(ts, 112)) == 1
    groups = pb.assign_groups(ts, 0)
    assert len(groups) == 28
    for g in groups:
        assert len(g.members) == 4 and g.leader == g.members[0]
        assert len({ts[m].dst_pe for m in g.members}) == 1
    with pytest.raises(pb.ConfigError):
        pb.assign_groups(ts, 5)


def test_planner_agrees_with_oracle_on_random_layouts(oracle):
    rng = np.random.default_rng(5)
    for _ in range(20):
        P = int(rng.choice([2, 4, 8]))
        E = P * int(rng.integers(1, 9))
        k = int(rng.integers(1, min(E, 8) + 1))
        S = int(rng.integers(1, 300))
        H = 64 * int(rng.integers(1, 5))
        skew = float(rng.choice([0.3, 1.0, 2.5]))
        tb = int(rng.choice([0, H * 2 * 16, H * 2 * 7]))
        wl = pb.build_dispatch(pb.ModelConfig("r", H, 64, E, k), pb.ClusterConfig(P, 1, 1), S, skew, tb, 17)
        rem, loc, dig = oracle.build_dispatch(H, E, k, P, 1, S, skew, tb, 17)
        assert wl.digest() == dig
        assert np.array_equal(wl.remote_array(), rem)


def test_fit_alpha_beta_matches_reference():
    """perseus_fit_alpha_beta == sigsim::fit_alpha_beta of the reference library
    (metrics.cpp:69-95) on random message-size / time points, incl. the error case."""
    import pytest as _pt
    from oracle.oracle import RefLib
    if not RefLib.available():
        _pt.skip("reference library not built")
    ref = RefLib()
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(2, 12))
        pts = [(float(rng.integers(1, 1 << 24)), float(rng.random() * 1e6)) for _ in range(n)]
        if len({p[0] for p in pts}) == 1:
            continue
        got = pb.fit_alpha_beta(pts)
        want = ref.fit_alpha_beta(pts)
        assert np.allclose(got, want, rtol=1e-12, atol=1e-9), (got, want)
    with _pt.raises(pb.ConfigError):
        pb.fit_alpha_beta([(5.0, 1.0), (5.0, 2.0)])


def test_cpp_dropin_headers_compile_link_and_pass_reference_kats(tmp_path):
    """A C++ program written against include/sigsim/*.hpp (the reference's header
    names) compiles, links against libperseus.so and reproduces the reference's
    known answers — the drop-in path a reference user takes."""
    import shutil
    import subprocess
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "dropin_kats")
    libdir = os.path.join(root, "paper_2605_00686_b200")
    subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(root, "include"),
                    os.path.join(root, "tests", "cpp", "dropin_kats.cpp"), "-L", libdir, "-lperseus",
                    f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin_kats: pass" in r.stdout
