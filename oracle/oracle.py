"""oracle/oracle.py — CPU ORACLE, TEST INFRASTRUCTURE ONLY.

Python face of the checkers:
  * ``Oracle``  — ctypes over oracle/liboracle.so (the plain-C restatement in
    oracle.c, each function citing the reference file:line it restates) plus the
    fp32 numpy SwiGLU-FFN / combine that has no reference counterpart
    ("parity unpinned", SURVEY.md §0.2 — tolerance lives in the tests).
  * ``RefLib``  — ctypes over oracle/_ref/libsigsim_ref.so, the UNMODIFIED
    reference library compiled from /root/reference sources (oracle/Makefile).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's reference /
cpu_baseline legs may import this module.  The product never does.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsigsim_ref.so")

# tensor ids of the synthetic-input hash (oracle.c: orc_fill_bf16)
T_X, T_WG, T_W1, T_W2 = 1, 2, 3, 4


class Transfer(C.Structure):
    """Flat TransferSpec (workload.hpp:42-49); same layout in oracle.c, the
    reference shim and include/perseus.h:perseus_transfer."""
    _fields_ = [("src_pe", C.c_uint32), ("dst_pe", C.c_uint32), ("expert", C.c_int64),
                ("bytes", C.c_uint64), ("tile_id", C.c_int64), ("heap_offset", C.c_uint64)]


def transfers_to_np(arr, n):
    return np.array([(arr[i].src_pe, arr[i].dst_pe, arr[i].expert, arr[i].bytes, arr[i].tile_id,
                      arr[i].heap_offset) for i in range(n)], dtype=np.int64).reshape(-1, 6)


def build(force: bool = False) -> None:
    """Compile the checkers (oracle.c, and oracle/_ref when /root/reference exists)."""
    if force or not os.path.exists(ORACLE_SO) or (
            os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "oracle.c"))):
        subprocess.run(["make", "-s", "-C", HERE, os.path.join(HERE, "liboracle.so")], check=True)
    if os.path.isdir("/root/reference/proj/src") and (force or not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class LayerShape:
    hidden: int
    inter: int
    experts: int
    top_k: int
    tokens: int          # S, tokens per PE
    pes: int = 1         # P (EP degree)

    def scales(self):
        """uniform(-a, a) with a = sqrt(3 / fan_in): unit variance x, N(0,1/fan_in)-like weights."""
        return (float(np.float32(math.sqrt(3.0))), float(np.float32(math.sqrt(3.0 / self.hidden))),
                float(np.float32(math.sqrt(3.0 / self.hidden))), float(np.float32(math.sqrt(3.0 / self.inter))))


class Oracle:
    def __init__(self):
        build()
        L = C.CDLL(ORACLE_SO)
        self.L = L
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_rng_stream.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        L.orc_fnv1a64.restype = C.c_uint64
        L.orc_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.orc_remote_transfer_count.restype = C.c_int64
        L.orc_remote_transfer_count.argtypes = [C.c_int64] * 3
        L.orc_message_size.restype = C.c_uint64
        L.orc_message_size.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64]
        L.orc_zipf_route.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_int64, C.c_uint64,
                                     C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]
        L.orc_balanced_ids.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_int32)]
        L.orc_route_counts.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_uint64,
                                       C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]
        L.orc_layout_from_counts.argtypes = [C.POINTER(C.c_uint64), C.c_int64, C.c_int64, C.c_int,
                                             C.c_int, C.c_uint64, C.POINTER(Transfer), C.c_size_t,
                                             C.POINTER(C.c_size_t), C.POINTER(Transfer), C.c_size_t,
                                             C.POINTER(C.c_size_t)]
        L.orc_workload_digest.restype = C.c_uint64
        L.orc_workload_digest.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_uint64,
                                          C.POINTER(Transfer), C.c_size_t, C.POINTER(Transfer),
                                          C.c_size_t]
        L.orc_heap_digest.restype = C.c_uint64
        L.orc_heap_digest.argtypes = [C.POINTER(C.c_uint64), C.c_size_t, C.POINTER(C.c_uint64),
                                      C.c_size_t]
        L.orc_assign_groups.argtypes = [C.POINTER(Transfer), C.c_size_t, C.c_int64,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_size_t)]
        L.orc_fences_for_src.restype = C.c_int64
        L.orc_fences_for_src.argtypes = [C.POINTER(Transfer), C.c_size_t, C.c_uint32, C.c_int,
                                         C.c_int64, C.c_int]
        L.orc_tensor_base.restype = C.c_uint64
        L.orc_tensor_base.argtypes = [C.c_uint64, C.c_uint32]
        L.orc_fill_bf16.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_float,
                                    C.POINTER(C.c_uint16)]
        L.orc_bf16_to_f32.argtypes = [C.POINTER(C.c_uint16), C.c_uint64, C.POINTER(C.c_float)]
        L.orc_f32_to_bf16.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.POINTER(C.c_uint16)]
        L.orc_gate_logits.argtypes = [C.POINTER(C.c_uint16), C.POINTER(C.c_uint16), C.c_uint64,
                                      C.c_int64, C.c_int64, C.POINTER(C.c_float)]
        L.orc_topk.argtypes = [C.POINTER(C.c_float), C.c_uint64, C.c_int64, C.c_int64,
                               C.POINTER(C.c_int32)]
        L.orc_route_weights.argtypes = [C.POINTER(C.c_float), C.POINTER(C.c_int32), C.c_uint64,
                                        C.c_int64, C.c_int64, C.POINTER(C.c_float)]
        L.orc_permute.argtypes = [C.POINTER(C.c_int32), C.c_uint64, C.c_int64, C.c_int64,
                                  C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32)]

    # ---------------- integer / planner restatements ----------------
    def rng_stream(self, seed, n):
        out = np.zeros(n, dtype=np.uint64)
        self.L.orc_rng_stream(seed, n, _p(out, C.c_uint64))
        return out

    def remote_transfer_count(self, E, P, P_local):
        v = self.L.orc_remote_transfer_count(E, P, P_local)
        if v < 0:
            raise ValueError("ConfigError")
        return v

    def message_size(self, S, k, E, H):
        return self.L.orc_message_size(S, k, E, H)

    def zipf_route(self, S, E, s, k, seed, want_ids=False):
        counts = np.zeros(E, dtype=np.uint64)
        ids = np.zeros(S * k, dtype=np.int32) if want_ids else None
        rc = self.L.orc_zipf_route(S, E, s, k, seed, _p(counts, C.c_uint64),
                                   _p(ids, C.c_int32) if want_ids else None)
        if rc:
            raise ValueError("ConfigError")
        return (counts, ids) if want_ids else counts

    def route_counts(self, S, E, k, skew, seed, P, want_ids=False):
        counts = np.zeros((P, E), dtype=np.uint64)
        ids = np.zeros((P, S * k), dtype=np.int32) if want_ids else None
        rc = self.L.orc_route_counts(S, E, k, skew, seed, P, _p(counts, C.c_uint64),
                                     _p(ids, C.c_int32) if want_ids else None)
        if rc:
            raise ValueError("ConfigError")
        return (counts, ids) if want_ids else counts

    def layout_from_counts(self, counts, H, E, nodes, gpn, tile_bytes):
        counts = np.ascontiguousarray(counts, dtype=np.uint64)
        nr, nl = C.c_size_t(0), C.c_size_t(0)
        rc = self.L.orc_layout_from_counts(_p(counts, C.c_uint64), H, E, nodes, gpn, tile_bytes,
                                           None, 0, C.byref(nr), None, 0, C.byref(nl))
        if rc:
            raise ValueError("ConfigError")
        R = (Transfer * max(nr.value, 1))()
        Lo = (Transfer * max(nl.value, 1))()
        self.L.orc_layout_from_counts(_p(counts, C.c_uint64), H, E, nodes, gpn, tile_bytes, R,
                                      nr.value, C.byref(nr), Lo, nl.value, C.byref(nl))
        return R, nr.value, Lo, nl.value

    def build_dispatch(self, H, E, k, nodes, gpn, S, skew, tile_bytes, seed):
        """Restatement of sigsim::build_dispatch (workload.cpp:155-213)."""
        counts = self.route_counts(S, E, k, skew, seed, nodes * gpn)
        R, nr, Lo, nl = self.layout_from_counts(counts, H, E, nodes, gpn, tile_bytes)
        dig = self.L.orc_workload_digest(nodes, gpn, S, skew, tile_bytes, R, nr, Lo, nl)
        return transfers_to_np(R, nr), transfers_to_np(Lo, nl), dig

    def heap_digest(self, extents, flags):
        ext = np.ascontiguousarray(np.asarray(extents, dtype=np.uint64).reshape(-1, 3))
        fl = np.ascontiguousarray(np.asarray(flags, dtype=np.uint64).reshape(-1))
        return self.L.orc_heap_digest(_p(ext, C.c_uint64), ext.shape[0], _p(fl, C.c_uint64),
                                      fl.shape[0])

    @staticmethod
    def _np_to_transfers(t):
        arr = (Transfer * max(len(t), 1))()
        for i, row in enumerate(t):
            arr[i] = Transfer(int(row[0]), int(row[1]), int(row[2]), int(row[3]), int(row[4]),
                              int(row[5]))
        return arr

    def assign_groups(self, t, group_size):
        arr = self._np_to_transfers(t)
        gof = np.zeros(max(len(t), 1), dtype=np.int64)
        lead = np.zeros(max(len(t), 1), dtype=np.int64)
        ng = C.c_size_t(0)
        if self.L.orc_assign_groups(arr, len(t), group_size, _p(gof, C.c_int64),
                                    _p(lead, C.c_int64), C.byref(ng)):
            raise ValueError("ConfigError")
        return gof[:len(t)], lead[:ng.value]

    def fences_for_src(self, remote, src, signaling, group_size, gpu_direct=False):
        arr = self._np_to_transfers(remote)
        v = self.L.orc_fences_for_src(arr, len(remote), src, signaling, group_size, int(gpu_direct))
        if v < 0:
            raise ValueError("ConfigError")
        return v

    # ---------------- synthetic tensors (bit-identical to the device) ----------------
    def fill_bf16(self, seed, tensor, first, n, scale):
        out = np.empty(n, dtype=np.uint16)
        self.L.orc_fill_bf16(seed, tensor, first, n, scale, _p(out, C.c_uint16))
        return out

    @staticmethod
    def bf16_to_f32(a):
        return (a.astype(np.uint32) << 16).view(np.float32)

    def f32_to_bf16(self, a):
        a = np.ascontiguousarray(a, dtype=np.float32)
        out = np.empty(a.shape, dtype=np.uint16)
        self.L.orc_f32_to_bf16(_p(a, C.c_float), a.size, _p(out, C.c_uint16))
        return out

    def gen_x(self, shape: LayerShape, seed, rank, tokens=None):
        t0 = rank * shape.tokens
        n = shape.tokens if tokens is None else tokens
        return self.fill_bf16(seed, T_X, t0 * shape.hidden, n * shape.hidden,
                              shape.scales()[0]).reshape(n, shape.hidden)

    def gen_wg(self, shape: LayerShape, seed):
        return self.fill_bf16(seed, T_WG, 0, shape.experts * shape.hidden,
                              shape.scales()[1]).reshape(shape.experts, shape.hidden)

    def gen_w1(self, shape: LayerShape, seed, e):
        n = 2 * shape.inter * shape.hidden
        return self.fill_bf16(seed, T_W1, e * n, n, shape.scales()[2]).reshape(2 * shape.inter,
                                                                                shape.hidden)

    def gen_w2(self, shape: LayerShape, seed, e):
        n = shape.hidden * shape.inter
        return self.fill_bf16(seed, T_W2, e * n, n, shape.scales()[3]).reshape(shape.hidden,
                                                                                shape.inter)

    # ---------------- gate / routing / permutation ----------------
    def gate_logits(self, x_bf16, wg_bf16):
        T, H = x_bf16.shape
        E = wg_bf16.shape[0]
        x = np.ascontiguousarray(x_bf16)
        w = np.ascontiguousarray(wg_bf16)
        out = np.empty((T, E), dtype=np.float32)
        self.L.orc_gate_logits(_p(x, C.c_uint16), _p(w, C.c_uint16), T, H, E, _p(out, C.c_float))
        return out

    def topk(self, logits, k):
        T, E = logits.shape
        l = np.ascontiguousarray(logits, dtype=np.float32)
        ids = np.zeros((T, k), dtype=np.int32)
        self.L.orc_topk(_p(l, C.c_float), T, E, k, _p(ids, C.c_int32))
        return ids

    def route_weights(self, logits, ids):
        T, E = logits.shape
        k = ids.shape[1]
        l = np.ascontiguousarray(logits, dtype=np.float32)
        i = np.ascontiguousarray(ids, dtype=np.int32)
        w = np.zeros((T, k), dtype=np.float32)
        self.L.orc_route_weights(_p(l, C.c_float), _p(i, C.c_int32), T, E, k, _p(w, C.c_float))
        return w

    def permute(self, ids, E):
        S, k = ids.shape
        i = np.ascontiguousarray(ids, dtype=np.int32)
        off = np.zeros(E + 1, dtype=np.uint64)
        rows = np.zeros(S * k, dtype=np.int32)
        pos = np.zeros(S * k, dtype=np.int32)
        self.L.orc_permute(_p(i, C.c_int32), S, k, E, _p(off, C.c_uint64), _p(rows, C.c_int32),
                           _p(pos, C.c_int32))
        return off, rows, pos.reshape(S, k)

    def route(self, shape: LayerShape, mode: str, seed: int, rank: int, x_bf16, wg_bf16,
              skew: float = 0.0):
        """ids [S,k] and fp32 combine weights [S,k] for one rank.
        mode: 'balanced' | 'zipf' (reference routing, ids from the reference RNG
        stream) | 'gate' (learned top-k on fp32 logits)."""
        logits = self.gate_logits(x_bf16, wg_bf16)
        S, E, k = x_bf16.shape[0], shape.experts, shape.top_k
        if mode == "gate":
            ids = self.topk(logits, k)
        elif mode == "balanced":
            ids = np.zeros(S * k, dtype=np.int32)
            if self.L.orc_balanced_ids(S, E, k, _p(ids, C.c_int32)):
                raise ValueError("ConfigError: balanced routing needs E | S*k")
            ids = ids.reshape(S, k)
        elif mode == "zipf":
            s_seed = (seed ^ ((0x9E3779B97F4A7C15 * (rank + 1)) & 0xFFFFFFFFFFFFFFFF))
            _, ids = self.zipf_route(S, E, skew, k, s_seed, want_ids=True)
            ids = ids.reshape(S, k)
        else:
            raise ValueError(mode)
        return ids, self.route_weights(logits, ids), logits

    # ---------------- fp32 layer (parity unpinned by the reference) ----------------
    def expert_ffn(self, shape: LayerShape, seed, e, xrows_f32):
        """y = (silu(x W_gate^T) * (x W_up^T)) W_down^T in fp32."""
        w1 = self.bf16_to_f32(self.gen_w1(shape, seed, e))
        w2 = self.bf16_to_f32(self.gen_w2(shape, seed, e))
        I = shape.inter
        g = xrows_f32 @ w1[:I].T
        u = xrows_f32 @ w1[I:].T
        h = (g / (1.0 + np.exp(-g))) * u
        return h @ w2.T

    def layer_forward(self, shape: LayerShape, mode: str, seed: int, rank: int, skew=0.0,
                      token_subset=None):
        """fp32 output [S or |subset|, H] of one rank's tokens, plus routing."""
        x = self.gen_x(shape, seed, rank)
        wg = self.gen_wg(shape, seed)
        ids, w, logits = self.route(shape, mode, seed, rank, x, wg, skew)
        toks = np.arange(shape.tokens) if token_subset is None else np.asarray(token_subset)
        xf = self.bf16_to_f32(x)
        out = np.zeros((len(toks), shape.hidden), dtype=np.float32)
        sub_ids = ids[toks]
        for e in np.unique(sub_ids):
            sel_t, sel_j = np.nonzero(sub_ids == e)
            y = self.expert_ffn(shape, seed, int(e), xf[toks[sel_t]])
            out[sel_t] += w[toks[sel_t], sel_j][:, None] * y
        return out, ids, w


class RefLib:
    """The UNMODIFIED reference (oracle/_ref/libsigsim_ref.so)."""

    class RunResult(C.Structure):
        _fields_ = [("workload_digest", C.c_uint64), ("heap_digest", C.c_uint64),
                    ("fence_count", C.c_int64), ("flagged_signal_count", C.c_int64),
                    ("proxy_stop_episodes", C.c_int64), ("nic_stall_episodes", C.c_int64),
                    ("proxy_blocked_total_ns", C.c_int64), ("makespan_ns", C.c_int64),
                    ("n_records", C.c_int64), ("n_violations", C.c_int64),
                    ("conservation_pass", C.c_int64), ("total_put_bytes", C.c_uint64),
                    ("n_signals_visible", C.c_int64)]

    MODES = {"vanilla": 0, "decoupled": 1, "nic_ordering": 2, "combined": 3, "gpu_direct": 4,
             "gpu_direct_decoupled": 5}

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        build()
        L = C.CDLL(REF_SO)
        self.L = L
        L.ref_last_error.restype = C.c_char_p
        L.ref_fit_alpha_beta.argtypes = [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_size_t,
                                         C.POINTER(C.c_double)]
        L.ref_remote_transfer_count.argtypes = [C.c_int64] * 3 + [C.POINTER(C.c_int64)]
        L.ref_message_size.restype = C.c_uint64
        L.ref_message_size.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64]
        L.ref_zipf_route.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_int64, C.c_uint64,
                                     C.POINTER(C.c_uint64)]
        L.ref_build_dispatch.argtypes = [C.c_int64] * 4 + [C.c_int] * 3 + [
            C.c_uint64, C.c_double, C.c_uint64, C.c_uint64, C.POINTER(Transfer), C.c_size_t,
            C.POINTER(C.c_size_t), C.POINTER(Transfer), C.c_size_t, C.POINTER(C.c_size_t),
            C.POINTER(C.c_uint64)]
        L.ref_assign_groups.argtypes = [C.POINTER(Transfer), C.c_size_t, C.c_int64,
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_size_t)]
        L.ref_run_dispatch.argtypes = [C.c_int, C.c_int64] + [C.c_int64] * 4 + [C.c_int] * 3 + [
            C.c_uint64, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_int64),
            C.POINTER(RefLib.RunResult)]
        L.ref_fnv1a64.restype = C.c_uint64
        L.ref_fnv1a64.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
        L.ref_analyze_records.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint64, C.POINTER(Transfer),
                                          C.c_size_t, C.c_int, C.POINTER(RefLib.CheckReport), C.c_char_p,
                                          C.c_size_t]

    class CheckReport(C.Structure):
        _fields_ = [(n, C.c_int64) for n in (
            "fence_count", "flagged_signal_count", "proxy_stop_episodes", "nic_stall_episodes",
            "proxy_blocked_total_ns", "nic_stall_total_ns", "n_violations", "conservation_pass", "n_failures")]

    def analyze_records(self, records, n, submitted, delivered, transfers, swap=False):
        """The reference's fence_accounting / verify_ordering / conservation_check
        (metrics.cpp:10-59,118-190), unmodified, on a RunTrace built from flat
        records (perseus_trace_record layout); transfers: [m, 6] int64 rows in
        TransferSpec field order (swap: combine-direction mirror)."""
        rep = RefLib.CheckReport()
        arr = Oracle._np_to_transfers(np.asarray(transfers, dtype=np.int64).reshape(-1, 6))
        msg = C.create_string_buffer(65536)
        self._chk(self.L.ref_analyze_records(C.addressof(records), n, submitted, delivered, arr,
                                             len(transfers), int(swap), C.byref(rep), msg, len(msg)))
        d = {f: getattr(rep, f) for f, _ in RefLib.CheckReport._fields_}
        d["failures"] = [x for x in msg.value.decode().split("\n") if x]
        return d


    def fit_alpha_beta(self, points):
        xs = (C.c_double * len(points))(*[p[0] for p in points])
        ys = (C.c_double * len(points))(*[p[1] for p in points])
        out = (C.c_double * 3)()
        if self.L.ref_fit_alpha_beta(xs, ys, len(points), out) != 0:
            raise ValueError(self.L.ref_last_error().decode())
        return tuple(out)
    def _chk(self, rc):
        if rc == 1:
            raise ValueError("ConfigError: " + self.L.ref_last_error().decode())
        if rc:
            raise RuntimeError(self.L.ref_last_error().decode())

    def remote_transfer_count(self, E, P, P_local):
        out = C.c_int64(0)
        self._chk(self.L.ref_remote_transfer_count(E, P, P_local, C.byref(out)))
        return out.value

    def message_size(self, S, k, E, H):
        return self.L.ref_message_size(S, k, E, H)

    def zipf_route(self, S, E, s, k, seed):
        counts = np.zeros(E, dtype=np.uint64)
        self._chk(self.L.ref_zipf_route(S, E, s, k, seed, _p(counts, C.c_uint64)))
        return counts

    def build_dispatch(self, H, I, E, k, nodes, gpn, nqps, S, skew, tile_bytes, seed):
        nr, nl, dig = C.c_size_t(0), C.c_size_t(0), C.c_uint64(0)
        self._chk(self.L.ref_build_dispatch(H, I, E, k, nodes, gpn, nqps, S, skew, tile_bytes,
                                            seed, None, 0, C.byref(nr), None, 0, C.byref(nl),
                                            C.byref(dig)))
        R = (Transfer * max(nr.value, 1))()
        Lo = (Transfer * max(nl.value, 1))()
        self._chk(self.L.ref_build_dispatch(H, I, E, k, nodes, gpn, nqps, S, skew, tile_bytes,
                                            seed, R, nr.value, C.byref(nr), Lo, nl.value,
                                            C.byref(nl), C.byref(dig)))
        return transfers_to_np(R, nr.value), transfers_to_np(Lo, nl.value), dig.value

    def assign_groups(self, t, group_size):
        arr = Oracle._np_to_transfers(t)
        gof = np.zeros(max(len(t), 1), dtype=np.int64)
        lead = np.zeros(max(len(t), 1), dtype=np.int64)
        ng = C.c_size_t(0)
        self._chk(self.L.ref_assign_groups(arr, len(t), group_size, _p(gof, C.c_int64),
                                           _p(lead, C.c_int64), C.byref(ng)))
        return gof[:len(t)], lead[:ng.value]

    def run_dispatch(self, mode, group_size, H, I, E, k, nodes, gpn, nqps, S, skew, tile_bytes,
                     wl_seed, run_seed=1):
        res = RefLib.RunResult()
        per_pe = np.zeros(nodes * gpn, dtype=np.int64)
        self._chk(self.L.ref_run_dispatch(self.MODES[mode], group_size, H, I, E, k, nodes, gpn,
                                          nqps, S, skew, tile_bytes, wl_seed, run_seed,
                                          _p(per_pe, C.c_int64), C.byref(res)))
        d = {f: getattr(res, f) for f, _ in RefLib.RunResult._fields_}
        d["fences_per_pe"] = per_pe.tolist()
        return d
