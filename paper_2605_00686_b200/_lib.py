"""ctypes binding of libperseus.so (include/perseus.h).

The product path: every call goes through the C ABI into the CUDA library.
There is no fallback — if the library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libperseus.so")

OK, ERR_CONFIG, ERR_VERIFY, ERR_RUNTIME = 0, 1, 2, 3
ROUTE_BALANCED, ROUTE_ZIPF, ROUTE_GATE = 0, 1, 2
SIGNAL_COUPLED, SIGNAL_DECOUPLED, SIGNAL_NONE, SIGNAL_FAULT_EARLY = 0, 1, 2, 3
GROUP_AUTO = -1
PHASE_ROUTE, PHASE_DISPATCH, PHASE_EXPERT, PHASE_COMBINE, PHASE_ALL = 0, 1, 2, 3, 15
F_SYNTH_WEIGHTS = 1
F_UNFUSED = 2
F_NO_PAIR = 4
F_FORCE_PAIR = 8
F_NO_PDL = 16
F_LOCAL_DISPATCH = 32
F_LOCAL_COMBINE = 64
F_DF_COMBINE = 128
F_DEDUP = 256
TILE_ROWS = 128


class ConfigError(ValueError):
    """sigsim::ConfigError (sim.hpp:20-22) — status 1."""


class VerifyError(RuntimeError):
    """verification / ordering failure — status 2."""


class ModelError(RuntimeError):
    """sigsim::ModelError / CUDA / timeout — status 3."""


class Transfer(C.Structure):
    _fields_ = [("src_pe", C.c_uint32), ("dst_pe", C.c_uint32), ("expert", C.c_int64),
                ("bytes", C.c_uint64), ("tile_id", C.c_int64), ("heap_offset", C.c_uint64)]


class TraceEvent(C.Structure):
    _fields_ = [("t", C.c_uint64), ("kind", C.c_int32), ("pe", C.c_int32), ("peer", C.c_int32),
                ("tile", C.c_int32), ("group", C.c_int32), ("bytes", C.c_uint32), ("aux", C.c_uint32),
                ("pad", C.c_uint32)]


EV_DISPATCH_PUT, EV_DISPATCH_FENCE, EV_DISPATCH_SIGNAL, EV_DISPATCH_SEEN = 1, 2, 3, 4
EV_COMBINE_PUT, EV_COMBINE_FENCE, EV_COMBINE_SIGNAL, EV_COMBINE_SEEN = 5, 6, 7, 8


class TraceReport(C.Structure):
    _fields_ = [("records", C.c_int64), ("fence_count", C.c_int64 * 2), ("flagged_signal_count", C.c_int64 * 2),
                ("ordering_violations", C.c_int64 * 2), ("late_tiles", C.c_int64 * 2),
                ("conservation_ok", C.c_int32 * 2), ("put_bytes", C.c_int64 * 2),
                ("conservation_error", C.c_char * 256)]

    def as_dict(self):
        d = {"records": self.records}
        for i, direction in enumerate(("dispatch", "combine")):
            d[direction] = {"fence_count": self.fence_count[i], "flagged_signal_count": self.flagged_signal_count[i],
                            "ordering_violations": self.ordering_violations[i], "late_tiles": self.late_tiles[i],
                            "conservation_ok": bool(self.conservation_ok[i]), "put_bytes": self.put_bytes[i]}
        d["conservation_error"] = self.conservation_error.decode()
        return d


class TraceRecord(C.Structure):
    """include/perseus.h:perseus_trace_record (a flat sigsim::TraceRecord)."""
    _fields_ = [("time", C.c_int64), ("pe", C.c_uint32), ("kind", C.c_int32), ("req_kind", C.c_int32),
                ("src_pe", C.c_uint32), ("dst_pe", C.c_uint32), ("fence_flag", C.c_int32), ("size", C.c_uint64),
                ("qp", C.c_int32), ("pad", C.c_int32), ("group_id", C.c_int64), ("tile_id", C.c_int64),
                ("submit_seq", C.c_uint64)]


class LayerConfig(C.Structure):
    _fields_ = [("hidden_dim", C.c_int64), ("intermediate_dim", C.c_int64),
                ("experts", C.c_int64), ("top_k", C.c_int64), ("tokens_per_pe", C.c_uint64),
                ("routing", C.c_int32), ("skew", C.c_double), ("seed", C.c_uint64),
                ("signaling", C.c_int32), ("group_size", C.c_int64), ("flags", C.c_int32)]


class Counters(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "epoch", "dispatch_fences", "dispatch_signals", "dispatch_puts", "dispatch_put_bytes",
        "combine_fences", "combine_signals", "combine_puts", "combine_put_bytes", "recv_tiles",
        "wait_timeouts", "errors", "wait_dispatch_ns", "wait_g1_ns", "copy_ns", "cta_ns",
        "wait_remote_ns", "dispatch_span_ns", "combine_span_ns", "combine_wait_ns",
        "mma_cycles", "mma_ring_wait", "mma_acc_wait", "mma_data_wait")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, sz, i64, u64, i32 = C.c_void_p, C.c_size_t, C.c_int64, C.c_uint64, C.c_int32
    P = C.POINTER
    sig = {
        "perseus_last_error": (C.c_char_p, []),
        "perseus_abi_version": (C.c_int, []),
        "perseus_remote_transfer_count": (C.c_int, [i64, i64, i64, P(i64)]),
        "perseus_message_size": (u64, [u64, i64, i64, i64]),
        "perseus_zipf_route": (C.c_int, [u64, i64, C.c_double, i64, u64, P(u64), P(i32)]),
        "perseus_build_dispatch": (C.c_int, [i64, i64, i64, i64, C.c_int, C.c_int, C.c_int, u64,
                                             C.c_double, u64, u64, P(Transfer), sz, P(sz),
                                             P(Transfer), sz, P(sz), P(u64)]),
        "perseus_assign_groups": (C.c_int, [P(Transfer), sz, i64, P(i64), P(i64), P(sz)]),
        "perseus_heap_digest": (u64, [P(u64), sz, P(u64), sz]),
        "perseus_fnv1a64": (u64, [vp, sz, u64]),
        "perseus_layer_create": (C.c_int, [P(LayerConfig), C.c_int, C.c_int, C.c_int, P(vp)]),
        "perseus_layer_destroy": (C.c_int, [vp]),
        "perseus_layer_ipc_export": (C.c_int, [vp, vp, sz, P(sz)]),
        "perseus_layer_ipc_import": (C.c_int, [vp, vp, sz]),
        "perseus_layer_connect_local": (C.c_int, [P(vp), C.c_int]),
        "perseus_layer_set_weights": (C.c_int, [vp, vp, vp, vp, vp]),
        "perseus_layer_init_synthetic": (C.c_int, [vp, u64, vp]),
        "perseus_fill_synthetic_x": (C.c_int, [vp, vp, u64, vp]),
        "perseus_layer_forward": (C.c_int, [vp, vp, vp, vp]),
        "perseus_layer_forward_host": (C.c_int, [vp, vp, vp, vp]),
        "perseus_layer_forward_host_async": (C.c_int, [vp, vp, vp]),
        "perseus_layer_host_wait": (C.c_int, [vp]),
        "perseus_layer_forward_phase": (C.c_int, [vp, C.c_int, vp, vp, vp]),
        "perseus_layer_counters": (C.c_int, [vp, P(Counters)]),
        "perseus_layer_read_routing": (C.c_int, [vp, P(i32), P(C.c_float), P(i32), P(i32)]),
        "perseus_layer_read_layout": (C.c_int, [vp, P(Transfer), sz, P(sz), P(i64), sz, P(sz)]),
        "perseus_layer_read_count_table": (C.c_int, [vp, P(i32)]),
        "perseus_layer_read_timing": (C.c_int, [vp, P(C.c_float), C.c_int]),
        "perseus_layer_set_stage_timing": (C.c_int, [vp, C.c_int]),
        "perseus_layer_set_timeline": (C.c_int, [vp, C.c_int]),
        "perseus_layer_set_trace": (C.c_int, [vp, C.c_int]),
        "perseus_layer_info": (C.c_int, [vp, P(C.c_int), P(C.c_int)]),
        "perseus_layer_group_size": (C.c_int, [vp, P(i64)]),
        "perseus_resolve_group_size": (C.c_int, [P(LayerConfig), C.c_int, P(i64)]),
        "perseus_layer_read_trace": (C.c_int, [vp, P(TraceEvent), sz, P(sz)]),
        "perseus_fit_alpha_beta": (C.c_int, [P(C.c_double), P(C.c_double), sz, P(C.c_double), P(C.c_double),
                                            P(C.c_double)]),
        "perseus_trace_serialize": (C.c_int, [P(TraceEvent), sz, C.c_int, C.c_int, C.c_char_p, sz, P(sz)]),
        "perseus_trace_records": (C.c_int, [P(TraceEvent), sz, C.c_int, C.c_int, P(TraceRecord), sz, P(sz), P(u64),
                                            P(u64)]),
        "perseus_trace_analyze": (C.c_int, [P(TraceEvent), sz, C.c_int, P(Transfer), sz, P(TraceReport)]),
        "perseus_layer_read_timeline": (C.c_int, [vp, P(C.c_uint64), C.c_int]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()

# every symbol include/perseus.h declares (checked by the CPU tests)
EXPORTED = [n for n in dir(lib) if n.startswith("perseus_")]


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib.perseus_last_error().decode(errors="replace")
    if rc == ERR_CONFIG:
        raise ConfigError(msg)
    if rc == ERR_VERIFY:
        raise VerifyError(msg)
    raise ModelError(msg)
