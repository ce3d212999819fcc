"""MoELayer — the user-facing handle of one expert-parallel rank of the B200
Perseus MoE layer (the C ABI perseus_layer_* of include/perseus.h).

It replaces the reference's hot path, ``run_dispatch`` (protocols.cpp:346-362,
a simulator of the dispatch puts/signals with a timing stand-in for the expert
FFN), with the real layer forward on the GPU: gate/route -> permutation ->
dispatch puts + signals over NVLink -> SwiGLU expert FFN on tcgen05 -> combine
puts + signals -> weighted reduce.  torch is used only for device memory,
streams and the multi-process bootstrap.
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib
from .sigsim import ModelConfig, ProtocolConfig, combined_protocol

ROUTING = {"balanced": _lib.ROUTE_BALANCED, "zipf": _lib.ROUTE_ZIPF, "gate": _lib.ROUTE_GATE}


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return stream if isinstance(stream, int) else stream.cuda_stream


def layer_config(model: ModelConfig, tokens_per_pe: int, routing: str = "balanced", skew: float = 0.0,
                 seed: int = 1, protocol: Optional[ProtocolConfig] = None, flags: int = 0) -> "_lib.LayerConfig":
    """perseus_layer_config of a layer (include/perseus.h)."""
    protocol = protocol or combined_protocol(0)
    return _lib.LayerConfig(model.hidden_dim, model.intermediate_dim, model.experts, model.top_k,
                            tokens_per_pe, ROUTING[routing], float(skew), seed,
                            protocol.device_signaling(), protocol.group_size, flags)


def resolve_group_size(model: ModelConfig, tokens_per_pe: int, world: int, routing: str = "balanced",
                       skew: float = 0.0, seed: int = 1, protocol: Optional[ProtocolConfig] = None) -> int:
    """Host only: the DECOUPLED group size a layer would resolve at create
    (perseus_resolve_group_size; ConfigError like run_dispatch's precheck)."""
    cfg = layer_config(model, tokens_per_pe, routing, skew, seed, protocol)
    g = C.c_int64()
    check(lib.perseus_resolve_group_size(C.byref(cfg), world, C.byref(g)))
    return g.value


class MoELayer:
    def __init__(self, model: ModelConfig, tokens_per_pe: int, rank: int = 0, world: int = 1,
                 device: int = 0, routing: str = "balanced", skew: float = 0.0, seed: int = 1,
                 protocol: Optional[ProtocolConfig] = None, synthetic_weights: bool = True,
                 fused: bool = True, pair: Optional[bool] = None, pdl: Optional[bool] = None, flags: int = 0):
        protocol = protocol or combined_protocol(0)
        if pdl is None:
            # PDL unless several EP ranks (processes) share one device: a grid
            # waiting for its PDL primary holds up the device's work distributor,
            # and with it the other ranks' grids that primary waits for
            import os
            shared = os.environ.get("PERSEUS_SHARED_DEVICE")
            if shared is None:
                import torch
                n_dev = torch.cuda.device_count()
                pdl = not (world > 1 and n_dev > 0 and world > n_dev)
            else:
                pdl = not int(shared)
        self.fused = fused
        self.model, self.S, self.rank, self.world, self.device = model, tokens_per_pe, rank, world, device
        self.routing_mode, self.skew, self.seed, self.protocol = routing, skew, seed, protocol
        cfg = _lib.LayerConfig(model.hidden_dim, model.intermediate_dim, model.experts, model.top_k,
                               tokens_per_pe, ROUTING[routing], float(skew), seed,
                               protocol.device_signaling(), protocol.group_size,
                               (_lib.F_SYNTH_WEIGHTS if synthetic_weights else 0)
                               | (0 if fused else _lib.F_UNFUSED)
                               | {None: 0, True: _lib.F_FORCE_PAIR, False: _lib.F_NO_PAIR}[pair]
                               | (0 if pdl else _lib.F_NO_PDL) | flags)
        self._cfg = cfg
        h = C.c_void_p()
        check(lib.perseus_layer_create(C.byref(cfg), rank, world, device, C.byref(h)))
        self._h = h

    # ------------------------------------------------------------ bootstrap --
    def ipc_blob(self) -> bytes:
        n = C.c_size_t(0)
        check(lib.perseus_layer_ipc_export(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib.perseus_layer_ipc_export(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def connect_ipc(self, blobs: Sequence[bytes]) -> None:
        each = len(blobs[0])
        data = b"".join(blobs)
        check(lib.perseus_layer_ipc_import(self._h, data, each))

    def connect_dist(self, group=None) -> None:
        """Exchange symmetric-heap IPC handles over torch.distributed (one
        process per GPU)."""
        import torch.distributed as dist
        blobs: List[bytes] = [b""] * self.world
        dist.all_gather_object(blobs, self.ipc_blob(), group=group)
        self.connect_ipc(blobs)

    @staticmethod
    def connect_local(layers: Sequence["MoELayer"]) -> None:
        """P ranks emulated in one process (one device): raw peer pointers."""
        arr = (C.c_void_p * len(layers))(*[l._h.value for l in layers])
        check(lib.perseus_layer_connect_local(arr, len(layers)))

    # -------------------------------------------------------------- weights --
    def set_weights(self, wg, w1, w2, stream=None) -> None:
        check(lib.perseus_layer_set_weights(self._h, _ptr(wg), _ptr(w1), _ptr(w2), _stream(stream)))

    def init_synthetic(self, seed: int, stream=None) -> None:
        check(lib.perseus_layer_init_synthetic(self._h, seed, _stream(stream)))

    def fill_synthetic_x(self, x, seed: Optional[int] = None, stream=None) -> None:
        check(lib.perseus_fill_synthetic_x(self._h, _ptr(x), self.seed if seed is None else seed,
                                           _stream(stream)))

    # -------------------------------------------------------------- forward --
    def forward(self, x, out, stream=None) -> None:
        check(lib.perseus_layer_forward(self._h, _ptr(x), _ptr(out), _stream(stream)))

    def forward_phase(self, phase: int, x, out, stream=None) -> None:
        check(lib.perseus_layer_forward_phase(self._h, phase, _ptr(x), _ptr(out), _stream(stream)))

    def forward_host(self, x_host: np.ndarray, out_host: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
        """End-to-end entry: HOST bf16 bits [S, H] (uint16) in, HOST bf16 bits out."""
        x_host = np.ascontiguousarray(x_host, dtype=np.uint16)
        if out_host is None:
            out_host = np.empty_like(x_host)
        check(lib.perseus_layer_forward_host(self._h, x_host.ctypes.data, out_host.ctypes.data,
                                             None if stream is None else _stream(stream)))
        return out_host

    def forward_host_async(self, x_host: np.ndarray, out_host: np.ndarray) -> None:
        """Pipelined end-to-end entry (serving a stream of batches): enqueue
        H2D(x_host) -> forward -> D2H(out_host) and return; batch n+1's upload and
        n-1's download overlap batch n's forward.  Both arrays must be uint16
        [S, H], should be pinned, and must stay alive until host_wait()."""
        assert x_host.dtype == np.uint16 and out_host.dtype == np.uint16
        assert x_host.flags.c_contiguous and out_host.flags.c_contiguous
        check(lib.perseus_layer_forward_host_async(self._h, x_host.ctypes.data, out_host.ctypes.data))

    def host_wait(self) -> None:
        check(lib.perseus_layer_host_wait(self._h))

    # ------------------------------------------------------------- evidence --
    def counters(self) -> Dict[str, int]:
        c = _lib.Counters()
        check(lib.perseus_layer_counters(self._h, C.byref(c)))
        return c.as_dict()

    def routing(self):
        Sk = self.S * self.model.top_k
        ids = np.zeros(Sk, dtype=np.int32)
        w = np.zeros(Sk, dtype=np.float32)
        cnt = np.zeros(self.model.experts, dtype=np.int32)
        pos = np.zeros(Sk, dtype=np.int32)
        P = C.POINTER
        check(lib.perseus_layer_read_routing(self._h, ids.ctypes.data_as(P(C.c_int32)),
                                             w.ctypes.data_as(P(C.c_float)),
                                             cnt.ctypes.data_as(P(C.c_int32)),
                                             pos.ctypes.data_as(P(C.c_int32))))
        k = self.model.top_k
        return ids.reshape(-1, k), w.reshape(-1, k), cnt, pos.reshape(-1, k)

    def layout(self):
        """(sent remote transfer tiles as an [n, 6] int64 array in TransferSpec
        field order, flag ids observed set at this rank this forward)."""
        n, nf = C.c_size_t(0), C.c_size_t(0)
        check(lib.perseus_layer_read_layout(self._h, None, 0, C.byref(n), None, 0, C.byref(nf)))
        arr = (_lib.Transfer * max(n.value, 1))()
        flags = (C.c_int64 * max(nf.value, 1))()
        check(lib.perseus_layer_read_layout(self._h, arr, n.value, C.byref(n), flags, nf.value,
                                            C.byref(nf)))
        sent = np.array([(arr[i].src_pe, arr[i].dst_pe, arr[i].expert, arr[i].bytes, arr[i].tile_id,
                          arr[i].heap_offset) for i in range(n.value)], dtype=np.int64).reshape(-1, 6)
        return sent, np.array(flags[:nf.value], dtype=np.int64)

    def count_table(self) -> np.ndarray:
        t = np.zeros((self.world, self.model.experts), dtype=np.int32)
        check(lib.perseus_layer_read_count_table(self._h, t.ctypes.data_as(C.POINTER(C.c_int32))))
        return t

    def set_stage_timing(self, on: bool = True) -> None:
        """Record per-stage CUDA events in the following forwards (off by default)."""
        check(lib.perseus_layer_set_stage_timing(self._h, int(bool(on))))

    TIMELINE_KERNELS = ("router", "route", "permute", "plan", "fused", "combine", "dispatch", "gemm1", "gemm2",
                        "mma_out_of_work", "copy_warps_done", "epilogue_done", "counts_published", "plan_counts_ready",
                        "fused_cta_entry", "plan_phase_b", "plan_phase_c", "perm_block_start", "perm_block_end",
                        "perm_hist_read", "perm_scan", "perm_bits")

    def info(self) -> dict:
        """The forward path chosen at create: fused kernel, CTA-pair tiles."""
        fused, pairs = C.c_int(), C.c_int()
        check(lib.perseus_layer_info(self._h, C.byref(fused), C.byref(pairs)))
        return {"fused": bool(fused.value), "cta_pairs": bool(pairs.value)}

    def group_size(self) -> int:
        """The DECOUPLED signal-group size resolved at create (0 = per destination;
        group_size=-1 / GROUP_AUTO resolved to a size; 1 for per-tile protocols)."""
        g = C.c_int64()
        check(lib.perseus_layer_group_size(self._h, C.byref(g)))
        return g.value

    def set_trace(self, on: bool = True) -> None:
        """Device event log of every following forward (puts, fences, flag writes,
        receiver-side first observations with a content check; receive buffers
        are poisoned per forward).  Diagnostics: costs time."""
        check(lib.perseus_layer_set_trace(self._h, int(bool(on))))

    def trace(self) -> np.ndarray:
        """Events of the last forward as a structured array (perseus_trace_event)."""
        n = C.c_size_t(0)
        check(lib.perseus_layer_read_trace(self._h, None, 0, C.byref(n)))
        buf = (_lib.TraceEvent * max(1, n.value))()
        check(lib.perseus_layer_read_trace(self._h, buf, n.value, C.byref(n)))
        dt = np.dtype([("t", np.uint64), ("kind", np.int32), ("pe", np.int32), ("peer", np.int32),
                       ("tile", np.int32), ("group", np.int32), ("bytes", np.uint32), ("aux", np.uint32),
                       ("pad", np.uint32)])
        return np.frombuffer(bytes(buf), dtype=dt, count=n.value).copy()

    def set_timeline(self, on: bool = True) -> None:
        """Record a per-kernel device timeline of the following forwards (diagnostics)."""
        check(lib.perseus_layer_set_timeline(self._h, int(bool(on))))

    def timeline(self) -> dict:
        """{kernel: (start_ns, end_ns)} of the last forward, relative to its first kernel start."""
        n = len(self.TIMELINE_KERNELS)
        buf = (C.c_uint64 * (2 * n))()
        check(lib.perseus_layer_read_timeline(self._h, buf, n))
        starts = [buf[2 * i] for i in range(n) if buf[2 * i]]
        t0 = min(starts) if starts else 0
        return {name: ((buf[2 * i] - t0), (buf[2 * i + 1] - t0) if buf[2 * i + 1] else None)
                for i, name in enumerate(self.TIMELINE_KERNELS) if buf[2 * i]}

    def timing(self) -> List[float]:
        """Stage times (ms) of the last forward; needs set_stage_timing(True)."""
        ms = (C.c_float * 5)()
        check(lib.perseus_layer_read_timing(self._h, ms, 5))
        return list(ms)

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            check(lib.perseus_layer_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ordering_mode(protocol: ProtocolConfig) -> int:
    """0 ProxyFence (fence markers), 1 NicFence (flagged signals), 2 GPU-direct (neither)."""
    if protocol.transport == "gpu_direct":
        return 2
    return 1 if protocol.ordering == "nic_fence" else 0


def analyze_trace(events: np.ndarray, protocol: ProtocolConfig, transfers: np.ndarray) -> dict:
    """One forward's device events (all PEs, concatenated) -> sigsim::RunTrace per
    direction -> the reference's fence_accounting / verify_ordering /
    conservation_check (perseus_trace_analyze).  `transfers`: the realised
    dispatch transfers of all PEs (MoELayer.layout()[0] rows, concatenated)."""
    ev = np.ascontiguousarray(events)
    n = len(ev)
    ebuf = (_lib.TraceEvent * max(1, n)).from_buffer_copy(ev.tobytes() or bytes(C.sizeof(_lib.TraceEvent)))
    tr = np.asarray(transfers, dtype=np.int64).reshape(-1, 6)
    tbuf = (_lib.Transfer * max(1, len(tr)))()
    for i, row in enumerate(tr):
        tbuf[i] = _lib.Transfer(int(row[0]), int(row[1]), int(row[2]), int(row[3]), int(row[4]), int(row[5]))
    rep = _lib.TraceReport()
    check(lib.perseus_trace_analyze(ebuf, n, _ordering_mode(protocol), tbuf, len(tr), C.byref(rep)))
    return rep.as_dict()


def serialize_trace(events: np.ndarray, protocol: ProtocolConfig, direction: int = 0) -> str:
    """One direction's device RunTrace in the reference's text format (sigsim::serialize_trace)."""
    ev = np.ascontiguousarray(events)
    n = len(ev)
    ebuf = (_lib.TraceEvent * max(1, n)).from_buffer_copy(ev.tobytes() or bytes(C.sizeof(_lib.TraceEvent)))
    ln = C.c_size_t(0)
    nic = _ordering_mode(protocol)
    check(lib.perseus_trace_serialize(ebuf, n, nic, direction, None, 0, C.byref(ln)))
    buf = C.create_string_buffer(ln.value + 1)
    check(lib.perseus_trace_serialize(ebuf, n, nic, direction, buf, ln.value + 1, C.byref(ln)))
    return buf.value.decode()


def trace_records(events: np.ndarray, protocol: ProtocolConfig, direction: int = 0):
    """One direction's device RunTrace as flat records (perseus_trace_records):
    (ctypes array of _lib.TraceRecord, n, total_put_bytes_submitted,
    total_put_bytes_delivered) — what perseus_trace_analyze checks, handed out so
    the reference's own checkers can run on it."""
    ev = np.ascontiguousarray(events)
    n = len(ev)
    ebuf = (_lib.TraceEvent * max(1, n)).from_buffer_copy(ev.tobytes() or bytes(C.sizeof(_lib.TraceEvent)))
    ln, sub, dlv = C.c_size_t(0), C.c_uint64(0), C.c_uint64(0)
    mode = _ordering_mode(protocol)
    check(lib.perseus_trace_records(ebuf, n, mode, direction, None, 0, C.byref(ln), C.byref(sub), C.byref(dlv)))
    buf = (_lib.TraceRecord * max(1, ln.value))()
    check(lib.perseus_trace_records(ebuf, n, mode, direction, buf, ln.value, C.byref(ln), C.byref(sub),
                                    C.byref(dlv)))
    return buf, ln.value, sub.value, dlv.value
