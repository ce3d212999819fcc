"""Python mirror of the reference operator API for the hot path
(proj/include/sigsim/{workload,protocols,metrics}.hpp), calling the C ABI of
libperseus.so.  Same names, argument meaning and error behaviour
(ConfigError on bad geometry), so parity tests read like the reference's own
doctest cases (proj/tests/test_workload.cpp, test_protocols.cpp).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from ._lib import ConfigError, check, lib

__all__ = ["ModelConfig", "ClusterConfig", "TransferSpec", "DispatchWorkload", "SignalGroup",
           "ProtocolConfig", "model_preset", "model_preset_names", "remote_transfer_count",
           "message_size", "zipf_route", "build_dispatch", "assign_groups", "heap_digest",
           "fnv1a64", "vanilla_protocol", "decoupled_protocol", "nic_ordering_protocol",
           "combined_protocol", "gpu_direct_protocol", "expected_fences", "fit_alpha_beta"]


@dataclass
class ModelConfig:  # workload.hpp:16-25
    name: str = "custom"
    hidden_dim: int = 0
    intermediate_dim: int = 0
    experts: int = 0
    top_k: int = 0
    compute_intensity: float = 0.0

    def validate(self):
        if min(self.hidden_dim, self.intermediate_dim, self.experts, self.top_k) <= 0:
            raise ConfigError(f"model '{self.name}': all dimensions must be positive")
        if self.top_k > self.experts:
            raise ConfigError(f"model '{self.name}': top_k exceeds expert count")


_PRESETS = {  # workload.cpp:25-33 / PAPER.md:335-345
    "qwen3-30b": ModelConfig("qwen3-30b", 2048, 768, 128, 8, 4.6),
    "gpt-oss-120b": ModelConfig("gpt-oss-120b", 2880, 2880, 128, 4, 17.3),
    "deepseek-v3": ModelConfig("deepseek-v3", 7168, 2048, 256, 8, 0.0),
    "llama4-scout": ModelConfig("llama4-scout", 5120, 8192, 16, 1, 49.2),
}


def model_preset(name: str) -> Optional[ModelConfig]:
    m = _PRESETS.get(name)
    return None if m is None else ModelConfig(**m.__dict__)


def model_preset_names() -> List[str]:
    return list(_PRESETS)


@dataclass
class ClusterConfig:  # workload.hpp:31-38; EP=P on one NVSwitch box -> {P, 1, 1}
    nodes: int = 1
    gpus_per_node: int = 4
    num_qps: int = 1

    def total_pes(self) -> int:
        return self.nodes * self.gpus_per_node


@dataclass
class TransferSpec:  # workload.hpp:42-49
    src_pe: int = 0
    dst_pe: int = 0
    expert: int = -1
    bytes: int = 0
    tile_id: int = -1
    heap_offset: int = 0


@dataclass
class DispatchWorkload:  # workload.hpp:51-66
    model: ModelConfig
    cluster: ClusterConfig
    tokens_per_pe: int
    skew: float
    seed: int
    tile_bytes: int
    remote_transfers: List[TransferSpec] = field(default_factory=list)
    local_transfers: List[TransferSpec] = field(default_factory=list)
    _digest: int = 0

    def total_remote_bytes(self) -> int:
        return sum(t.bytes for t in self.remote_transfers)

    def digest(self) -> int:
        return self._digest

    def remote_array(self) -> np.ndarray:
        return np.array([(t.src_pe, t.dst_pe, t.expert, t.bytes, t.tile_id, t.heap_offset)
                         for t in self.remote_transfers], dtype=np.int64).reshape(-1, 6)


def remote_transfer_count(experts: int, pes: int, pes_per_node: int) -> int:
    out = C.c_int64(0)
    check(lib.perseus_remote_transfer_count(experts, pes, pes_per_node, C.byref(out)))
    return out.value


def message_size(tokens: int, top_k: int, experts: int, hidden_dim: int) -> int:
    return lib.perseus_message_size(tokens, top_k, experts, hidden_dim)


def zipf_route(tokens: int, experts: int, exponent: float, top_k: int, seed: int,
               want_ids: bool = False):
    counts = np.zeros(experts, dtype=np.uint64)
    ids = np.zeros(tokens * top_k, dtype=np.int32) if want_ids else None
    check(lib.perseus_zipf_route(tokens, experts, exponent, top_k, seed,
                                 counts.ctypes.data_as(C.POINTER(C.c_uint64)),
                                 ids.ctypes.data_as(C.POINTER(C.c_int32)) if want_ids else None))
    return (counts, ids) if want_ids else counts


def _to_specs(arr, n):
    return [TransferSpec(arr[i].src_pe, arr[i].dst_pe, arr[i].expert, arr[i].bytes, arr[i].tile_id,
                         arr[i].heap_offset) for i in range(n)]


def build_dispatch(model: ModelConfig, cluster: ClusterConfig, tokens: int, skew: float,
                   tile_bytes: int, seed: int) -> DispatchWorkload:
    nr, nl, dig = C.c_size_t(0), C.c_size_t(0), C.c_uint64(0)
    args = (model.hidden_dim, model.intermediate_dim, model.experts, model.top_k, cluster.nodes,
            cluster.gpus_per_node, cluster.num_qps, tokens, skew, tile_bytes, seed)
    check(lib.perseus_build_dispatch(*args, None, 0, C.byref(nr), None, 0, C.byref(nl),
                                     C.byref(dig)))
    R = (_lib.Transfer * max(nr.value, 1))()
    Lo = (_lib.Transfer * max(nl.value, 1))()
    check(lib.perseus_build_dispatch(*args, R, nr.value, C.byref(nr), Lo, nl.value, C.byref(nl),
                                     C.byref(dig)))
    return DispatchWorkload(model, cluster, tokens, skew, seed, tile_bytes, _to_specs(R, nr.value),
                            _to_specs(Lo, nl.value), dig.value)


@dataclass
class SignalGroup:  # protocols.hpp:47-56
    group_id: int
    members: List[int]
    leader: int
    target: int
    counter: int = 0


def _c_transfers(ts):
    arr = (_lib.Transfer * max(len(ts), 1))()
    for i, t in enumerate(ts):
        arr[i] = _lib.Transfer(t.src_pe, t.dst_pe, t.expert, t.bytes, t.tile_id, t.heap_offset)
    return arr


def assign_groups(transfers: List[TransferSpec], group_size: int) -> List[SignalGroup]:
    n = len(transfers)
    gof = (C.c_int64 * max(n, 1))()
    lead = (C.c_int64 * max(n, 1))()
    ng = C.c_size_t(0)
    check(lib.perseus_assign_groups(_c_transfers(transfers), n, group_size, gof, lead, C.byref(ng)))
    groups = [SignalGroup(g, [], lead[g], 0) for g in range(ng.value)]
    # members in (dst, expert, tile) order, like the reference
    order = sorted(range(n), key=lambda i: (transfers[i].dst_pe, transfers[i].expert,
                                            transfers[i].tile_id))
    for i in order:
        groups[gof[i]].members.append(i)
    for g in groups:
        g.target = len(g.members)
    return groups


def heap_digest(extents, flags) -> int:
    ext = np.ascontiguousarray(np.asarray(extents, dtype=np.uint64).reshape(-1, 3))
    fl = np.ascontiguousarray(np.asarray(flags, dtype=np.uint64).reshape(-1))
    return lib.perseus_heap_digest(ext.ctypes.data_as(C.POINTER(C.c_uint64)), ext.shape[0],
                                   fl.ctypes.data_as(C.POINTER(C.c_uint64)), fl.shape[0])


def fnv1a64(data: bytes, h: int = 0xcbf29ce484222325) -> int:
    return lib.perseus_fnv1a64(data, len(data), h)


@dataclass
class ProtocolConfig:  # protocols.hpp:20-37
    signaling: str = "coupled"        # coupled | decoupled
    ordering: str = "proxy_fence"     # proxy_fence | nic_fence
    transport: str = "proxy"          # proxy | gpu_direct
    group_size: int = 0               # 0 per destination PE; > 0 fixed; -1 (GROUP_AUTO, layer only) auto
    suppress_fences: bool = False
    # fault injection beyond the reference's suppress_fences: dispatch flags
    # written when a tile's put is issued, before its data (PERSEUS_SIGNAL_FAULT_EARLY)
    fault_early_signal: bool = False

    def mode_name(self) -> str:
        if self.transport == "gpu_direct":
            return "gpu_direct" if self.signaling == "coupled" else "gpu_direct_decoupled"
        nic = self.ordering == "nic_fence"
        if self.signaling == "coupled":
            return "nic_ordering" if nic else "vanilla"
        return "combined" if nic else "decoupled"

    def device_signaling(self) -> int:
        """The device variant this protocol selects (include/perseus.h)."""
        if self.fault_early_signal:
            return _lib.SIGNAL_FAULT_EARLY
        if self.suppress_fences:
            return _lib.SIGNAL_NONE
        return _lib.SIGNAL_COUPLED if self.signaling == "coupled" else _lib.SIGNAL_DECOUPLED


def vanilla_protocol():
    return ProtocolConfig()


def decoupled_protocol(group_size: int = 0):
    return ProtocolConfig(signaling="decoupled", group_size=group_size)


def nic_ordering_protocol():
    return ProtocolConfig(ordering="nic_fence")


def combined_protocol(group_size: int = 0):
    return ProtocolConfig(signaling="decoupled", ordering="nic_fence", group_size=group_size)


def gpu_direct_protocol(signaling: str = "coupled"):
    return ProtocolConfig(signaling=signaling, transport="gpu_direct")


def expected_fences(protocol: ProtocolConfig, wl: DispatchWorkload, src_pe: int) -> int:
    """FenceMarker submits of one PE (what fence_accounting counts, metrics.cpp:10-59)."""
    if protocol.transport == "gpu_direct" or protocol.suppress_fences:
        return 0
    own = [t for t in wl.remote_transfers if t.src_pe == src_pe]
    if protocol.signaling == "coupled":
        return len(own)
    return len(assign_groups(own, protocol.group_size)) if own else 0


def fit_alpha_beta(points):
    """sigsim::fit_alpha_beta (metrics.cpp:69-95): least-squares t = alpha + beta*bytes
    over [(bytes, ns), ...]; returns (alpha_ns, beta_ns_per_byte, r_squared)."""
    xs = (C.c_double * len(points))(*[float(p[0]) for p in points])
    ys = (C.c_double * len(points))(*[float(p[1]) for p in points])
    a, b, r2 = C.c_double(), C.c_double(), C.c_double()
    check(lib.perseus_fit_alpha_beta(xs, ys, len(points), C.byref(a), C.byref(b), C.byref(r2)))
    return a.value, b.value, r2.value
