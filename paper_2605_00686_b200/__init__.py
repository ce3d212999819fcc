"""paper_2605_00686_b200 — B200-native Perseus MoE expert-parallel layer.

Hot path: one MoE-layer forward (gate/route -> dispatch -> SwiGLU expert FFN
-> combine, with Perseus decoupled signalling) in hand-written sm_100a CUDA
(libperseus.so), behind the reference's sigsim operator API.
"""
from ._lib import ConfigError, ModelError, VerifyError, lib  # noqa: F401  (fails loudly if the .so is missing)
from .layer import MoELayer, analyze_trace, resolve_group_size, serialize_trace, trace_records  # noqa: F401
from .sigsim import *  # noqa: F401,F403
