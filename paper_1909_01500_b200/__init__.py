"""B200-native replay + return-estimation hot path of rlpyt (arXiv 1909.01500).

librpl.so (CUDA, sm_100a) behind the C ABI in include/rpl.h; `ops` is the thin
torch binding with the ABI's names; `replay` holds the host-side shard logic.
Importing the package loads librpl.so and fails loudly if it is missing.
"""
from . import _lib  # noqa: F401  (loads librpl.so or raises)
from . import nvtx as _nvtx
from . import ops as _ops

_nvtx.install(_ops)  # RPL_NVTX=1: NVTX range per binding call (no-op otherwise)
from .ops import *  # noqa: E402,F401,F403

__version__ = "0.1.0"
