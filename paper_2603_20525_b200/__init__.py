"""B200-native batched candidate-rollout planner (arxiv 2603.20525 hot path).

The product is libtmpc_b200.so (sm_100a CUDA + C ABI, include/tmpc_b200.h);
this package is its Python host mirror of the reference planner interface.
"""
from . import _abi  # noqa: F401
from .planner import *  # noqa: F401,F403

__version__ = "0.1.0"
