"""B200-native SE-MoE MoE-layer hot path (arXiv 2205.10034).

The compute lives in libmoe_b200.so (sm_100a CUDA behind the C-ABI of
include/moe_b200.h); this package is the host-side mirror of the reference's
interface (moesim.py) plus the MoE-layer operator (layer.py) and the
ring-of-sections runner (ring.py).  Importing it without the built library
raises ImportError: there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (loads libmoe_b200.so or raises)
from ._lib import ConfigError, CudaError, LogicError, NcclError  # noqa: F401
from .layer import (EPGroup, MoEConfig, MoELayer, capacity, fill_uniform,  # noqa: F401
                    grouped_gemm, kernel_launch_count, route, substream_seed)

__all__ = [
    "ConfigError", "CudaError", "LogicError", "NcclError", "EPGroup", "MoEConfig", "MoELayer",
    "capacity", "fill_uniform", "grouped_gemm", "kernel_launch_count", "route", "substream_seed",
]
