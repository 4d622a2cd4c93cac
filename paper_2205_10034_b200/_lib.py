"""ctypes binding of the C-ABI in include/moe_b200.h (libmoe_b200.so).

The shared library is the product: there is no Python or CPU fallback.  If the
library is missing this module raises at import time.  Status codes map to the
reference's exception taxonomy:

    MOE_ERR_INVALID_ARGUMENT -> ValueError   (std::invalid_argument)
    MOE_ERR_OUT_OF_RANGE     -> IndexError   (std::out_of_range)
    MOE_ERR_CONFIG           -> ConfigError  (moesim::ConfigError, types.hpp:24-26)
    MOE_ERR_LOGIC            -> LogicError   (std::logic_error)
    MOE_ERR_CUDA / _NCCL     -> CudaError / NcclError
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# MOE_B200_LIB: load another build of the same ABI (A/B benchmarking only)
LIB_PATH = os.environ.get("MOE_B200_LIB") or os.path.join(_HERE, "libmoe_b200.so")

MOE_OK = 0
MOE_ERR_INVALID_ARGUMENT = 1
MOE_ERR_OUT_OF_RANGE = 2
MOE_ERR_CONFIG = 3
MOE_ERR_LOGIC = 4
MOE_ERR_CUDA = 5
MOE_ERR_NCCL = 6

MOE_DTYPE_F32 = 0
MOE_DTYPE_BF16 = 1

MOE_GEMM_RAGGED_M = 0
MOE_GEMM_RAGGED_K = 1
MOE_EPI_STORE = 0
MOE_EPI_GELU = 1
MOE_EPI_DGELU = 2
MOE_EPI_ATOMIC_ADD = 3
MOE_EPI_GATHER_ADD = 4


class ConfigError(RuntimeError):
    """moesim::ConfigError: message is '<field>: <reason>'."""


class LogicError(RuntimeError):
    """std::logic_error."""


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


_EXC = {
    MOE_ERR_INVALID_ARGUMENT: ValueError,
    MOE_ERR_OUT_OF_RANGE: IndexError,
    MOE_ERR_CONFIG: ConfigError,
    MOE_ERR_LOGIC: LogicError,
    MOE_ERR_CUDA: CudaError,
    MOE_ERR_NCCL: NcclError,
}


class SliceIndexEntry(C.Structure):
    _fields_ = [("slice_id", C.c_uint64), ("offset", C.c_uint64), ("length", C.c_uint64)]


class RoutingOut(C.Structure):
    _fields_ = [
        ("expert", C.c_void_p),
        ("gate", C.c_void_p),
        ("position", C.c_void_p),
        ("keep", C.c_void_p),
        ("count1", C.c_void_p),
        ("count2", C.c_void_p),
        ("kept", C.c_void_p),
        ("aux_loss", C.c_void_p),
    ]


class GemmProblem(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("epilogue", C.c_int),
        ("dtype_ab", C.c_int),
        ("dtype_c", C.c_int),
        ("b_mn_major", C.c_int),
        ("transpose_c", C.c_int),
        ("groups", C.c_uint32),
        ("M", C.c_uint32),
        ("N", C.c_uint32),
        ("K", C.c_uint32),
        ("a_rows", C.c_uint64),
        ("num_b", C.c_uint32),
        ("m", C.c_void_p),
        ("a_row", C.c_void_p),
        ("c_row", C.c_void_p),
        ("b", C.c_void_p),
        ("A", C.c_void_p),
        ("B", C.c_void_p),
        ("C", C.c_void_p),
        ("C2", C.c_void_p),
        ("aux", C.c_void_p),
        ("bias", C.c_void_p),
        ("ldc", C.c_uint64),
        ("lda", C.c_uint64),
        ("ldb", C.c_uint64),
        ("b_rows", C.c_uint64),
        ("c_rows", C.c_uint64),
        ("colsum", C.c_void_p),
        ("gather_src", C.c_void_p),
        ("gather_idx", C.c_void_p),
        ("gather_k", C.c_uint32),
        ("colsum_ws", C.c_void_p),
        ("colsum_max_m", C.c_uint64),
        ("split_terms", C.c_uint32),
        ("k_begin", C.c_uint32),
        ("k_len", C.c_uint32),
        ("k_begin_g", C.c_void_p),
    ]


class CacheParams(C.Structure):
    _fields_ = [("cpu_size", C.c_uint64), ("threshold", C.c_double), ("beta", C.c_double),
                ("decay_steps", C.c_uint32)]


class CacheAccess(C.Structure):
    _fields_ = [("kind", C.c_int32), ("victim", C.c_uint64)]


class PrefetchDesc(C.Structure):
    _fields_ = [("num_layers", C.c_uint32), ("lookahead", C.c_uint32), ("cache", CacheParams),
                ("flush_period", C.c_uint32), ("host_sections", C.c_void_p),
                ("gate_weights", C.c_void_p), ("backing_path", C.c_char_p)]


class PrefetchRecord(C.Structure):
    _fields_ = [("step", C.c_uint32), ("layer", C.c_uint32), ("kind", C.c_int32),
                ("victim", C.c_uint64), ("io_ms", C.c_float), ("h2d_start", C.c_float),
                ("h2d_end", C.c_float), ("compute_start", C.c_float), ("compute_end", C.c_float)]


class PrefetchSummary(C.Structure):
    _fields_ = [("makespan_ms", C.c_float), ("compute_total_ms", C.c_float),
                ("stall_total_ms", C.c_float), ("io_total_ms", C.c_float),
                ("bytes_read", C.c_uint64), ("bytes_written", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("section_bytes", C.c_uint64), ("gpu_slots", C.c_uint32)]


class LayerDesc(C.Structure):
    _fields_ = [
        ("num_experts", C.c_uint32),
        ("top_k", C.c_uint32),
        ("d_model", C.c_uint32),
        ("d_ff", C.c_uint32),
        ("capacity_factor", C.c_double),
        ("tokens", C.c_uint64),
        ("dtype", C.c_int),
        ("has_gate_bias", C.c_int),
        ("ep_size", C.c_uint32),
        ("ep_rank", C.c_uint32),
        ("nccl_comm", C.c_void_p),
        ("exchange", C.c_uint32),
        ("placement", C.c_uint32),
        ("gate_grad_reduce", C.c_uint32),
    ]


class LayerParams(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("wg", "bg", "w1", "b1", "w2", "b2")]


class LayerGrads(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("dwg", "dbg", "dw1", "db1", "dw2", "db2")]


class RingDesc(C.Structure):
    _fields_ = [
        ("num_layers", C.c_uint32),
        ("ring_slots", C.c_uint32),
        ("host_sections", C.c_void_p),
        ("gate_weights", C.c_void_p),
        ("gate_bias", C.c_void_p),
    ]


class RingTimeline(C.Structure):
    _fields_ = [
        ("load_start", C.c_void_p),
        ("load_end", C.c_void_p),
        ("compute_start", C.c_void_p),
        ("compute_end", C.c_void_p),
        ("makespan_ms", C.c_float),
        ("compute_total_ms", C.c_float),
        ("peak_gpu_bytes", C.c_uint64),
        ("baseline_gpu_bytes", C.c_uint64),
        ("slots", C.c_uint32),
        ("clamped", C.c_int),
    ]


# name -> (restype, argtypes); every symbol declared in include/moe_b200.h
_VP, _U64, _U32, _I, _D, _F = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double, C.c_float
SIGNATURES = {
    "moe_last_error": (C.c_char_p, []),
    "moe_abi_version": (C.c_int, []),
    "moe_kernel_launch_count": (_U64, []),
    "moe_abi_sizeof": (_U64, [C.c_char_p]),
    "moesim_alltoall_flat": (_I, [_U64, _U64, _VP, _VP, _VP, _VP]),
    "moesim_alltoall_hierarchical": (_I, [_U32, _U32, _U32, _U64, _U64, _VP, _VP, _VP, _VP,
                                          _VP]),
    "moesim_fuse_slices": (_I, [_U64, _VP, _VP, _VP, _VP]),
    "moesim_split_blob": (_I, [_U64, _VP, _U64, _VP, _VP]),
    "moesim_gen_trace": (_I, [_U64, _U32, _U32, _U32, _U64, _D, _VP]),
    "moesim_imbalance_ratio": (_I, [_U32, _U32, _U32, _VP, _VP]),
    "moesim_ring_build_schedule": (_I, [_U32, _U32, _VP, _U64, _VP, _VP, _VP]),
    "moe_fill_uniform": (_I, [_VP, _U64, _I, _U64, _D, _D, _VP]),
    "moe_gen_trace_device": (_I, [_U64, _U32, _U32, _U32, _U64, _D, _VP, _VP]),
    "moe_alltoall_flat_device": (_I, [_U64, _VP, _VP, _VP, _VP, _VP, _VP]),
    "moe_fuse_slices_device": (_I, [_U64, _VP, _VP, _VP, _VP, _VP]),
    "moe_split_blob_device": (_I, [_U64, _VP, _U64, _VP, _VP, _VP, _VP]),
    "moe_route": (_I, [_U64, _U32, _U32, _U64, _VP, C.POINTER(RoutingOut), _VP]),
    "moe_grouped_gemm": (_I, [C.POINTER(GemmProblem), _VP]),
    "moe_layer_create": (_I, [C.POINTER(LayerDesc), C.POINTER(_VP)]),
    "moe_layer_destroy": (_I, [_VP]),
    "moe_layer_capacity": (_U64, [_VP]),
    "moe_layer_forward": (_I, [_VP, C.POINTER(LayerParams), _VP, _VP, _VP, _VP,
                               C.POINTER(RoutingOut), _VP]),
    "moe_layer_backward": (_I, [_VP, C.POINTER(LayerParams), _VP, _F, _VP,
                                C.POINTER(LayerGrads), _VP]),
    "moe_layer_train_step_host": (_I, [_VP, C.POINTER(LayerParams), _VP, _VP, _F, _VP, _VP,
                                       C.POINTER(LayerGrads), _VP]),
    "moe_layer_train_step_host_async": (_I, [_VP, C.POINTER(LayerParams), _VP, _VP, _F, _VP,
                                             _VP, C.POINTER(LayerGrads), _VP]),
    "moe_layer_host_sync": (_I, [_VP, _VP]),
    "moe_split_f32_bf16x3": (_I, [_VP, _U64, _VP, _VP]),
    "moe_layer_set_profiling": (_I, [_VP, _I]),
    "moe_layer_set_peer_timeout": (_I, [_VP, C.c_double]),
    "moe_layer_comm_status": (_I, [_VP, C.POINTER(C.c_int32)]),
    "moe_layer_phase_times": (_I, [_VP, C.POINTER(C.c_char_p), C.POINTER(_F), _U32,
                                   C.POINTER(_U32)]),
    "moe_layer_phase_times_of": (_I, [_VP, _I, C.POINTER(C.c_char_p), C.POINTER(_F), _U32,
                                   C.POINTER(_U32)]),
    "moe_comm_unique_id": (_I, [_VP]),
    "moe_comm_create": (_I, [_VP, _U32, _U32, C.POINTER(_VP)]),
    "moe_comm_destroy": (_I, [_VP]),
    "moe_alltoall_packed": (_I, [_VP, _VP, _VP, _U64, _U32, _I, _VP]),
    "moe_prefetch_create": (_I, [_VP, C.POINTER(PrefetchDesc), C.POINTER(_VP)]),
    "moe_prefetch_destroy": (_I, [_VP]),
    "moe_prefetch_run": (_I, [_VP, _U32, _VP, _VP, _VP, C.POINTER(PrefetchSummary), _VP]),
    "moe_sparse_cache_create": (_I, [C.POINTER(CacheParams), C.POINTER(_VP)]),
    "moe_sparse_cache_destroy": (_I, [_VP]),
    "moe_sparse_cache_access": (_I, [_VP, _U64, C.POINTER(CacheAccess)]),
    "moe_sparse_cache_end_step": (_I, [_VP]),
    "moe_sparse_cache_state": (_I, [_VP, C.POINTER(_U64), C.POINTER(_U32), _VP, _VP, _U64,
                                    C.POINTER(_U64)]),
    "moe_grad_buckets_create": (_I, [_VP, _U32, _VP, _VP, _VP, _U32, C.c_float, C.POINTER(_VP)]),
    "moe_grad_buckets_destroy": (_I, [_VP]),
    "moe_grad_buckets_push": (_I, [_VP, _U64, _VP, C.POINTER(C.c_int32)]),
    "moe_grad_buckets_reset": (_I, [_VP]),
    "moe_grad_buckets_count": (_U32, [_VP]),
    "moe_grad_buckets_ids": (_I, [_VP, _U32, _VP, _U32, C.POINTER(_U32)]),
    "moe_ring_create": (_I, [_VP, C.POINTER(RingDesc), C.POINTER(_VP)]),
    "moe_ring_destroy": (_I, [_VP]),
    "moe_ring_section_bytes": (_U64, [_VP]),
    "moe_ring_pack_section": (_I, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "moe_ring_run": (_I, [_VP, _VP, _VP, C.POINTER(RingTimeline), _VP]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA extension is not built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
            "There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

STRUCTS = {
    "moe_slice_index_entry_t": SliceIndexEntry, "moe_routing_out_t": RoutingOut,
    "moe_gemm_problem_t": GemmProblem, "moe_layer_desc_t": LayerDesc,
    "moe_layer_params_t": LayerParams, "moe_layer_grads_t": LayerGrads,
    "moe_ring_desc_t": RingDesc, "moe_ring_timeline_t": RingTimeline,
    "moe_cache_params_t": CacheParams, "moe_cache_access_t": CacheAccess,
    "moe_prefetch_desc_t": PrefetchDesc, "moe_prefetch_record_t": PrefetchRecord,
    "moe_prefetch_summary_t": PrefetchSummary,
}
for _n, _t in STRUCTS.items():  # layouts must match include/moe_b200.h exactly
    _sz = lib.moe_abi_sizeof(_n.encode())
    if _sz != C.sizeof(_t):
        raise ImportError(f"ABI mismatch: {_n} is {_sz} bytes in the library, "
                          f"{C.sizeof(_t)} in the Python binding")


def check(status: int) -> None:
    """Raise the Python mirror of the reference exception for a status."""
    if status == MOE_OK:
        return
    msg = lib.moe_last_error().decode()
    raise _EXC.get(status, RuntimeError)(msg)


def call(name: str, *args):
    check(getattr(lib, name)(*args))
