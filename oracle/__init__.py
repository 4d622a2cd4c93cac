"""ORACLE — TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end of oracle/liboracle.so (the C restatement in
oracle/moe_oracle.c) and, when present, oracle/_ref/libmoesim_ref.so (the
reference compiled from /root/reference/proj sources by oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package, and only as the checker or the reported CPU baseline.
Gating / capacity / FFN arithmetic is PARITY UNPINNED (no reference
implementation exists); DESIGN.md Appendix A fixes it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoesim_ref.so")
MASK64 = (1 << 64) - 1


def build(ref: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", HERE, "all"] + (["ref"] if ref else []), check=True)


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        _lib = C.CDLL(ORACLE_SO)
        _lib.oracle_splitmix64_next.restype = C.c_uint64
        _lib.oracle_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
        _lib.oracle_substream_seed.restype = C.c_uint64
        _lib.oracle_substream_seed.argtypes = [C.c_uint64] * 3
        _lib.oracle_fill_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_double, C.c_double,
                                             C.c_void_p]
        _lib.oracle_round_bf16.argtypes = [C.c_uint64, C.c_void_p]
        _lib.oracle_gen_trace.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint64, C.c_double, C.c_void_p]
        _lib.oracle_imbalance_ratio.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                                C.POINTER(C.c_double)]
        _lib.oracle_alltoall_flat.argtypes = [C.c_uint64] * 2 + [C.c_void_p] * 4
        _lib.oracle_alltoall_hierarchical.argtypes = [C.c_uint32] * 3 + [C.c_uint64] * 2 + [
            C.c_void_p] * 5
        _lib.oracle_fuse_slices.argtypes = [C.c_uint64] + [C.c_void_p] * 4
        _lib.oracle_split_blob.argtypes = [C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                           C.c_void_p]
        _lib.oracle_ring_schedule.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p]
        _lib.oracle_ring_simulate.argtypes = ([C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                               C.c_void_p, C.c_uint64, C.c_int64]
                                              + [C.c_void_p] * 9)
        _lib.oracle_route.argtypes = ([C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]
                                      + [C.c_void_p] * 10)
        _lib.oracle_moe_forward.argtypes = ([C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.c_uint32, C.c_uint64, C.c_int] + [C.c_void_p] * 17)
        _lib.oracle_moe_backward.argtypes = ([C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                              C.c_uint32, C.c_uint64, C.c_int]
                                             + [C.c_void_p] * 13 + [C.c_double]
                                             + [C.c_void_p] * 8)
        _lib.oracle_num_threads.restype = C.c_int
        _lib.oracle_set_threads.argtypes = [C.c_int]
    return _lib


def ref():
    """The compiled reference (None when oracle/_ref was not built)."""
    global _ref
    if _ref is None:
        _ref = _load(REF_SO)
        if _ref is not None:
            _ref.ref_splitmix64_next.restype = C.c_uint64
            _ref.ref_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
            _ref.ref_substream_seed.restype = C.c_uint64
            _ref.ref_substream_seed.argtypes = [C.c_uint64] * 3
            _ref.ref_sparse_cache_run.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint32,
                                                  C.c_void_p, C.c_uint64] + [C.c_void_p] * 4 + [
                C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
            _ref.ref_trace_to_json.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                               C.c_void_p, C.c_char_p, C.c_uint64,
                                               C.POINTER(C.c_uint64)]
            _ref.ref_trace_from_json.argtypes = [C.c_char_p] + [C.c_void_p] * 5 + [
                C.c_uint64, C.c_char_p, C.c_uint64]
            _ref.ref_gen_trace.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                           C.c_uint64, C.c_double, C.c_void_p]
            _ref.ref_imbalance_ratio.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                                 C.POINTER(C.c_double)]
            _ref.ref_alltoall_flat.argtypes = [C.c_uint64] * 2 + [C.c_void_p] * 4
            _ref.ref_alltoall_hierarchical.argtypes = [C.c_uint32] * 3 + [C.c_uint64] * 2 + [
                C.c_void_p] * 5
            _ref.ref_fuse_slices.argtypes = [C.c_uint64] + [C.c_void_p] * 4
            _ref.ref_split_blob.argtypes = [C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                            C.c_void_p]
            _ref.ref_ring_schedule.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_void_p]
            _ref.ref_ring_simulate.argtypes = ([C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                                C.c_void_p, C.c_uint64, C.c_int64]
                                               + [C.c_void_p] * 9)
    return _ref


def P(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def substream_seed(seed: int, step: int, rank: int) -> int:
    return int(lib().oracle_substream_seed(seed & MASK64, step, rank))


def fill_uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    lib().oracle_fill_uniform(seed & MASK64, n, lo, hi, P(out))
    return out


def round_bf16(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float32).copy()
    lib().oracle_round_bf16(a.size, P(a))
    return a


# ---------------------------------------------------------------- workload --
def gen_trace(seed, steps, ranks, experts, tokens, skew, which="oracle") -> np.ndarray:
    counts = np.zeros((steps, ranks, max(experts, 1)), dtype=np.uint64)
    fn = lib().oracle_gen_trace if which == "oracle" else ref().ref_gen_trace
    rc = fn(seed & MASK64, steps, ranks, experts, tokens, float(skew), P(counts))
    if rc:
        raise ValueError(f"gen_trace: status {rc}")
    return counts[:, :, :experts]


def imbalance_ratio(counts: np.ndarray, which="oracle") -> float:
    s, r, e = counts.shape
    c = np.ascontiguousarray(counts, dtype=np.uint64)
    out = C.c_double()
    fn = lib().oracle_imbalance_ratio if which == "oracle" else ref().ref_imbalance_ratio
    rc = fn(s, r, e, P(c), C.byref(out))
    if rc:
        raise ValueError(f"imbalance_ratio: status {rc}")
    return out.value


# ---------------------------------------------------------------- routing --
def route(logits: np.ndarray, k: int, capacity: int) -> Dict[str, np.ndarray]:
    L = np.ascontiguousarray(logits, dtype=np.float32)
    T, E = L.shape
    o = {
        "expert": np.zeros((T, k), np.int32), "gate": np.zeros((T, k), np.float64),
        "position": np.zeros((T, k), np.int32), "keep": np.zeros((T, k), np.uint8),
        "count1": np.zeros(E, np.int32), "count2": np.zeros(E, np.int32),
        "kept": np.zeros(E, np.int32), "probs": np.zeros((T, E), np.float64),
    }
    aux = C.c_double()
    rc = lib().oracle_route(T, E, k, capacity, P(L), P(o["expert"]), P(o["gate"]),
                            P(o["position"]), P(o["keep"]), P(o["count1"]), P(o["count2"]),
                            P(o["kept"]), C.byref(aux), P(o["probs"]))
    if rc:
        raise ValueError(f"route: status {rc}")
    o["aux_loss"] = aux.value
    return o


# -------------------------------------------------------------- MoE layer --
def moe_forward(x, wg, bg, w1, b1, w2, b2, k, capacity, emulate_bf16, logits_in=None):
    """All arrays float32 numpy (bf16 values already rounded).  Returns dict."""
    T, d = x.shape
    E = wg.shape[0]
    dff = w1.shape[1]
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    x, wg, bg, w1, b1, w2, b2, li = map(f, (x, wg, bg, w1, b1, w2, b2, logits_in))
    o = {
        "logits": np.zeros((T, E), np.float32), "expert": np.zeros((T, k), np.int32),
        "gate": np.zeros((T, k), np.float64), "position": np.zeros((T, k), np.int32),
        "keep": np.zeros((T, k), np.uint8), "count1": np.zeros(E, np.int32),
        "count2": np.zeros(E, np.int32), "kept": np.zeros(E, np.int32),
        "y": np.zeros((T, d), np.float64),
    }
    aux = C.c_double()
    rc = lib().oracle_moe_forward(T, d, dff, E, k, capacity, 1 if emulate_bf16 else 0, P(x),
                                  P(wg), P(bg), P(w1), P(b1), P(w2), P(b2), P(li), P(o["logits"]),
                                  P(o["expert"]), P(o["gate"]), P(o["position"]), P(o["keep"]),
                                  P(o["count1"]), P(o["count2"]), P(o["kept"]), C.byref(aux),
                                  P(o["y"]))
    if rc:
        raise ValueError(f"moe_forward: status {rc}")
    o["aux_loss"] = aux.value
    return o


def moe_backward(x, wg, bg, w1, b1, w2, b2, k, capacity, emulate_bf16, fwd, dy, d_aux):
    T, d = x.shape
    E = wg.shape[0]
    dff = w1.shape[1]
    f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float32)  # noqa: E731
    x, wg, bg, w1, b1, w2, b2, dy = map(f, (x, wg, bg, w1, b1, w2, b2, dy))
    logits = np.ascontiguousarray(fwd["logits_used"], dtype=np.float32)
    o = {
        "dx": np.zeros((T, d)), "dwg": np.zeros((E, d)), "dbg": np.zeros(E),
        "dw1": np.zeros((E, dff, d)), "db1": np.zeros((E, dff)), "dw2": np.zeros((E, d, dff)),
        "db2": np.zeros((E, d)), "dlogits": np.zeros((T, E)),
    }
    rc = lib().oracle_moe_backward(T, d, dff, E, k, capacity, 1 if emulate_bf16 else 0, P(x),
                                   P(wg), P(bg), P(w1), P(b1), P(w2), P(b2), P(logits),
                                   P(fwd["expert"]), P(fwd["gate"]), P(fwd["keep"]),
                                   P(fwd["count1"]), P(dy), float(d_aux), P(o["dx"]),
                                   P(o["dwg"]), P(o["dbg"]), P(o["dw1"]), P(o["db1"]),
                                   P(o["dw2"]), P(o["db2"]), P(o["dlogits"]))
    if rc:
        raise ValueError(f"moe_backward: status {rc}")
    return o


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


# ----------------------------------------------------- synthetic tensors ----
def make_layer_tensors(seed, T, d, dff, E, bf16, rank=0, gate_bias=None):
    """Same tensors as paper_2205_10034_b200.layer.MoELayer.init_params /
    make_input (SplitMix64 substreams, tensor ids 0..7)."""
    import math
    bd, bf = 1.0 / math.sqrt(d), 1.0 / math.sqrt(dff)
    rb = round_bf16 if bf16 else (lambda a: a)
    wg = rb(fill_uniform(substream_seed(seed, 0, 0), E * d, -bd, bd)).reshape(E, d)
    w1 = np.stack([rb(fill_uniform(substream_seed(seed, 2, e), dff * d, -bd, bd)).reshape(dff, d)
                   for e in range(E)])
    b1 = np.stack([fill_uniform(substream_seed(seed, 3, e), dff, -bd, bd) for e in range(E)])
    w2 = np.stack([rb(fill_uniform(substream_seed(seed, 4, e), d * dff, -bf, bf)).reshape(d, dff)
                   for e in range(E)])
    b2 = np.stack([fill_uniform(substream_seed(seed, 5, e), d, -bf, bf) for e in range(E)])
    x = rb(fill_uniform(substream_seed(seed, 6, rank), T * d, -1.0, 1.0)).reshape(T, d)
    dy = rb(fill_uniform(substream_seed(seed, 7, rank), T * d, -1.0, 1.0)).reshape(T, d)
    bg = None if gate_bias is None else np.asarray(gate_bias, dtype=np.float32)
    return dict(x=x, dy=dy, wg=wg, bg=bg, w1=w1, b1=b1, w2=w2, b2=b2)
