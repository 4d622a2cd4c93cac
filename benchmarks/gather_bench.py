"""Micro-benchmark of the gate-dgrad + gather-add GEMM (dx = dlogits wg +
sum_i dXe[slot_i]) at the layer shapes: c2 (T=65536, d=1024, top-1) and c4
(T=16384, d=4096, top-2).  Prints time, algorithmic bytes and GB/s.

    python benchmarks/gather_bench.py [--reps 20] [--only c2,c4]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2205_10034_b200 import _lib, grouped_gemm  # noqa: E402
from paper_2205_10034_b200._lib import GemmProblem  # noqa: E402

dev = torch.device("cuda")
SHAPES = {"c2": (65536, 1024, 64, 1, 1.25), "c3": (65536, 1024, 32, 2, 1.25),
          "c4": (16384, 4096, 64, 2, 1.25)}


def timed(fn, reps):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def problem(T, d, E, k, cf, seq=False):
    C = int(-(-k * cf * T // E))
    R = E * C
    Epad = 64
    dl = (torch.randn(T, Epad, device=dev) * 0.1).to(torch.bfloat16)
    wg = (torch.randn(Epad, d, device=dev) * 0.1).to(torch.bfloat16)
    src = torch.randn(R, d, device=dev).to(torch.bfloat16)
    if seq:
        slot = torch.arange(T * k, device=dev, dtype=torch.int32).remainder(R).view(T, k)
    else:
        slot = torch.randperm(R, device=dev)[: T * k].to(torch.int32).view(T, k)
    dx = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
    tab = torch.tensor([T, 0, 0, 0], dtype=torch.int32, device=dev)
    p = GemmProblem()
    p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_M, _lib.MOE_EPI_GATHER_ADD
    p.dtype_ab = p.dtype_c = _lib.MOE_DTYPE_BF16
    p.b_mn_major = 1
    p.groups, p.N, p.K, p.a_rows, p.num_b, p.b_rows = 1, d, Epad, T, 1, Epad
    p.m, p.a_row, p.c_row, p.b = (tab.data_ptr(), tab.data_ptr() + 4, tab.data_ptr() + 8,
                                  tab.data_ptr() + 12)
    p.A, p.B, p.C, p.ldc = dl.data_ptr(), wg.data_ptr(), dx.data_ptr(), d
    p.gather_src, p.gather_idx, p.gather_k = src.data_ptr(), slot.data_ptr(), k
    nbytes = T * Epad * 2 + Epad * d * 2 + T * k * d * 2 + T * d * 2 + T * k * 4
    return p, (dl, wg, src, slot, dx, tab), nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="c2,c4")
    ap.add_argument("--seq", action="store_true", help="sequential gather rows")
    a = ap.parse_args()
    for name in a.only.split(","):
        p, keep, nbytes = problem(*SHAPES[name], seq=a.seq)
        ms = timed(lambda: grouped_gemm(p), a.reps)
        print(f"{name} gather GEMM  {ms * 1e3:8.1f} us  {nbytes / 1e6:7.1f} MB  "
              f"{nbytes / ms / 1e6:7.1f} GB/s", flush=True)
        del keep


if __name__ == "__main__":
    main()
