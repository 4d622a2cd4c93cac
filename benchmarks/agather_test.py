"""Experiment: expert GEMM whose A rows are gathered by TMA gather4 through a
row-index map (the dispatch folded into the GEMM's producer) vs the same GEMM
on the materialised permuted rows.  Needs a library built with
-DMOE_A_GATHER=1 (benchmarks/build_variant.sh agather ...)."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2205_10034_b200 import _lib, grouped_gemm  # noqa: E402
from paper_2205_10034_b200._lib import GemmProblem  # noqa: E402
from gemm_sweep import timed  # noqa: E402

dev = torch.device("cuda")


def run(G, rows, N, K, b_mn=False, reps=20):
    T = G * rows
    X = torch.randn(T, K, device=dev).to(torch.bfloat16)
    perm = torch.randperm(T, device=dev).to(torch.int32)
    Xp = X[perm.long()].contiguous()
    B = (torch.randn(G, K, N, device=dev) if b_mn else torch.randn(G, N, K, device=dev)).to(torch.bfloat16)
    i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)
    m, ar, b = i32([rows] * G), i32([g * rows for g in range(G)]), i32(list(range(G)))
    outs, times = [], []
    for gather in (False, True):
        C = torch.empty(T, N, device=dev, dtype=torch.bfloat16)
        p = GemmProblem()
        p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_M, _lib.MOE_EPI_STORE
        p.dtype_ab = p.dtype_c = _lib.MOE_DTYPE_BF16
        p.b_mn_major = 1 if b_mn else 0
        p.groups, p.N, p.K, p.a_rows, p.num_b = G, N, K, T, G
        p.m, p.a_row, p.c_row, p.b = m.data_ptr(), ar.data_ptr(), ar.data_ptr(), b.data_ptr()
        p.A = (X if gather else Xp).data_ptr()
        p.B, p.C, p.ldc = B.data_ptr(), C.data_ptr(), N
        if gather:
            p.gather_idx, p.gather_k = perm.data_ptr(), 0
        ms = timed(lambda: grouped_gemm(p), reps)
        torch.cuda.synchronize()
        outs.append(C.clone())
        times.append(ms)
    ok = torch.equal(outs[0], outs[1])
    f = 2.0 * T * N * K
    print(f"G={G} rows={rows} N={N} K={K} b_mn={b_mn}: materialised {times[0]*1e3:.1f} us "
          f"({f/times[0]/1e9:.0f} TF/s), gathered {times[1]*1e3:.1f} us ({f/times[1]/1e9:.0f} TF/s), "
          f"bitwise equal: {ok}", flush=True)


if __name__ == "__main__":
    run(64, 1024, 4096, 1024)          # ffn1 shape (K = d)
    run(64, 1024, 1024, 4096)          # ffn2 shape (K = d_ff)
    run(64, 1030, 4096, 1024)          # ragged tails
