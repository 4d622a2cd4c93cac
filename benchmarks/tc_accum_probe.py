"""Probe the fp32 accumulation of the tcgen05 bf16 MMA (our grouped GEMM):
positive operands, compare against an fp64 reference of the same bf16 values.
Round-to-nearest accumulation gives an unbiased error ~sqrt(K) ulp; a
truncating adder gives a negative bias growing ~K ulp."""
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2205_10034_b200 import _lib, grouped_gemm  # noqa: E402
from paper_2205_10034_b200._lib import GemmProblem  # noqa: E402

dev = torch.device("cuda")
for K in (512, 4096, 16384):
    M, N = 256, 256
    g = torch.Generator(device="cuda").manual_seed(K)
    A = (torch.rand(M, K, device=dev, generator=g) * 0.5 + 0.5).to(torch.bfloat16)
    B = (torch.rand(N, K, device=dev, generator=g) * 0.5 + 0.5).to(torch.bfloat16)
    C = torch.empty(M, N, device=dev)
    i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)  # noqa: E731
    m, ar, b = i32([M]), i32([0]), i32([0])
    p = GemmProblem()
    p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_M, _lib.MOE_EPI_STORE
    p.dtype_ab, p.dtype_c = _lib.MOE_DTYPE_BF16, _lib.MOE_DTYPE_F32
    p.groups, p.N, p.K, p.a_rows, p.num_b = 1, N, K, M, 1
    p.m, p.a_row, p.c_row, p.b = m.data_ptr(), ar.data_ptr(), ar.data_ptr(), b.data_ptr()
    p.A, p.B, p.C = A.data_ptr(), B.data_ptr(), C.data_ptr()
    p.ldc = N
    grouped_gemm(p)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().t()
    rel = (C.double() - ref) / ref
    ulp = rel / 2.0 ** -24
    f32 = (A.float() @ B.float().t()).double()
    print(f"K={K}: mean err {ulp.mean().item():+.2f} ulp(2^-24 rel), std {ulp.std().item():.2f}, "
          f"max |rel| {rel.abs().max().item():.2e}; cuBLAS fp32 max |rel| "
          f"{((f32 - ref) / ref).abs().max().item():.2e}", flush=True)
