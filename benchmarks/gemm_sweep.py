"""Grouped-GEMM micro-benchmark at the c2 layer shapes (E=64 groups, 1024 rows
each, d=1024, d_ff=4096): isolates operand layout (K- vs MN-major), output
dtype and epilogue cost of the tcgen05 kernel.  Prints one line per variant:
time (CUDA events, median of reps) and TFLOP/s.

    python benchmarks/gemm_sweep.py [--reps 20] [--rows 1024]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2205_10034_b200 import _lib, grouped_gemm  # noqa: E402
from paper_2205_10034_b200._lib import GemmProblem  # noqa: E402

dev = torch.device("cuda")


def i32(v):
    return torch.tensor(v, dtype=torch.int32, device=dev)


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


SHARED_B = False
B_MOD = 0


def ragged_m(G, rows, N, K, epi=0, b_mn=False, out_f32=False, colsum=True):
    A = torch.randn(G * rows, K, device=dev).to(torch.bfloat16)
    B = (torch.randn(G, K, N, device=dev) if b_mn else torch.randn(G, N, K, device=dev)).to(torch.bfloat16)
    cdt = torch.float32 if out_f32 else torch.bfloat16
    Cm = torch.empty(G * rows, N, device=dev, dtype=cdt)
    C2 = torch.empty_like(Cm)
    aux = torch.randn(G * rows, N, device=dev).to(cdt)
    bias = torch.randn(G, N, device=dev)
    m, ar, b = i32([rows] * G), i32([g * rows for g in range(G)]), i32([0] * G if SHARED_B else [g % B_MOD if B_MOD else g for g in range(G)])
    cs = torch.zeros(G, N, device=dev)
    p = GemmProblem()
    p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_M, epi
    p.dtype_ab = _lib.MOE_DTYPE_BF16
    p.dtype_c = _lib.MOE_DTYPE_F32 if out_f32 else _lib.MOE_DTYPE_BF16
    p.b_mn_major = 1 if b_mn else 0
    p.groups, p.N, p.K, p.a_rows, p.num_b = G, N, K, G * rows, G
    p.m, p.a_row, p.c_row, p.b = m.data_ptr(), ar.data_ptr(), ar.data_ptr(), b.data_ptr()
    p.A, p.B, p.C, p.C2, p.aux = A.data_ptr(), B.data_ptr(), Cm.data_ptr(), C2.data_ptr(), aux.data_ptr()
    p.bias = bias.data_ptr() if epi in (0, 1) else None
    ws = torch.empty(G * ((rows + 31) // 32) * N, device=dev)
    if epi == 2 and colsum:
        p.colsum = cs.data_ptr()
        p.colsum_ws, p.colsum_max_m = ws.data_ptr(), rows
    p.ldc = N
    keep = (A, B, Cm, C2, aux, bias, m, ar, b, cs, ws)
    return p, keep, 2.0 * G * rows * N * K


def ragged_k(G, rows, M, N, out_f32=True):
    A = torch.randn(G * rows, M, device=dev).to(torch.bfloat16)
    B = torch.randn(G * rows, N, device=dev).to(torch.bfloat16)
    cdt = torch.float32 if out_f32 else torch.bfloat16
    Cm = torch.empty(G, M, N, device=dev, dtype=cdt)
    m, ar, b = i32([rows] * G), i32([g * rows for g in range(G)]), i32(list(range(G)))
    p = GemmProblem()
    p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_K, 0
    p.dtype_ab = _lib.MOE_DTYPE_BF16
    p.dtype_c = _lib.MOE_DTYPE_F32 if out_f32 else _lib.MOE_DTYPE_BF16
    p.groups, p.M, p.N, p.a_rows, p.num_b = G, M, N, G * rows, G
    p.m, p.a_row, p.b = m.data_ptr(), ar.data_ptr(), b.data_ptr()
    p.A, p.B, p.C = A.data_ptr(), B.data_ptr(), Cm.data_ptr()
    p.ldc = N
    return p, (A, B, Cm, m, ar, b), 2.0 * G * rows * M * N


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--rows", type=int, default=1024)
    ap.add_argument("--groups", type=int, default=64)
    ap.add_argument("--only", default="", help="comma-separated substrings of variant names")
    ap.add_argument("--json", action="store_true")
    ap.add_argument("--cublas", action="store_true",
                    help="also time torch.matmul (cuBLAS) on the dense equivalents")
    ap.add_argument("--shared-b", action="store_true", help="every group uses weight 0 (L2-resident)")
    ap.add_argument("--b-mod", type=int, default=0, help="group g uses weight g %% B_MOD")
    a = ap.parse_args()
    global SHARED_B, B_MOD
    SHARED_B = a.shared_b
    B_MOD = a.b_mod
    G, R, d, f = a.groups, a.rows, 1024, 4096
    variants = [
        ("ffn1 shape  K-major  bf16 STORE", lambda: ragged_m(G, R, f, d)),
        ("ffn1 shape  K-major  bf16 GELU ", lambda: ragged_m(G, R, f, d, epi=1)),
        ("ffn1 shape  K-major  f32  STORE", lambda: ragged_m(G, R, f, d, out_f32=True)),
        ("ffn2 shape  K-major  bf16 STORE", lambda: ragged_m(G, R, d, f)),
        ("dgrad2 shp  B MN     bf16 STORE", lambda: ragged_m(G, R, f, d, b_mn=True)),
        ("dgrad2 shp  B MN     bf16 DGELU", lambda: ragged_m(G, R, f, d, epi=2, b_mn=True)),
        ("dgrad2 shp  B MN     DGELU nocs", lambda: ragged_m(G, R, f, d, epi=2, b_mn=True, colsum=False)),
        ("dgrad1 shp  B MN     bf16 STORE", lambda: ragged_m(G, R, d, f, b_mn=True)),
        ("wgrad1 shp  MN/MN    f32  STORE", lambda: ragged_k(G, R, d, f)),
        ("wgrad2 shp  MN/MN    f32  STORE", lambda: ragged_k(G, R, f, d)),
    ]
    for name, mk in variants:
        if a.only and not any(o in name for o in a.only.split(",")):
            continue
        p, keep, flops = mk()
        ms = timed(lambda: grouped_gemm(p), a.reps)
        if a.json:
            import json
            print(json.dumps({"name": name.strip(), "us": ms * 1e3}), flush=True)
        else:
            print(f"{name}  {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TFLOP/s", flush=True)
        del keep
    if a.cublas:
        T = G * R
        for name, (M, N, K) in (("cuBLAS ffn1 dense", (T, f, d)), ("cuBLAS ffn2 dense", (T, d, f))):
            X = torch.randn(M, K, device=dev).to(torch.bfloat16)
            W = torch.randn(N, K, device=dev).to(torch.bfloat16)
            Y = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
            ms = timed(lambda: torch.matmul(X, W.t(), out=Y), a.reps)
            print(f"{name:32s}  {ms * 1e3:8.1f} us  {2.0 * M * N * K / ms / 1e9:7.1f} TFLOP/s", flush=True)
            del X, W, Y


if __name__ == "__main__":
    main()
