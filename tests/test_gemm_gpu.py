"""GPU: K5 grouped GEMM (tcgen05 bf16 and SIMT fp32) against a torch fp32
reference of the same op, for every layout/epilogue the layer uses, with
ragged/empty groups and row masking."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2205_10034_b200 import _lib, grouped_gemm  # noqa: E402
from paper_2205_10034_b200._lib import GemmProblem  # noqa: E402

dev = torch.device("cuda")


def gelu(h):
    return 0.5 * h * (1.0 + torch.erf(h * 0.7071067811865476))


def gelu_grad(h):
    return 0.5 * (1.0 + torch.erf(h * 0.7071067811865476)) + h * 0.3989422804014327 * torch.exp(-0.5 * h * h)


def i32(v):
    return torch.tensor(v, dtype=torch.int32, device=dev)


def ragged_m_case(dtype, b_mn, epi, N=512, K=256, groups=(200, 0, 128, 37, 300), bvec=(0, 1, 2, 1, 0),
                  Cs=320, bias=True, out_f32=False, colsum=False, gather=None):
    torch.manual_seed(0)
    G = len(groups)
    nb = max(bvec) + 1
    rows = G * Cs
    A = (torch.rand(rows, K, device=dev) * 2 - 1).to(dtype)
    W = (torch.rand(nb, N, K, device=dev) * 2 - 1) / K ** 0.5  # [b][N][K]
    Bmat = W.to(dtype)
    Bstore = Bmat.transpose(1, 2).contiguous() if b_mn else Bmat.contiguous()
    bias_t = torch.rand(nb, N, device=dev) - 0.5 if bias else None
    cdt = torch.float32 if (out_f32 or dtype == torch.float32) else dtype
    Cm = torch.full((rows, N), 7.0, device=dev, dtype=cdt)
    C2 = torch.full((rows, N), 7.0, device=dev, dtype=cdt)
    aux = (torch.rand(rows, N, device=dev) * 4 - 2).to(cdt)
    m, a_row, b = i32(list(groups)), i32([g * Cs for g in range(G)]), i32(list(bvec))
    p = GemmProblem()
    p.kind = _lib.MOE_GEMM_RAGGED_M
    p.epilogue = epi
    p.dtype_ab = _lib.MOE_DTYPE_BF16 if dtype == torch.bfloat16 else _lib.MOE_DTYPE_F32
    p.dtype_c = _lib.MOE_DTYPE_F32 if cdt == torch.float32 else _lib.MOE_DTYPE_BF16
    p.b_mn_major = 1 if b_mn else 0
    p.groups, p.N, p.K, p.a_rows, p.num_b = G, N, K, rows, nb
    p.m, p.a_row, p.c_row, p.b = m.data_ptr(), a_row.data_ptr(), a_row.data_ptr(), b.data_ptr()
    p.A, p.B, p.C = A.data_ptr(), Bstore.data_ptr(), Cm.data_ptr()
    p.C2 = C2.data_ptr()
    p.aux = aux.data_ptr()
    p.bias = bias_t.data_ptr() if bias_t is not None else None
    p.ldc = N
    cs = torch.full((nb, N), 5.0, device=dev) if colsum else None  # written, not accumulated
    if colsum:
        ws = torch.empty(G * ((max(groups) + 31) // 32) * N, device=dev)
        p.colsum = cs.data_ptr()
        p.colsum_ws, p.colsum_max_m = ws.data_ptr(), max(groups)
    if gather is not None:
        gsrc, gidx, gk = gather
        p.gather_src, p.gather_idx, p.gather_k = gsrc.data_ptr(), gidx.data_ptr(), gk
    grouped_gemm(p)
    torch.cuda.synchronize()
    # reference
    refC = torch.full((rows, N), 7.0, device=dev)
    refC2 = torch.full((rows, N), 7.0, device=dev)
    for g in range(G):
        r0, mm = g * Cs, groups[g]
        if mm == 0:
            continue
        acc = A[r0:r0 + mm].float() @ Bmat[bvec[g]].float().t()
        if epi == _lib.MOE_EPI_DGELU:
            acc = acc * aux[r0:r0 + mm].float()
        elif epi == _lib.MOE_EPI_GATHER_ADD:
            gsrc, gidx, gk = gather
            for i in range(gk):
                ix = gidx[r0:r0 + mm, i].long()
                ok = ix >= 0
                acc[ok] += gsrc[ix[ok]].float()
        elif bias_t is not None:
            acc = acc + bias_t[bvec[g]]
        if epi == _lib.MOE_EPI_GELU:
            refC2[r0:r0 + mm] = gelu_grad(acc)
            acc = gelu(acc)
        refC[r0:r0 + mm] = acc
    if colsum:
        ref_cs = torch.zeros(nb, N, device=dev)
        for g in range(G):
            r0, mm = g * Cs, groups[g]
            ref_cs[bvec[g]] += Cm[r0:r0 + mm].float().sum(0)  # sums of the stored values
        return Cm.float(), refC, cs, ref_cs
    return Cm.float(), refC, C2.float(), refC2


def assert_close(got, ref, rel):
    scale = ref[ref != 7.0].abs().max().clamp_min(1e-6) if (ref != 7.0).any() else torch.tensor(1.0)
    err = (got - ref).abs().max()
    assert err <= rel * scale, f"max err {err.item()} vs scale {scale.item()}"


@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("out_f32", [False, True])
def test_tc_ragged_m_store(b_mn, out_f32):
    got, ref, _, _ = ragged_m_case(torch.bfloat16, b_mn, _lib.MOE_EPI_STORE, out_f32=out_f32)
    assert_close(got, ref, 1e-2)
    assert (got[ref == 7.0] == 7.0).all()  # rows past m[g] untouched


def test_tc_ragged_m_gelu():
    got, ref, got2, ref2 = ragged_m_case(torch.bfloat16, False, _lib.MOE_EPI_GELU)
    assert_close(got, ref, 1e-2)
    assert_close(got2, ref2, 1e-2)


def test_tc_gelu_large_preactivations():
    """GeLU epilogue far into both tails (|h| up to ~40): gelu -> h / 0, gelu' ->
    1 / 0, no NaN (the epilogue's quartic is clamped; SURVEY Appendix A act = erf-GeLU)."""
    torch.manual_seed(5)
    M, N, K = 256, 512, 64
    A = (torch.rand(M, K, device=dev) * 2 - 1).to(torch.bfloat16)
    W = ((torch.rand(1, N, K, device=dev) * 2 - 1) * 4.0).to(torch.bfloat16)  # |h| up to ~50
    Cm = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
    C2 = torch.empty_like(Cm)
    m, a_row, b = i32([M]), i32([0]), i32([0])
    p = GemmProblem()
    p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_M, _lib.MOE_EPI_GELU
    p.dtype_ab = p.dtype_c = _lib.MOE_DTYPE_BF16
    p.groups, p.N, p.K, p.a_rows, p.num_b = 1, N, K, M, 1
    p.m, p.a_row, p.c_row, p.b = m.data_ptr(), a_row.data_ptr(), a_row.data_ptr(), b.data_ptr()
    p.A, p.B, p.C, p.C2 = A.data_ptr(), W.data_ptr(), Cm.data_ptr(), C2.data_ptr()
    p.ldc = N
    grouped_gemm(p)
    torch.cuda.synchronize()
    h = A.float() @ W[0].float().t()
    assert h.abs().max() > 20
    act, grad = Cm.float(), C2.float()
    assert torch.isfinite(act).all() and torch.isfinite(grad).all()
    assert ((act - gelu(h)).abs() <= 1e-2 * h.abs().clamp_min(1)).all()
    assert ((grad - gelu_grad(h)).abs() <= 1.5e-2).all()


def test_tc_ragged_m_dgelu_with_colsum():
    got, ref, cs, ref_cs = ragged_m_case(torch.bfloat16, True, _lib.MOE_EPI_DGELU, bias=False,
                                         colsum=True)
    assert_close(got, ref, 1e-2)
    assert_close(cs, ref_cs, 1e-4)


@pytest.mark.parametrize("T,k", [(1000, 2), (1000, 1), (20000, 1), (20000, 2)])
def test_tc_gather_add(T, k):
    """gate dgrad + gather (dx = dlogits wg + sum_i dXe[slot_i]); T = 20000 gives
    each SM pair several tiles (k = 1 prefetches the next tile's rows)."""
    torch.manual_seed(3)
    N, K = 512, 64
    gsrc = (torch.rand(3 * T, N, device=dev) * 2 - 1).to(torch.bfloat16)
    gidx = torch.randint(-1, 3 * T, (T, k), device=dev, dtype=torch.int32)
    got, ref, _, _ = ragged_m_case(torch.bfloat16, True, _lib.MOE_EPI_GATHER_ADD, N=N, K=K,
                                   groups=(T,), bvec=(0,), Cs=T, bias=False,
                                   gather=(gsrc, gidx, k))
    assert_close(got, ref, 1e-2)


@pytest.mark.parametrize("dtype", [torch.float32])
def test_simt_gather_add_and_colsum(dtype):
    torch.manual_seed(4)
    T, N, K, k = 300, 96, 32, 2
    gsrc = torch.rand(500, N, device=dev) * 2 - 1
    gidx = torch.randint(-1, 500, (T, k), device=dev, dtype=torch.int32)
    got, ref, _, _ = ragged_m_case(dtype, True, _lib.MOE_EPI_GATHER_ADD, N=N, K=K, groups=(T,),
                                   bvec=(0,), Cs=T, bias=False, gather=(gsrc, gidx, k))
    assert_close(got, ref, 2e-6)
    got, ref, cs, ref_cs = ragged_m_case(dtype, True, _lib.MOE_EPI_DGELU, N=N, K=K, bias=False,
                                         colsum=True)
    assert_close(got, ref, 2e-6)
    assert_close(cs, ref_cs, 2e-6)


def test_tc_small_n_masked():
    """gate-logits shape: N = 32 < BN = 64, K-major B, fp32 out."""
    got, ref, _, _ = ragged_m_case(torch.bfloat16, False, _lib.MOE_EPI_STORE, N=32, K=128,
                                   groups=(1000,), bvec=(0,), Cs=1000, out_f32=True)
    assert_close(got, ref, 1e-2)


def test_tc_large_k():
    got, ref, _, _ = ragged_m_case(torch.bfloat16, False, _lib.MOE_EPI_STORE, N=256, K=2048,
                                   groups=(129, 255), bvec=(0, 1), Cs=256)
    assert_close(got, ref, 1e-2)


@pytest.mark.parametrize("b_mn", [False, True])
@pytest.mark.parametrize("epi", [0, 1, 2])
def test_simt_ragged_m(b_mn, epi):
    if epi == 1 and b_mn:
        pytest.skip("layer uses GELU with K-major B only")
    got, ref, got2, ref2 = ragged_m_case(torch.float32, b_mn, epi, N=192, K=96,
                                         bias=(epi != 2))
    assert_close(got, ref, 2e-6)
    if epi == 1:
        assert_close(got2, ref2, 2e-6)


def ragged_k_case(dtype, atomic, M=256, N=512, groups=(100, 0, 64, 300, 17), bvec=(0, 0, 1, 1, 2),
                  Cs=320, transpose=False):
    torch.manual_seed(1)
    G = len(groups)
    nb = max(bvec) + 1
    rows = G * Cs
    A = (torch.rand(rows, M, device=dev) * 2 - 1).to(dtype)
    B = (torch.rand(rows, N, device=dev) * 2 - 1).to(dtype)
    for g in range(G):  # zero pad rows (the layer guarantees this up to 64)
        A[g * Cs + groups[g]:(g + 1) * Cs] = 0
    if atomic:
        out = torch.zeros(nb * (N if transpose else M), M if transpose else N, device=dev)
    else:
        out = torch.full((nb * M, N), 7.0, device=dev)
    m, a_row, b = i32(list(groups)), i32([g * Cs for g in range(G)]), i32(list(bvec))
    p = GemmProblem()
    p.kind = _lib.MOE_GEMM_RAGGED_K
    p.epilogue = _lib.MOE_EPI_ATOMIC_ADD if atomic else _lib.MOE_EPI_STORE
    p.dtype_ab = _lib.MOE_DTYPE_BF16 if dtype == torch.bfloat16 else _lib.MOE_DTYPE_F32
    p.dtype_c = _lib.MOE_DTYPE_F32
    p.transpose_c = 1 if transpose else 0
    p.groups, p.M, p.N, p.a_rows, p.num_b = G, M, N, rows, nb
    p.m, p.a_row, p.b = m.data_ptr(), a_row.data_ptr(), b.data_ptr()
    p.A, p.B, p.C = A.data_ptr(), B.data_ptr(), out.data_ptr()
    p.ldc = M if transpose else N
    grouped_gemm(p)
    torch.cuda.synchronize()
    ref = torch.zeros(nb, M, N, device=dev)
    for g in range(G):
        r0, mm = g * Cs, groups[g]
        ref[bvec[g]] += A[r0:r0 + mm].float().t() @ B[r0:r0 + mm].float()
    if transpose:
        ref = ref.transpose(1, 2).reshape(nb * N, M)
    else:
        ref = ref.reshape(nb * M, N)
    return out, ref


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_ragged_k_store(dtype):
    got, ref = ragged_k_case(dtype, atomic=False)
    assert_close(got, ref, 1e-2 if dtype == torch.bfloat16 else 2e-6)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_ragged_k_atomic_transposed(dtype):
    """gate weight-gradient shape: N = E = 64 (BN=64 path), split-K groups, C^T."""
    got, ref = ragged_k_case(dtype, atomic=True, M=256, N=64, groups=(64, 64, 40, 128),
                             bvec=(0, 0, 0, 0), Cs=128, transpose=True)
    assert_close(got, ref, 1e-2 if dtype == torch.bfloat16 else 2e-6)


def test_tc_many_groups_persistent_schedule():
    """More tiles than SMs, many groups, so the persistent scheduler wraps."""
    groups = tuple((i * 37) % 300 for i in range(64))
    bvec = tuple(i % 8 for i in range(64))
    got, ref, _, _ = ragged_m_case(torch.bfloat16, False, _lib.MOE_EPI_STORE, N=1024, K=128,
                                   groups=groups, bvec=bvec, Cs=320)
    assert_close(got, ref, 1e-2)


def _split3(x):
    from paper_2205_10034_b200._lib import call
    x = x.contiguous()
    out = torch.empty(3 * x.numel(), dtype=torch.bfloat16, device=x.device)
    call("moe_split_f32_bf16x3", x.data_ptr(), x.numel(), out.data_ptr(),
         torch.cuda.current_stream().cuda_stream)
    return out


def test_split_f32_planes_exact():
    x = (torch.randn(4096, device=dev) * torch.logspace(-20, 20, 4096, device=dev)).float()
    p = _split3(x).view(3, -1).double()
    assert torch.equal(p.sum(0), x.double())


@pytest.mark.parametrize("b_mn", [False, True])
def test_split_f32_ragged_m_chunked(b_mn):
    """fp32 GEMM as six split-bf16 plane products on tcgen05, K chunks of 512
    summed in fp32: ~fp32 accuracy (the c1 path) vs an fp64 reference."""
    G, rows, N, K = 3, 300, 256, 1024
    torch.manual_seed(1)
    A = torch.randn(G * rows, K, device=dev)
    W = torch.randn(G, N, K, device=dev) / K ** 0.5
    Bst = W.transpose(1, 2).contiguous() if b_mn else W.contiguous()
    A3, B3 = _split3(A), _split3(Bst)
    m, ar, b = i32([rows, 0, 171]), i32([g * rows for g in range(G)]), i32([0, 1, 2])
    parts = torch.zeros(2, G * rows, N, device=dev)
    for c in range(2):
        p = GemmProblem()
        p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_M, _lib.MOE_EPI_STORE
        p.dtype_ab, p.dtype_c = _lib.MOE_DTYPE_BF16, _lib.MOE_DTYPE_F32
        p.b_mn_major = 1 if b_mn else 0
        p.groups, p.N, p.K, p.a_rows, p.num_b = G, N, K, G * rows, G
        p.m, p.a_row, p.c_row, p.b = m.data_ptr(), ar.data_ptr(), ar.data_ptr(), b.data_ptr()
        p.A, p.B, p.C = A3.data_ptr(), B3.data_ptr(), parts[c].data_ptr()
        p.ldc, p.split_terms, p.k_begin, p.k_len = N, 6, 512 * c, 512
        grouped_gemm(p)
    torch.cuda.synchronize()
    got = parts.sum(0).double()
    for g, mm in enumerate([rows, 0, 171]):
        if mm == 0:
            continue
        r0 = g * rows
        ref = A[r0:r0 + mm].double() @ W[g].double().t()
        err = (got[r0:r0 + mm] - ref).abs().max() / ref.abs().max()
        assert err < 2e-6, (g, err.item())


def test_split_f32_ragged_k():
    G, rows, M, N = 2, 448, 256, 128
    torch.manual_seed(2)
    A = torch.randn(G * rows, M, device=dev)
    B = torch.randn(G * rows, N, device=dev)
    m = [rows, 300]
    for g, mm in enumerate(m):  # rows past m up to the next 64 are zero
        A[g * rows + mm:(g + 1) * rows] = 0
        B[g * rows + mm:(g + 1) * rows] = 0
    A3, B3 = _split3(A), _split3(B)
    C = torch.zeros(G, M, N, device=dev)
    p = GemmProblem()
    p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_K, _lib.MOE_EPI_STORE
    p.dtype_ab, p.dtype_c = _lib.MOE_DTYPE_BF16, _lib.MOE_DTYPE_F32
    p.groups, p.M, p.N, p.a_rows, p.num_b = G, M, N, G * rows, G
    mt, at, bt = i32(m), i32([0, rows]), i32([0, 1])
    p.m, p.a_row, p.b = mt.data_ptr(), at.data_ptr(), bt.data_ptr()
    p.A, p.B, p.C, p.ldc, p.split_terms = A3.data_ptr(), B3.data_ptr(), C.data_ptr(), N, 6
    grouped_gemm(p)
    torch.cuda.synchronize()
    for g in range(G):
        ref = A[g * rows:(g + 1) * rows].double().t() @ B[g * rows:(g + 1) * rows].double()
        err = (C[g].double() - ref).abs().max() / ref.abs().max()
        assert err < 2e-6, (g, err.item())


_MC_SCRIPT = r"""
import sys, torch
sys.path.insert(0, sys.argv[1])
from paper_2205_10034_b200 import _lib, grouped_gemm
from paper_2205_10034_b200._lib import GemmProblem
dev = torch.device("cuda")
torch.manual_seed(1)
groups, Cs, N, K = (1030, 0, 37, 700, 256, 129), 1088, 1024, 512
G = len(groups)
A = (torch.rand(G * Cs, K, device=dev) * 2 - 1).to(torch.bfloat16)
B = ((torch.rand(G, N, K, device=dev) * 2 - 1) / K ** 0.5).to(torch.bfloat16)
out = []
for b_mn in (0, 1):
    Bs = B.transpose(1, 2).contiguous() if b_mn else B
    C = torch.zeros(G * Cs, N, device=dev, dtype=torch.bfloat16)
    i32 = lambda v: torch.tensor(v, dtype=torch.int32, device=dev)
    m, ar, b = i32(list(groups)), i32([g * Cs for g in range(G)]), i32(list(range(G)))
    p = GemmProblem()
    p.kind, p.epilogue = _lib.MOE_GEMM_RAGGED_M, _lib.MOE_EPI_STORE
    p.dtype_ab = p.dtype_c = _lib.MOE_DTYPE_BF16
    p.b_mn_major = b_mn
    p.groups, p.N, p.K, p.a_rows, p.num_b = G, N, K, G * Cs, G
    p.m, p.a_row, p.c_row, p.b = m.data_ptr(), ar.data_ptr(), ar.data_ptr(), b.data_ptr()
    p.A, p.B, p.C, p.ldc = A.data_ptr(), Bs.data_ptr(), C.data_ptr(), N
    grouped_gemm(p)
    torch.cuda.synchronize()
    out.append(C.cpu())
torch.save(out, sys.argv[2])
"""


def test_multicast_clusters_bitwise_equal_pair_mode(tmp_path):
    """The 2-pair multicast clusters (bf16 STORE GEMMs, preferred cluster
    size 4) change only where the A rows come from: results are bitwise the
    pair-mode ones (MOE_GEMM_MC=0), ragged groups, tails and empty groups
    included, both B layouts."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for mc in ("0", "1"):
        f = tmp_path / f"mc{mc}.pt"
        env = dict(os.environ, MOE_GEMM_MC=mc)
        subprocess.run([sys.executable, "-c", _MC_SCRIPT, repo, str(f)], env=env, check=True,
                       timeout=300)
        outs.append(torch.load(f))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    assert outs[1][0].abs().sum() > 0
