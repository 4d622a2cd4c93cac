// K5 (fp32 path, config c1) — grouped GEMM on the FP32 FMA pipe.
//
// Config c1 requires fp32 results within 1e-5 of an fp64 oracle, which rules
// out TF32 tensor cores; this kernel keeps fp32 operands and fp32 FFMA
// accumulation with the same group tables and epilogues as the tcgen05 kernel
// (gemm_tc.cu), so the layer orchestration is dtype-agnostic.
#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace simt {

constexpr int BM = 64, BN = 64, BK = 16, THREADS = 256, MAX_GROUPS = 1024;

struct Args {
  int kind, epi, groups, M, N, K, b_mn, transpose_c;
  const int *gm, *ga, *gc, *gb;
  const float *A, *B;
  float *C, *C2;
  const float* aux;
  const float* bias;
  long long lda, ldb, ldc;
  long long b_rows;
  float* colsum;
  const float* gsrc;
  const int* gidx;
  int gk;
};

__global__ void __launch_bounds__(THREADS) simt_gemm_kernel(const Args a) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  __shared__ int tab[MAX_GROUPS + 1];
  __shared__ int cnt[MAX_GROUPS];
  const int tid = threadIdx.x;
  const int G = a.groups;
  const int nbn = (a.N + BN - 1) / BN;
  const int nbm_k = (a.M + BM - 1) / BM;  // RAGGED_K tiles along M

  for (int g = tid; g < G; g += THREADS) {
    if (a.kind == 0) {
      cnt[g] = ((a.gm[g] + BM - 1) / BM) * nbn;
    } else {
      const bool start = a.epi == MOE_EPI_ATOMIC_ADD || g == 0 || a.gb[g] != a.gb[g - 1];
      cnt[g] = start ? 1 : 0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (a.kind == 0) {
      int run = 0;
      for (int g = 0; g < G; ++g) { tab[g] = run; run += cnt[g]; }
      tab[G] = run;
    } else {
      int ns = 0;
      for (int g = 0; g < G; ++g)
        if (cnt[g]) tab[ns++] = g;
      tab[ns] = G;
      cnt[0] = ns;  // reuse: number of segments
    }
  }
  __syncthreads();
  const int total = a.kind == 0 ? tab[G] : cnt[0] * nbm_k * nbn;

  const int tx = tid % 16, ty = tid / 16;
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    int g, mb, nb;
    if (a.kind == 0) {
      int lo = 0, hi = G;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (tab[mid] <= w) lo = mid; else hi = mid;
      }
      g = lo;
      const int local = w - tab[g];
      mb = local / nbn;
      nb = local % nbn;
    } else {
      const int per = nbm_k * nbn;
      g = w / per;
      mb = (w % per) / nbn;
      nb = (w % per) % nbn;
    }
    float acc[4][4] = {};
    // K iteration: RAGGED_M -> one range [0,K) on row base ga[g]+mb*BM;
    // RAGGED_K -> rows of every group of segment g.
    const int q0 = a.kind == 0 ? g : tab[g];
    const int q1 = a.kind == 0 ? g + 1 : tab[g + 1];
    for (int q = q0; q < q1; ++q) {
      const int klen = a.kind == 0 ? a.K : a.gm[q];
      const int mrows = a.kind == 0 ? a.gm[q] : a.M;
      const long long r0 = a.ga[q];
      for (int k0 = 0; k0 < klen; k0 += BK) {
        for (int i = tid; i < BM * BK; i += THREADS) {
          int mm, kk;
          float v = 0.f;
          if (a.kind == 0) {
            mm = i / BK; kk = i % BK;
            const int m = mb * BM + mm, k = k0 + kk;
            if (m < mrows && k < klen) v = a.A[(r0 + m) * a.lda + k];
          } else {
            kk = i / BM; mm = i % BM;
            const int m = mb * BM + mm, k = k0 + kk;
            if (m < mrows && k < klen) v = a.A[(r0 + k) * a.lda + m];
          }
          As[kk][mm] = v;
        }
        for (int i = tid; i < BN * BK; i += THREADS) {
          int nn, kk;
          float v = 0.f;
          if (a.kind == 0 && !a.b_mn) {
            nn = i / BK; kk = i % BK;
            const int n = nb * BN + nn, k = k0 + kk;
            const long long br = (long long)a.gb[q] * a.N + n;
            if (n < a.N && k < klen && br < a.b_rows) v = a.B[br * a.ldb + k];
          } else if (a.kind == 0) {
            kk = i / BN; nn = i % BN;
            const int n = nb * BN + nn, k = k0 + kk;
            const long long br = (long long)a.gb[q] * a.K + k;
            if (n < a.N && k < klen && br < a.b_rows) v = a.B[br * a.ldb + n];
          } else {
            kk = i / BN; nn = i % BN;
            const int n = nb * BN + nn, k = k0 + kk;
            if (n < a.N && k < klen) v = a.B[(r0 + k) * a.ldb + n];
          }
          Bs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          float av[4], bv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
          for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
      }
    }
    // epilogue
    const int bidx = a.kind == 0 ? a.gb[g] : a.gb[tab[g]];
    for (int i = 0; i < 4; ++i) {
      const int m = mb * BM + ty * 4 + i;
      long long orow;
      if (a.kind == 0) {
        if (m >= a.gm[g]) continue;
        orow = (long long)a.gc[g] + m;
      } else {
        if (m >= a.M) continue;
        orow = (long long)bidx * a.M + m;
      }
      for (int j = 0; j < 4; ++j) {
        const int n = nb * BN + tx * 4 + j;
        if (n >= a.N) continue;
        float v = acc[i][j];
        if (a.epi == MOE_EPI_ATOMIC_ADD) {
          const long long idx = a.transpose_c ? (long long)n * a.ldc + orow : orow * a.ldc + n;
          atomicAdd(a.C + idx, v);
          continue;
        }
        if (a.bias && a.epi != MOE_EPI_DGELU && a.epi != MOE_EPI_GATHER_ADD)
          v += a.bias[(long long)bidx * a.N + n];
        const long long idx = orow * a.ldc + n;
        if (a.epi == MOE_EPI_GELU) {
          a.C2[idx] = gelu_grad_f(v);  // stored derivative gelu'(h)
          v = gelu_f(v);
        } else if (a.epi == MOE_EPI_DGELU) {
          v *= a.aux[idx];
          if (a.colsum) atomicAdd(a.colsum + (long long)bidx * a.N + n, v);
        } else if (a.epi == MOE_EPI_GATHER_ADD) {
          for (int i = 0; i < a.gk; ++i) {
            const int s = a.gidx[orow * a.gk + i];
            if (s >= 0) v += a.gsrc[(long long)s * a.N + n];
          }
        }
        a.C[idx] = v;
      }
    }
  }
}

}  // namespace simt

void simt_grouped_gemm(const moe_gemm_problem_t& p, cudaStream_t st) {
  using namespace simt;
  arg_check(p.groups >= 1 && p.groups <= MAX_GROUPS, "gemm.groups: must be in [1, 1024]");
  arg_check(p.dtype_ab == MOE_DTYPE_F32 && p.dtype_c == MOE_DTYPE_F32,
            "gemm.dtype: SIMT path is fp32 in / fp32 out");
  Args a;
  a.kind = p.kind;
  a.epi = p.epilogue;
  a.groups = (int)p.groups;
  a.M = (int)p.M;
  a.N = (int)p.N;
  a.K = (int)p.K;
  a.b_mn = p.b_mn_major;
  a.transpose_c = p.transpose_c;
  a.gm = p.m;
  a.ga = p.a_row;
  a.gc = p.c_row;
  a.gb = p.b;
  a.A = static_cast<const float*>(p.A);
  a.B = static_cast<const float*>(p.B);
  a.C = static_cast<float*>(p.C);
  a.C2 = static_cast<float*>(p.C2);
  a.aux = static_cast<const float*>(p.aux);
  a.bias = p.bias;
  a.colsum = p.colsum;
  a.gsrc = static_cast<const float*>(p.gather_src);
  a.gidx = p.gather_idx;
  a.gk = (int)p.gather_k;
  a.ldc = (long long)p.ldc;
  if (p.kind == MOE_GEMM_RAGGED_M) {
    a.lda = p.lda ? p.lda : p.K;
    a.ldb = p.ldb ? p.ldb : (p.b_mn_major ? p.N : p.K);
    a.b_rows = p.b_rows ? (long long)p.b_rows
                        : (long long)p.num_b * (p.b_mn_major ? p.K : p.N);
  } else {
    a.b_rows = 0;
    a.lda = p.lda ? p.lda : p.M;
    a.ldb = p.ldb ? p.ldb : p.N;
  }
  const int grid = num_sms() * 4;
  simt_gemm_kernel<<<grid, THREADS, 0, st>>>(a);
  MOE_LAUNCH_CHECK("simt_gemm_kernel");
  count_launch();
}

}  // namespace moe
