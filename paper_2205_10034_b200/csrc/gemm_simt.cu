// K5 (fp32 path, config c1) — grouped GEMM on the FP32 FMA pipe.
//
// Config c1 requires fp32 results within 1e-5 of an fp64 oracle, which rules
// out TF32 tensor cores; this kernel keeps fp32 operands and fp32 FFMA
// accumulation with the same group tables and epilogues as the tcgen05 kernel
// (gemm_tc.cu), so the layer orchestration is dtype-agnostic.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace simt {

// 128 x 128 tiles, 16-deep K slices, 256 threads each owning an 8 x 8 block
// of C (rows ty*4 + {0..3} and 64 + ty*4 + {0..3}, same for columns with tx):
// conflict-free 16-byte shared loads, packed FFMA2 (two fp32 FMAs per
// instruction, exact fp32 rounding), next K slice prefetched into registers
// while the current one is multiplied.
constexpr int BM = 128, BN = 128, BK = 16, THREADS = 256, MAX_GROUPS = 1024;
constexpr int PAD = 4;
#ifndef SIMT_MINB
#define SIMT_MINB 2  // 2 CTAs per SM: A/B on c1 +2.7% over 1 (small epilogue-only spills)
#endif

struct Args {
  int kind, epi, groups, M, N, K, b_mn, transpose_c;
  const int *gm, *ga, *gc, *gb;
  const float *A, *B;
  float *C, *C2;
  const float* aux;
  const float* bias;
  long long lda, ldb, ldc;
  long long b_rows;
  float* colsum;  // DGELU: per-tile partials [groups][cs_maxch][N] (reduced by seg_colsum)
  int cs_maxch;
  const float* gsrc;
  const int* gidx;
  int gk;
};

// One K slice of the A / B tile in registers: 2 float4 per thread each.
struct Slice {
  float4 a[2], b[2];
};

// Specialised per (kind, B layout, epilogue) so the bounds / layout branches
// fold at compile time (fewer live registers in the K loop).
// BNT = 128 (8 x 8 per thread) or 64 (8 x 4 per thread: twice the tiles, for
// the narrow GEMMs whose 128 x 128 tiles leave SMs idle in the last wave).
template <int KIND, int BMN, int EPI, int BNT>
__global__ void __launch_bounds__(THREADS, SIMT_MINB) simt_gemm_kernel(const Args a) {
  pdl_wait();
  pdl_trigger();
  constexpr int BN = BNT, NH = BNT / 64;  // column halves of 64 per thread tile
  constexpr int C4 = BN / 4;              // float4 per B row of the slice ([k][n])
  __shared__ __align__(16) float As[2][BK][BM + PAD];
  __shared__ __align__(16) float Bs[2][BK][BN + PAD];
  __shared__ int tab[MAX_GROUPS + 1];
  __shared__ int cnt[MAX_GROUPS];
  const int tid = threadIdx.x;
  const int G = a.groups;
  const int nbn = (a.N + BN - 1) / BN;
  const int nbm_k = (a.M + BM - 1) / BM;  // RAGGED_K tiles along M

  for (int g = tid; g < G; g += THREADS) {
    if (KIND == 0) {
      cnt[g] = ((a.gm[g] + BM - 1) / BM) * nbn;
    } else {
      const bool start = EPI == MOE_EPI_ATOMIC_ADD || g == 0 || a.gb[g] != a.gb[g - 1];
      cnt[g] = start ? 1 : 0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (KIND == 0) {
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
  const int total = KIND == 0 ? tab[G] : cnt[0] * nbm_k * nbn;
  // vector (16-byte) global loads need 4-element aligned rows
  const bool a_vec = (a.lda % 4) == 0 && (reinterpret_cast<uintptr_t>(a.A) & 15) == 0;
  const bool b_vec = (a.ldb % 4) == 0 && (reinterpret_cast<uintptr_t>(a.B) & 15) == 0;
  auto al16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool c_vec = (a.ldc % 4) == 0 && (a.N % 4) == 0 && al16(a.C) && al16(a.C2) &&
                     al16(a.aux) && al16(a.bias) && al16(a.gsrc);

  const int tx = tid % 16, ty = tid / 16;
  for (int w = blockIdx.x; w < total; w += gridDim.x) {
    int g, mb, nb;
    if (KIND == 0) {
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
    float2 acc[8][2 * NH];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 2 * NH; ++j) acc[i][j] = make_float2(0.f, 0.f);
    // K iteration: RAGGED_M -> one range [0,K) on row base ga[g]+mb*BM;
    // RAGGED_K -> rows of every group of segment g.
    const int q0 = KIND == 0 ? g : tab[g];
    const int q1 = KIND == 0 ? g + 1 : tab[g + 1];
    for (int q = q0; q < q1; ++q) {
      const int klen = KIND == 0 ? a.K : a.gm[q];
      const int mrows = KIND == 0 ? a.gm[q] : a.M;
      const long long r0 = a.ga[q];
      const long long bbase = KIND == 0 ? (long long)a.gb[q] * (BMN ? a.K : a.N) : r0;
      // element (m, k) of A / (n, k) of B with bounds (0 outside)
      auto ldA = [&](int m, int k) -> float {
        if (m >= mrows || k >= klen) return 0.f;
        return KIND == 0 ? a.A[(r0 + m) * a.lda + k] : a.A[(r0 + k) * a.lda + m];
      };
      auto ldB = [&](int n, int k) -> float {
        if (n >= a.N || k >= klen) return 0.f;
        if (KIND == 0 && !BMN) {
          const long long br = bbase + n;
          return br < a.b_rows ? a.B[br * a.ldb + k] : 0.f;
        }
        if (KIND == 0) {
          const long long br = bbase + k;
          return br < a.b_rows ? a.B[br * a.ldb + n] : 0.f;
        }
        return a.B[(bbase + k) * a.ldb + n];
      };
      // thread -> float4 of the slice: "contiguous-K" layouts (A of RAGGED_M,
      // B K-major) take 4 k of one row; "contiguous-M/N" layouts take 4 rows
      // of one k.  Index f = tid + 256 i, i = 0, 1.
      auto fetch = [&](int k0, Slice& sl) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int f = tid + THREADS * i;
          if (KIND == 0) {  // A: [m][k]
            const int mm = f >> 2, k = k0 + (f & 3) * 4, m = mb * BM + mm;
            if (a_vec && m < mrows && k + 3 < klen)
              sl.a[i] = __ldg(reinterpret_cast<const float4*>(a.A + (r0 + m) * a.lda + k));
            else
              sl.a[i] = make_float4(ldA(m, k), ldA(m, k + 1), ldA(m, k + 2), ldA(m, k + 3));
          } else {  // A: [k][m]
            const int kk = f >> 5, m = mb * BM + (f & 31) * 4, k = k0 + kk;
            if (a_vec && m + 3 < mrows && k < klen)
              sl.a[i] = __ldg(reinterpret_cast<const float4*>(a.A + (r0 + k) * a.lda + m));
            else
              sl.a[i] = make_float4(ldA(m, k), ldA(m + 1, k), ldA(m + 2, k), ldA(m + 3, k));
          }
          if (i >= NH) continue;  // B slice: BN * BK / 4 float4 = NH per thread
          if (KIND == 0 && !BMN) {  // B: [n][k]
            const int nn = f >> 2, k = k0 + (f & 3) * 4, n = nb * BN + nn;
            const long long br = bbase + n;
            if (b_vec && n < a.N && k + 3 < klen && br < a.b_rows)
              sl.b[i] = __ldg(reinterpret_cast<const float4*>(a.B + br * a.ldb + k));
            else
              sl.b[i] = make_float4(ldB(n, k), ldB(n, k + 1), ldB(n, k + 2), ldB(n, k + 3));
          } else {  // B: [k][n]
            const int kk = f / C4, n = nb * BN + (f % C4) * 4, k = k0 + kk;
            const long long br = bbase + k;
            if (b_vec && n + 3 < a.N && k < klen && (KIND != 0 || br < a.b_rows))
              sl.b[i] = __ldg(reinterpret_cast<const float4*>(a.B + br * a.ldb + n));
            else
              sl.b[i] = make_float4(ldB(n, k), ldB(n + 1, k), ldB(n + 2, k), ldB(n + 3, k));
          }
        }
      };
      auto stash = [&](int buf, const Slice& sl) {
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int f = tid + THREADS * i;
          if (KIND == 0) {
            const int mm = f >> 2, kq = (f & 3) * 4;
            As[buf][kq][mm] = sl.a[i].x;
            As[buf][kq + 1][mm] = sl.a[i].y;
            As[buf][kq + 2][mm] = sl.a[i].z;
            As[buf][kq + 3][mm] = sl.a[i].w;
          } else {
            *reinterpret_cast<float4*>(&As[buf][f >> 5][(f & 31) * 4]) = sl.a[i];
          }
          if (i >= NH) continue;
          if (KIND == 0 && !BMN) {
            const int nn = f >> 2, kq = (f & 3) * 4;
            Bs[buf][kq][nn] = sl.b[i].x;
            Bs[buf][kq + 1][nn] = sl.b[i].y;
            Bs[buf][kq + 2][nn] = sl.b[i].z;
            Bs[buf][kq + 3][nn] = sl.b[i].w;
          } else {
            *reinterpret_cast<float4*>(&Bs[buf][f / C4][(f % C4) * 4]) = sl.b[i];
          }
        }
      };
      Slice sl;
      fetch(0, sl);
      __syncthreads();  // previous tile's readers are done with both buffers
      stash(0, sl);
      __syncthreads();
      int buf = 0;
      for (int k0 = 0; k0 < klen; k0 += BK) {
        const bool more = k0 + BK < klen;
        if (more) fetch(k0 + BK, sl);  // in flight during the FMAs below
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
          const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
          const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
          float2 bv[2 * NH];
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 * h + tx * 4]);
            bv[2 * h] = make_float2(b.x, b.y);
            bv[2 * h + 1] = make_float2(b.z, b.w);
          }
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 2 * NH; ++j)
              acc[i][j] = __ffma2_rn(make_float2(av[i], av[i]), bv[j], acc[i][j]);
        }
        if (more) {
          stash(buf ^ 1, sl);
          __syncthreads();
          buf ^= 1;
        }
      }
      __syncthreads();
    }
    // epilogue: thread rows ty*4 + {0..3}, 64 + ty*4 + {0..3}; columns
    // nb*BN + h*64 + tx*4 + {0..3} (h = 0, 1) -- four contiguous columns, so
    // C / C2 / aux / bias / gathered rows move as float4 when aligned.
    const int bidx = KIND == 0 ? a.gb[g] : a.gb[tab[g]];
    float csum[4 * NH];  // DGELU: this thread's column sums
#pragma unroll
    for (int j = 0; j < 4 * NH; ++j) csum[j] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int m = mb * BM + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
      long long orow;
      if (KIND == 0) {
        if (m >= a.gm[g]) continue;
        orow = (long long)a.gc[g] + m;
      } else {
        if (m >= a.M) continue;
        orow = (long long)bidx * a.M + m;
      }
#pragma unroll
      for (int h = 0; h < NH; ++h) {
        const int n0 = nb * BN + h * 64 + tx * 4;
        if (n0 >= a.N) continue;
        float v[4] = {acc[i][2 * h].x, acc[i][2 * h].y, acc[i][2 * h + 1].x, acc[i][2 * h + 1].y};
        if (EPI == MOE_EPI_ATOMIC_ADD) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int n = n0 + c;
            if (n >= a.N) continue;
            const long long idx = a.transpose_c ? (long long)n * a.ldc + orow : orow * a.ldc + n;
            atomicAdd(a.C + idx, v[c]);
          }
          continue;
        }
        const long long idx = orow * a.ldc + n0;
        if (c_vec && n0 + 3 < a.N) {
          if (a.bias && EPI != MOE_EPI_DGELU && EPI != MOE_EPI_GATHER_ADD) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(a.bias + (long long)bidx * a.N + n0));
            v[0] += b.x; v[1] += b.y; v[2] += b.z; v[3] += b.w;
          }
          if (EPI == MOE_EPI_GELU) {
            float gr[4];
#pragma unroll
            for (int c = 0; c < 4; ++c) gelu_and_grad_f(v[c], v[c], gr[c]);
            *reinterpret_cast<float4*>(a.C2 + idx) = make_float4(gr[0], gr[1], gr[2], gr[3]);
          } else if (EPI == MOE_EPI_DGELU) {
            const float4 x4 = __ldg(reinterpret_cast<const float4*>(a.aux + idx));
            v[0] *= x4.x; v[1] *= x4.y; v[2] *= x4.z; v[3] *= x4.w;
#pragma unroll
            for (int c = 0; c < 4; ++c) csum[h * 4 + c] += v[c];
          } else if (EPI == MOE_EPI_GATHER_ADD) {
            for (int r = 0; r < a.gk; ++r) {
              const int sidx = a.gidx[orow * a.gk + r];
              if (sidx < 0) continue;
              const float4 x4 = __ldg(reinterpret_cast<const float4*>(a.gsrc + (long long)sidx * a.N + n0));
              v[0] += x4.x; v[1] += x4.y; v[2] += x4.z; v[3] += x4.w;
            }
          }
          *reinterpret_cast<float4*>(a.C + idx) = make_float4(v[0], v[1], v[2], v[3]);
          continue;
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int n = n0 + c;
          if (n >= a.N) continue;
          float x = v[c];
          if (a.bias && EPI != MOE_EPI_DGELU && EPI != MOE_EPI_GATHER_ADD)
            x += a.bias[(long long)bidx * a.N + n];
          if (EPI == MOE_EPI_GELU) {
            float gr;
            gelu_and_grad_f(x, x, gr);
            a.C2[idx + c] = gr;  // stored derivative gelu'(h)
          } else if (EPI == MOE_EPI_DGELU) {
            x *= a.aux[idx + c];
            csum[h * 4 + c] += x;
          } else if (EPI == MOE_EPI_GATHER_ADD) {
            for (int r = 0; r < a.gk; ++r) {
              const int sidx = a.gidx[orow * a.gk + r];
              if (sidx >= 0) x += a.gsrc[(long long)sidx * a.N + n];
            }
          }
          a.C[idx + c] = x;
        }
      }
    }
    if (EPI == MOE_EPI_DGELU && a.colsum) {
      // db1: column sums of the tile -- the two ty of a warp via shuffle, the
      // eight warps through shared memory, then one atomic per column and tile
      // (instead of one per element)
#pragma unroll
      for (int j = 0; j < 4 * NH; ++j) csum[j] += __shfl_xor_sync(0xffffffffu, csum[j], 16);
      float* red = &As[0][0][0];  // [8 warps][BN], the K-loop buffers are free here
      const int wp = tid >> 5;
      if ((tid & 16) == 0) {
#pragma unroll
        for (int j = 0; j < 4 * NH; ++j) red[wp * BN + (j >> 2) * 64 + tx * 4 + (j & 3)] = csum[j];
      }
      __syncthreads();
      if (tid < BN) {
        float s = 0.f;
#pragma unroll
        for (int w8 = 0; w8 < THREADS / 32; ++w8) s += red[w8 * BN + tid];
        const int n = nb * BN + tid;
        // the tile's 128-row block of group g owns this partial row
        if (n < a.N) a.colsum[((long long)g * a.cs_maxch + mb) * a.N + n] = s;
      }
      __syncthreads();  // red aliases As: next tile's stash waits for the readers
    }
  }
}

}  // namespace simt

namespace simt {
// Host-side tile-count estimate (row counts live on the device: the A row
// capacity stands in for them). MOE_SIMT_BN64=0/1 forces a width (A/B runs).
bool simt_use_bn64(const moe_gemm_problem_t& p) {
  static const char* env = std::getenv("MOE_SIMT_BN64");
  if (env && env[0] == '0') return false;
  if (env && env[0] == '1') return true;
  // measured on c1 (A/B): the weight-gradient GEMMs gain 6%, the ragged-M
  // ones do not (dgrad-ffn1 loses 14%), so only RAGGED_K switches
  if (p.kind != MOE_GEMM_RAGGED_K) return false;
  const uint64_t tiles =
      ceil_div(p.M, (uint64_t)BM) * ceil_div(p.N, (uint64_t)BN) * std::max<uint64_t>(1, p.num_b);
  return tiles < 4ull * (uint64_t)num_sms();
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
  arg_check(p.epilogue != MOE_EPI_DGELU || !p.colsum || (p.colsum_ws && p.colsum_max_m >= 1),
            "gemm.colsum_ws: DGELU column sums need colsum_ws / colsum_max_m");
  a.colsum = p.epilogue == MOE_EPI_DGELU && p.colsum ? p.colsum_ws : nullptr;
  a.cs_maxch = (int)((p.colsum_max_m + 31) / 32);
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
  // 64-wide column tiles when 128-wide ones would leave SMs idle in the last
  // wave (fewer than ~4 tiles per SM): c1's weight-gradient GEMMs
  const bool narrow = simt_use_bn64(p);
  auto go2 = [&](auto k128, auto k64) {
    if (narrow) launch_pdl(k64, grid, THREADS, 0, st, a);
    else launch_pdl(k128, grid, THREADS, 0, st, a);
  };
  if (p.kind == MOE_GEMM_RAGGED_K) {
    if (p.epilogue == MOE_EPI_ATOMIC_ADD) go2(simt_gemm_kernel<1, 0, MOE_EPI_ATOMIC_ADD, 128>, simt_gemm_kernel<1, 0, MOE_EPI_ATOMIC_ADD, 64>);
    else go2(simt_gemm_kernel<1, 0, MOE_EPI_STORE, 128>, simt_gemm_kernel<1, 0, MOE_EPI_STORE, 64>);
  } else {
    const bool bmn = p.b_mn_major != 0;
    switch (p.epilogue) {
      case MOE_EPI_GELU:
        bmn ? go2(simt_gemm_kernel<0, 1, MOE_EPI_GELU, 128>, simt_gemm_kernel<0, 1, MOE_EPI_GELU, 64>) : go2(simt_gemm_kernel<0, 0, MOE_EPI_GELU, 128>, simt_gemm_kernel<0, 0, MOE_EPI_GELU, 64>);
        break;
      case MOE_EPI_DGELU:
        bmn ? go2(simt_gemm_kernel<0, 1, MOE_EPI_DGELU, 128>, simt_gemm_kernel<0, 1, MOE_EPI_DGELU, 64>) : go2(simt_gemm_kernel<0, 0, MOE_EPI_DGELU, 128>, simt_gemm_kernel<0, 0, MOE_EPI_DGELU, 64>);
        break;
      case MOE_EPI_GATHER_ADD:
        bmn ? go2(simt_gemm_kernel<0, 1, MOE_EPI_GATHER_ADD, 128>, simt_gemm_kernel<0, 1, MOE_EPI_GATHER_ADD, 64>)
            : go2(simt_gemm_kernel<0, 0, MOE_EPI_GATHER_ADD, 128>, simt_gemm_kernel<0, 0, MOE_EPI_GATHER_ADD, 64>);
        break;
      case MOE_EPI_ATOMIC_ADD:
        bmn ? go2(simt_gemm_kernel<0, 1, MOE_EPI_ATOMIC_ADD, 128>, simt_gemm_kernel<0, 1, MOE_EPI_ATOMIC_ADD, 64>)
            : go2(simt_gemm_kernel<0, 0, MOE_EPI_ATOMIC_ADD, 128>, simt_gemm_kernel<0, 0, MOE_EPI_ATOMIC_ADD, 64>);
        break;
      default:
        bmn ? go2(simt_gemm_kernel<0, 1, MOE_EPI_STORE, 128>, simt_gemm_kernel<0, 1, MOE_EPI_STORE, 64>) : go2(simt_gemm_kernel<0, 0, MOE_EPI_STORE, 128>, simt_gemm_kernel<0, 0, MOE_EPI_STORE, 64>);
    }
  }
  MOE_LAUNCH_CHECK("simt_gemm_kernel");
  count_launch();
  if (p.kind == MOE_GEMM_RAGGED_M && p.epilogue == MOE_EPI_DGELU && p.colsum)
    seg_colsum(p.groups, p.m, p.b, p.num_b, p.N, BM, (uint32_t)a.cs_maxch, p.colsum_ws, p.colsum,
               st);
}

}  // namespace moe
