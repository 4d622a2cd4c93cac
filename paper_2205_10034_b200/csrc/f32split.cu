// fp32 expert GEMMs (config c1) on the bf16 tensor cores.
//
// Config c1 is fp32 with a 1e-5 tolerance.  Each fp32 operand is split into
// three bf16 planes x = p0 + p1 + p2 (p0 = bf16(x), p1 = bf16(x - p0), p2 =
// bf16(x - p0 - p1): 24 significand bits, exact up to ~2^-27 |x|), and the
// tcgen05 GEMM (moe_gemm_problem_t.split_terms = 6) sums the six leading plane
// products (error ~2^-22 relative per product).  The tensor core's fp32
// accumulation truncates (benchmarks/tc_accum_probe.py: -1.8 ulp mean at K =
// 512, -168 ulp at K = 4096), so the K loop is cut into chunks of at most 512
// (their products accumulate in TMEM, the main p0 q0 term last) and the chunk
// partials are summed here in fp32, round-to-nearest, in chunk order --
// bitwise reproducible -- fused with the layer epilogue (bias, GeLU / GeLU',
// x gelu', zero pad rows).
//
// All kernels are HBM-bound elementwise passes (float4 / bf16x4 vectors).
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace {

__device__ __forceinline__ void split3_store4(float4 v, __nv_bfloat16* out, uint64_t n,
                                              uint64_t at) {
  const float x[4] = {v.x, v.y, v.z, v.w};
  uint32_t w[3][2];
#pragma unroll
  for (int j = 0; j < 4; j += 2) {
    uint32_t lo[3], hi[3];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const __nv_bfloat16 a = __float2bfloat16_rn(x[j + h]);
      const float r1 = x[j + h] - __bfloat162float(a);  // exact
      const __nv_bfloat16 b = __float2bfloat16_rn(r1);
      const __nv_bfloat16 c = __float2bfloat16_rn(r1 - __bfloat162float(b));
      const uint32_t ua = __bfloat16_as_ushort(a), ub = __bfloat16_as_ushort(b),
                     uc = __bfloat16_as_ushort(c);
      if (h == 0) { lo[0] = ua; lo[1] = ub; lo[2] = uc; }
      else { hi[0] = ua; hi[1] = ub; hi[2] = uc; }
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) w[t][j / 2] = lo[t] | (hi[t] << 16);
  }
#pragma unroll
  for (int t = 0; t < 3; ++t)
    *reinterpret_cast<uint2*>(out + (uint64_t)t * n + at) = make_uint2(w[t][0], w[t][1]);
}

__global__ void split3_kernel(const float* __restrict__ in, uint64_t n4,
                              __nv_bfloat16* __restrict__ out, uint64_t n) {
  pdl_wait();
  pdl_trigger();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    split3_store4(__ldg(reinterpret_cast<const float4*>(in) + i), out, n, 4 * i);
  }
}

// Rows of group g: [ga[g], ga[g] + stride); rows < gm[g] get
//   h = sum_c part[c][row][n] (+ bias[gb[g]][n]); MODE 0: out = h;
//   MODE 1: out = gelu(h), out2 = gelu'(h); MODE 2: out = h * aux[row][n];
// rows in [gm[g], round_up(gm[g], 64)) are zeroed (the tcgen05 RAGGED_K GEMMs
// read whole 64-row K blocks); rows past that are never read and not written
// (c1: ~15% of each finish pass's bytes).  out3 (nullable): the result's three bf16 planes too (the
// next split GEMM's operand; n3 = elements per plane) -- for MODE 1 it
// replaces out (the fp32 activation itself is never read again).
// Grid: (groups, row blocks of 8, column blocks of 128).
template <int MODE>
__global__ void __launch_bounds__(256) finish_kernel(
    const float* __restrict__ part, int nparts, uint64_t pstride, const int32_t* __restrict__ gm,
    const int32_t* __restrict__ ga, const int32_t* __restrict__ gb, int stride, int N,
    const float* __restrict__ bias, const float* __restrict__ aux, float* __restrict__ out,
    float* __restrict__ out2, __nv_bfloat16* __restrict__ out3, uint64_t n3) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x;
  const int m = gm[g];
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (r >= min(stride, (m + 63) & ~63)) return;
  const int n = (blockIdx.z * 32 + (threadIdx.x & 31)) * 4;
  if (n >= N) return;
  const uint64_t off = ((uint64_t)ga[g] + r) * N + n;
  float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
  if (r < m) {
    for (int c = 0; c < nparts; ++c) {
      const float4 v = __ldcg(reinterpret_cast<const float4*>(part + (uint64_t)c * pstride + off));
      h.x += v.x;
      h.y += v.y;
      h.z += v.z;
      h.w += v.w;
    }
    if (bias) {
      const float4 b = __ldg(reinterpret_cast<const float4*>(bias + (uint64_t)gb[g] * N + n));
      h.x += b.x;
      h.y += b.y;
      h.z += b.z;
      h.w += b.w;
    }
  }
  if (MODE == 1) {
    float4 a, d;
    gelu_and_grad_f(h.x, a.x, d.x);
    gelu_and_grad_f(h.y, a.y, d.y);
    gelu_and_grad_f(h.z, a.z, d.z);
    gelu_and_grad_f(h.w, a.w, d.w);
    if (r >= m) a = d = make_float4(0.f, 0.f, 0.f, 0.f);
    if (out) *reinterpret_cast<float4*>(out + off) = a;
    if (out3) split3_store4(a, out3, n3, off);
    *reinterpret_cast<float4*>(out2 + off) = d;
    return;
  }
  if (MODE == 2 && r < m) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(aux + off));
    h.x *= x.x;
    h.y *= x.y;
    h.z *= x.z;
    h.w *= x.w;
  }
  if (out) *reinterpret_cast<float4*>(out + off) = h;
  if (out3) split3_store4(h, out3, n3, off);
}

// Planes + bias gradient in one pass: a block owns 32 rows (a warp 4
// consecutive rows) x 128 columns of one group, computes the rows' values --
// SRC 0: dH = (sum of the K-chunk partials) * gelu' (MODE 2 of finish_kernel);
// SRC 1: a plain fp32 input (dY) -- stores their three bf16 planes (and fp32,
// if `out`), and writes the column sums of its 32 rows (rows >= m are zero)
// to cs_part[(g * maxch + row block) * N + n]: the 32-row chunk partials
// seg_colsum sums in chunk order (deterministic) -- instead of a separate
// column-sum pass re-reading the values (db1 / db2).
template <int SRC>
__global__ void __launch_bounds__(256) planes_colsum_kernel(
    const float* __restrict__ part, int nparts, uint64_t pstride, const int32_t* __restrict__ gm,
    const int32_t* __restrict__ ga, int stride, int N, const float* __restrict__ aux,
    float* __restrict__ out, __nv_bfloat16* __restrict__ out3, uint64_t n3,
    float* __restrict__ cs_part, int maxch) {
  pdl_wait();
  pdl_trigger();
  __shared__ float4 red[8][32];
  const int g = blockIdx.x;
  const int m = gm[g];
  const int lim = min(stride, (m + 63) & ~63);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = (blockIdx.z * 32 + lane) * 4;
  float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = blockIdx.y * 32 + w * 4 + i;
    if (r >= lim || n >= N) continue;
    const uint64_t off = ((uint64_t)ga[g] + r) * N + n;
    float4 h = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < m && SRC == 1) {
      h = __ldcg(reinterpret_cast<const float4*>(part + off));
    } else if (r < m) {
      for (int c = 0; c < nparts; ++c) {
        const float4 v = __ldcg(reinterpret_cast<const float4*>(part + (uint64_t)c * pstride + off));
        h.x += v.x;
        h.y += v.y;
        h.z += v.z;
        h.w += v.w;
      }
      const float4 x = __ldg(reinterpret_cast<const float4*>(aux + off));
      h.x *= x.x;
      h.y *= x.y;
      h.z *= x.z;
      h.w *= x.w;
    }
    if (out) *reinterpret_cast<float4*>(out + off) = h;
    if (out3) split3_store4(h, out3, n3, off);
    cs.x += h.x;
    cs.y += h.y;
    cs.z += h.z;
    cs.w += h.w;
  }
  red[w][lane] = cs;
  __syncthreads();
  if (w == 0 && n < N && blockIdx.y < (unsigned)maxch) {
    float4 t = red[0][lane];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      t.x += red[k][lane].x;
      t.y += red[k][lane].y;
      t.z += red[k][lane].z;
      t.w += red[k][lane].w;
    }
    *reinterpret_cast<float4*>(cs_part + ((uint64_t)g * maxch + blockIdx.y) * N + n) = t;
  }
}

// K-chunk group tables, group (c, g) = c * groups + g:
//   RAGGED_M (kind 0): m = gm, a_row = ga, c_row = c * rows + ga, b = gb, k = c * chunk
//   RAGGED_K (kind 1): m = clamp(gm - c*chunk, 0, chunk), a_row = ga + c*chunk, b = c*nb + gb
__global__ void chunk_tables_kernel(int kind, uint32_t groups, int nchunks, int chunk, int rows,
                                    int nb, const int32_t* __restrict__ gm,
                                    const int32_t* __restrict__ ga, const int32_t* __restrict__ gb,
                                    int32_t* __restrict__ om, int32_t* __restrict__ oa,
                                    int32_t* __restrict__ oc, int32_t* __restrict__ ob,
                                    int32_t* __restrict__ ok) {
  pdl_wait();
  pdl_trigger();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= groups * (uint32_t)nchunks) return;
  const int c = (int)(i / groups), g = (int)(i % groups);
  if (kind == 0) {
    om[i] = gm[g];
    oa[i] = ga[g];
    oc[i] = c * rows + ga[g];
    ob[i] = gb[g];
    ok[i] = c * chunk;
  } else {
    om[i] = max(0, min(chunk, gm[g] - c * chunk));
    oa[i] = ga[g] + c * chunk;
    ob[i] = c * nb + gb[g];
  }
}

}  // namespace

void split_f32_bf16x3(const float* in, uint64_t n, void* out, cudaStream_t st) {
  if (!n) return;
  arg_check(n % 4 == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0 &&
                (reinterpret_cast<uintptr_t>(out) & 7) == 0,
            "split_f32: n % 4 == 0 and 16-byte aligned input required");
  const uint64_t n4 = n / 4;
  const unsigned blocks = (unsigned)std::min<uint64_t>(ceil_div(n4, (uint64_t)256), (uint64_t)num_sms() * 16);
  launch_pdl(split3_kernel, blocks, 256, 0, st, in, n4, static_cast<__nv_bfloat16*>(out), n);
  MOE_LAUNCH_CHECK("split3_kernel");
  count_launch();
}

void split_finish(int mode, const float* part, int nparts, uint64_t part_stride, uint32_t groups,
                  const int32_t* gm, const int32_t* ga, const int32_t* gb, uint32_t stride,
                  uint32_t N, const float* bias, const float* aux, float* out, float* out2,
                  void* out3, uint64_t n3, cudaStream_t st) {
  __nv_bfloat16* o3 = static_cast<__nv_bfloat16*>(out3);
  arg_check(N % 4 == 0, "split_finish: N % 4 == 0 required");
  const dim3 grid(groups, (unsigned)ceil_div((uint64_t)stride, (uint64_t)8),
                  (unsigned)ceil_div((uint64_t)N, (uint64_t)128));
  if (mode == 0)
    launch_pdl(finish_kernel<0>, grid, 256, 0, st, part, nparts, part_stride, gm, ga, gb,
               (int)stride, (int)N, bias, aux, out, out2, o3, n3);
  else if (mode == 1)
    launch_pdl(finish_kernel<1>, grid, 256, 0, st, part, nparts, part_stride, gm, ga, gb,
               (int)stride, (int)N, bias, aux, out, out2, o3, n3);
  else
    launch_pdl(finish_kernel<2>, grid, 256, 0, st, part, nparts, part_stride, gm, ga, gb,
               (int)stride, (int)N, bias, aux, out, out2, o3, n3);
  MOE_LAUNCH_CHECK("finish_kernel");
  count_launch();
}

void split_finish_dgelu_colsum(const float* part, int nparts, uint64_t part_stride,
                               uint32_t groups, const int32_t* gm, const int32_t* ga,
                               const int32_t* gb, uint32_t num_b, uint32_t stride, uint32_t N,
                               const float* aux, float* out, void* out3, uint64_t n3,
                               float* cs_part, float* db, cudaStream_t st) {
  arg_check(N % 4 == 0, "split_finish: N % 4 == 0 required");
  const int maxch = (int)ceil_div((uint64_t)stride, (uint64_t)32);
  const dim3 grid(groups, (unsigned)maxch, (unsigned)ceil_div((uint64_t)N, (uint64_t)128));
  launch_pdl(planes_colsum_kernel<0>, grid, 256, 0, st, part, nparts, part_stride, gm, ga,
             (int)stride, (int)N, aux, out, static_cast<__nv_bfloat16*>(out3), n3, cs_part, maxch);
  MOE_LAUNCH_CHECK("planes_colsum_kernel");
  count_launch();
  seg_colsum(groups, gm, gb, num_b, N, 32, (uint32_t)maxch, cs_part, db, st);
}

void split_colsum_f32(const float* in, uint32_t groups, const int32_t* gm, const int32_t* ga,
                      const int32_t* gb, uint32_t num_b, uint32_t stride, uint32_t N, void* out3,
                      uint64_t n3, float* cs_part, float* db, cudaStream_t st) {
  arg_check(N % 4 == 0, "split_colsum: N % 4 == 0 required");
  const int maxch = (int)ceil_div((uint64_t)stride, (uint64_t)32);
  const dim3 grid(groups, (unsigned)maxch, (unsigned)ceil_div((uint64_t)N, (uint64_t)128));
  launch_pdl(planes_colsum_kernel<1>, grid, 256, 0, st, in, 1, (uint64_t)0, gm, ga, (int)stride,
             (int)N, nullptr, nullptr, static_cast<__nv_bfloat16*>(out3), n3, cs_part, maxch);
  MOE_LAUNCH_CHECK("planes_colsum_kernel");
  count_launch();
  seg_colsum(groups, gm, gb, num_b, N, 32, (uint32_t)maxch, cs_part, db, st);
}

void chunk_tables(int kind, uint32_t groups, int nchunks, int chunk, int rows, int nb,
                  const int32_t* gm, const int32_t* ga, const int32_t* gb, int32_t* om,
                  int32_t* oa, int32_t* oc, int32_t* ob, int32_t* ok, cudaStream_t st) {
  const uint64_t n = (uint64_t)groups * nchunks;
  launch_pdl(chunk_tables_kernel, (unsigned)ceil_div(n, (uint64_t)256), 256, 0, st, kind, groups,
             nchunks, chunk, rows, nb, gm, ga, gb, om, oa, oc, ob, ok);
  MOE_LAUNCH_CHECK("chunk_tables_kernel");
  count_launch();
}

}  // namespace moe
