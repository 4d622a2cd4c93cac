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

__global__ void split3_kernel(const float* __restrict__ in, uint64_t n4,
                              __nv_bfloat16* __restrict__ out, uint64_t n) {
  pdl_wait();
  pdl_trigger();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(in) + i);
    const float x[4] = {v.x, v.y, v.z, v.w};
    __nv_bfloat16 p[3][4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat16 a = __float2bfloat16_rn(x[j]);
      const float r1 = x[j] - __bfloat162float(a);  // exact (Sterbenz)
      const __nv_bfloat16 b = __float2bfloat16_rn(r1);
      const __nv_bfloat16 c = __float2bfloat16_rn(r1 - __bfloat162float(b));
      p[0][j] = a;
      p[1][j] = b;
      p[2][j] = c;
    }
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      uint2 w;
      w.x = (uint32_t)__bfloat16_as_ushort(p[t][0]) | ((uint32_t)__bfloat16_as_ushort(p[t][1]) << 16);
      w.y = (uint32_t)__bfloat16_as_ushort(p[t][2]) | ((uint32_t)__bfloat16_as_ushort(p[t][3]) << 16);
      *reinterpret_cast<uint2*>(out + (uint64_t)t * n + 4 * i) = w;
    }
  }
}

// Rows of group g: [ga[g], ga[g] + stride); rows < gm[g] get
//   h = sum_c part[c][row][n] (+ bias[gb[g]][n]); MODE 0: out = h;
//   MODE 1: out = gelu(h), out2 = gelu'(h); MODE 2: out = h * aux[row][n];
// rows in [gm[g], stride) are zeroed (the tcgen05 RAGGED_K GEMMs read whole
// 64-row K blocks).  Grid: (groups, row blocks of 8, column blocks of 128).
template <int MODE>
__global__ void __launch_bounds__(256) finish_kernel(
    const float* __restrict__ part, int nparts, uint64_t pstride, const int32_t* __restrict__ gm,
    const int32_t* __restrict__ ga, const int32_t* __restrict__ gb, int stride, int N,
    const float* __restrict__ bias, const float* __restrict__ aux, float* __restrict__ out,
    float* __restrict__ out2) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x;
  const int m = gm[g];
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (r >= stride) return;
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
    *reinterpret_cast<float4*>(out + off) = a;
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
  *reinterpret_cast<float4*>(out + off) = h;
}

__global__ void chunk_groups_kernel(uint32_t groups, const int32_t* __restrict__ gm,
                                    const int32_t* __restrict__ ga, int chunk, int c,
                                    int32_t* __restrict__ cm, int32_t* __restrict__ ca) {
  pdl_wait();
  pdl_trigger();
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= groups) return;
  cm[g] = max(0, min(chunk, gm[g] - c * chunk));
  ca[g] = ga[g] + c * chunk;
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
                  cudaStream_t st) {
  arg_check(N % 4 == 0, "split_finish: N % 4 == 0 required");
  const dim3 grid(groups, (unsigned)ceil_div((uint64_t)stride, (uint64_t)8),
                  (unsigned)ceil_div((uint64_t)N, (uint64_t)128));
  if (mode == 0)
    launch_pdl(finish_kernel<0>, grid, 256, 0, st, part, nparts, part_stride, gm, ga, gb,
               (int)stride, (int)N, bias, aux, out, out2);
  else if (mode == 1)
    launch_pdl(finish_kernel<1>, grid, 256, 0, st, part, nparts, part_stride, gm, ga, gb,
               (int)stride, (int)N, bias, aux, out, out2);
  else
    launch_pdl(finish_kernel<2>, grid, 256, 0, st, part, nparts, part_stride, gm, ga, gb,
               (int)stride, (int)N, bias, aux, out, out2);
  MOE_LAUNCH_CHECK("finish_kernel");
  count_launch();
}

void chunk_groups(uint32_t groups, const int32_t* gm, const int32_t* ga, int chunk, int c,
                  int32_t* cm, int32_t* ca, cudaStream_t st) {
  launch_pdl(chunk_groups_kernel, (unsigned)ceil_div((uint64_t)groups, (uint64_t)256), 256, 0, st,
             groups, gm, ga, chunk, c, cm, ca);
  MOE_LAUNCH_CHECK("chunk_groups_kernel");
  count_launch();
}

}  // namespace moe
