// K1 / K1^T on the fp32 path (config c1): the gate GEMMs have N or M = E
// (<= 256), far too skinny for the 128 x 128 SIMT expert-GEMM tiles (at E = 8
// those ran 16x padded on 32 CTAs). Three dedicated FP32-pipe kernels instead,
// each one pass over its token-sized operand (memory / latency bound):
//
//   gate_logits_f32   logits[t][e] = x[t] . wg[e] (+ bg[e])
//   gate_wgrad_f32    dwg[e][n]  += sum_t dl[t][e] x[t][n]  (token chunks, atomics)
//   gate_dx_f32       dx[t][n]    = sum_e dl[t][e] wg[e][n] + sum_i dXe[slot[t][i]][n]
//
// Semantics: Appendix A items 1 and 9; fp32 accumulation (the
// north-star fp32 tolerance is 1e-5 against the fp64 oracle).
#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace {

constexpr int GT = 256;  // threads per block

// One warp per token, lanes across K (float4 when aligned), experts in
// chunks of 8: per chunk each lane accumulates 8 partial dot products, then
// eight warp reductions.  x row and the wg rows stream through L1 / L2.
template <bool VEC>
__global__ void __launch_bounds__(GT) gate_logits_f32_kernel(uint64_t T, int d, int E,
                                                             const float* __restrict__ x,
                                                             const float* __restrict__ wg,
                                                             const float* __restrict__ bg,
                                                             float* __restrict__ logits) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const uint64_t t = (uint64_t)blockIdx.x * (GT / 32) + (threadIdx.x >> 5);
  if (t >= T) return;
  const float* xr = x + t * d;
  for (int e0 = 0; e0 < E; e0 += 8) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (VEC) {
      for (int k = lane * 4; k < d; k += 128) {
        const float4 xv = __ldg(reinterpret_cast<const float4*>(xr + k));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (e0 + j >= E) break;
          const float4 w = __ldg(reinterpret_cast<const float4*>(wg + (uint64_t)(e0 + j) * d + k));
          acc[j] = fmaf(xv.x, w.x, fmaf(xv.y, w.y, fmaf(xv.z, w.z, fmaf(xv.w, w.w, acc[j]))));
        }
      }
    } else {
      for (int k = lane; k < d; k += 32) {
        const float xv = xr[k];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (e0 + j >= E) break;
          acc[j] = fmaf(xv, wg[(uint64_t)(e0 + j) * d + k], acc[j]);
        }
      }
    }
    float mine = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float v = acc[j];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == j) mine = v;
    }
    if (lane < 8 && e0 + lane < E) logits[t * E + e0 + lane] = mine + (bg ? bg[e0 + lane] : 0.f);
  }
}

// Block: TOKC tokens x 64 columns; thread (col = tid % 64, eg = tid / 64)
// accumulates experts e = eg + 4 j over the chunk and stores the chunk's
// partial; the chunks are summed in order afterwards (deterministic).
// 32-token chunks: 4x the blocks of 128-token ones (c1: 1024 instead of 256,
// the per-thread token loop was latency-bound); their partials are summed in
// chunk order by sum_parts
constexpr int TOKC = kGateWgradTok;
template <int NE>
__global__ void __launch_bounds__(GT) gate_wgrad_f32_kernel(uint64_t T, int d, int E,
                                                            const float* __restrict__ dl,
                                                            const float* __restrict__ x,
                                                            float* __restrict__ dwg) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float dls[];  // [TOKC][E]
  const uint64_t t0 = (uint64_t)blockIdx.x * TOKC;
  const int ntok = (int)(T - t0 < (uint64_t)TOKC ? T - t0 : (uint64_t)TOKC);
  for (int i = threadIdx.x; i < ntok * E; i += GT) dls[i] = dl[t0 * E + i];
  __syncthreads();
  const int col = blockIdx.y * 64 + (threadIdx.x & 63), eg = threadIdx.x >> 6;
  if (col >= d) return;
  float acc[NE];
#pragma unroll
  for (int j = 0; j < NE; ++j) acc[j] = 0.f;
  const int ne = (E - eg + 3) / 4;  // experts of this thread (<= NE)
#pragma unroll 4
  for (int t = 0; t < ntok; ++t) {
    const float xv = __ldg(x + (t0 + t) * d + col);
    const float* dr = dls + t * E + eg;
#pragma unroll
    for (int j = 0; j < NE; ++j)
      if (j < ne) acc[j] = fmaf(dr[4 * j], xv, acc[j]);
  }
  // this token chunk's partial (summed over chunks in order by sum_parts)
  float* const part = dwg + (uint64_t)blockIdx.x * E * d;
#pragma unroll
  for (int j = 0; j < NE; ++j)
    if (j < ne) part[(uint64_t)(eg + 4 * j) * d + col] = acc[j];
}

// Block: 32 tokens x 64 columns; thread (col = tid % 64, tg = tid / 64)
// owns tokens tg + 4 i. wg[:, cols] and dl[tokens, :] staged in smem.
constexpr int DX_TOK = 32;
__global__ void __launch_bounds__(GT) gate_dx_f32_kernel(uint64_t T, int d, int E, int k,
                                                         const float* __restrict__ dl,
                                                         const float* __restrict__ wg,
                                                         const float* __restrict__ dXe,
                                                         const int32_t* __restrict__ slot,
                                                         float* __restrict__ dx) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float sm[];
  float* wsm = sm;            // [E][64]
  float* dls = sm + E * 64;   // [DX_TOK][E + 1]
  const uint64_t t0 = (uint64_t)blockIdx.x * DX_TOK;
  const int c0 = blockIdx.y * 64;
  for (int i = threadIdx.x; i < E * 64; i += GT) {
    const int e = i / 64, c = i % 64;
    wsm[i] = c0 + c < d ? wg[(uint64_t)e * d + c0 + c] : 0.f;
  }
  for (int i = threadIdx.x; i < DX_TOK * E; i += GT) {
    const int r = i / E, e = i % E;
    dls[r * (E + 1) + e] = t0 + r < T ? dl[(t0 + r) * E + e] : 0.f;
  }
  __syncthreads();
  const int c = threadIdx.x & 63, tg = threadIdx.x >> 6;
  const int col = c0 + c;
  float acc[DX_TOK / 4];
#pragma unroll
  for (int i = 0; i < DX_TOK / 4; ++i) acc[i] = 0.f;
  for (int e = 0; e < E; ++e) {
    const float w = wsm[e * 64 + c];
#pragma unroll
    for (int i = 0; i < DX_TOK / 4; ++i) acc[i] = fmaf(dls[(tg + 4 * i) * (E + 1) + e], w, acc[i]);
  }
  if (col >= d) return;
  // every routing slot of the thread's tokens first, then every gathered
  // row element (16 independent loads in flight instead of a chain per token),
  // then the sums in the same order as before (acc + row 0 + row 1)
  constexpr int NT = DX_TOK / 4;
  int32_t sl[NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const uint64_t t = t0 + tg + 4 * i;
#pragma unroll
    for (int j = 0; j < 2; ++j) sl[i][j] = (t < T && j < k) ? slot[t * k + j] : -1;
  }
  float gv[NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
      gv[i][j] = sl[i][j] >= 0 ? __ldg(dXe + (uint64_t)sl[i][j] * d + col) : 0.f;
#pragma unroll
  for (int i = 0; i < NT; ++i) {
    const uint64_t t = t0 + tg + 4 * i;
    if (t >= T) break;
    float v = acc[i];
#pragma unroll
    for (int j = 0; j < 2; ++j)
      if (sl[i][j] >= 0) v += gv[i][j];
    dx[t * d + col] = v;
  }
}

}  // namespace

void gate_logits_f32(uint64_t T, uint32_t d, uint32_t E, const float* x, const float* wg,
                     const float* bg, float* logits, cudaStream_t st) {
  if (!T) return;
  arg_check(E >= 1 && E <= 256, "gate_logits_f32: E must be in [1, 256]");
  const bool vec = d % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(wg) & 15) == 0;
  const unsigned grid = (unsigned)ceil_div(T, (uint64_t)(GT / 32));
  if (vec)
    launch_pdl(gate_logits_f32_kernel<true>, grid, GT, 0, st, T, (int)d, (int)E, x, wg, bg, logits);
  else
    launch_pdl(gate_logits_f32_kernel<false>, grid, GT, 0, st, T, (int)d, (int)E, x, wg, bg, logits);
  MOE_LAUNCH_CHECK("gate_logits_f32_kernel");
  count_launch();
}

void gate_wgrad_f32(uint64_t T, uint32_t d, uint32_t E, const float* dl, const float* x,
                    float* dwg, float* ws, cudaStream_t st) {
  if (!T) {
    MOE_CUDA(cudaMemsetAsync(dwg, 0, sizeof(float) * E * d, st));
    return;
  }
  arg_check(ws != nullptr, "gate_wgrad_f32.ws: workspace required");
  arg_check(E >= 1 && E <= 256, "gate_wgrad_f32: E must be in [1, 256]");
  const size_t smem = sizeof(float) * TOKC * E;
  dim3 grid((unsigned)ceil_div(T, TOKC), (unsigned)ceil_div(d, 64));
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      MOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    launch_pdl(kern, grid, GT, smem, st, T, (int)d, (int)E, dl, x, ws);
  };
  const uint32_t ne = (E + 3) / 4;  // experts per thread
  if (ne <= 1) go(gate_wgrad_f32_kernel<1>);
  else if (ne <= 2) go(gate_wgrad_f32_kernel<2>);
  else if (ne <= 4) go(gate_wgrad_f32_kernel<4>);
  else if (ne <= 8) go(gate_wgrad_f32_kernel<8>);
  else if (ne <= 16) go(gate_wgrad_f32_kernel<16>);
  else if (ne <= 32) go(gate_wgrad_f32_kernel<32>);
  else go(gate_wgrad_f32_kernel<64>);
  MOE_LAUNCH_CHECK("gate_wgrad_f32_kernel");
  count_launch();
  sum_parts(ws, (uint32_t)ceil_div(T, (uint64_t)TOKC), (uint64_t)E * d, E, d, d, false, dwg, st);
}

void gate_dx_f32(uint64_t T, uint32_t d, uint32_t E, uint32_t k, const float* dl, const float* wg,
                 const float* dXe, const int32_t* slot, float* dx, cudaStream_t st) {
  if (!T) return;
  arg_check(E >= 1 && E <= 256, "gate_dx_f32: E must be in [1, 256]");
  arg_check(k >= 1 && k <= 2, "gate_dx_f32: k must be 1 or 2");
  const size_t smem = sizeof(float) * (E * 64 + DX_TOK * (E + 1));
  if (smem > 48 * 1024)
    MOE_CUDA(cudaFuncSetAttribute(gate_dx_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  dim3 grid((unsigned)ceil_div(T, DX_TOK), (unsigned)ceil_div(d, 64));
  launch_pdl(gate_dx_f32_kernel, grid, GT, smem, st, T, (int)d, (int)E, (int)k, dl, wg, dXe, slot, dx);
  MOE_LAUNCH_CHECK("gate_dx_f32_kernel");
  count_launch();
}

}  // namespace moe
