// Fixed-order reductions for the gradient paths.
//
// Every gradient that used to be accumulated with float atomics (split-K dWg,
// db1 in the DGELU epilogue, dbg in the routing backward, db2 column sums of
// several groups, the fp32 gate wgrad) now writes per-block partials with
// plain stores and is summed here in a fixed order, so a training step's
// gradients are bitwise reproducible run to run — the reference's simulator
// is deterministic by construction (acceptance_main.cpp:442-486).
//
// Both kernels are HBM/L2-bound streaming reductions: a warp reads 32
// adjacent outputs of one partial (a coalesced 128-byte line), eight warps
// split the partials and are combined in a fixed order.
#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace {

// Block = 32 output columns x PW part-groups: lane = column, warp w sums the
// partials p = w, w + PW, ... (all its loads independent), then warp 0 adds
// the PW group sums in order -- a fixed summation order, bitwise reproducible.
constexpr int PW = 8;
constexpr int RT = 32 * PW;

// out[r*cols + c] (transpose: out[c*rows + r]) = sum_{p < nparts} part[p*pstride + r*ldp + c]
__global__ void __launch_bounds__(RT) sum_parts_kernel(const float* __restrict__ part,
                                                       uint32_t nparts, uint64_t pstride,
                                                       uint64_t rows, uint64_t cols, uint64_t ldp,
                                                       int transpose, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[PW][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t i = (uint64_t)blockIdx.x * 32 + lane;
  const bool ok = i < rows * cols;
  const uint64_t r = ok ? i / cols : 0, c = ok ? i % cols : 0;
  const float* p = part + r * ldp + c;
  float s = 0.f;
  if (ok)
    for (uint32_t q = w; q < nparts; q += PW) s += __ldcg(p + (uint64_t)q * pstride);
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && ok) {
    float t = red[0][lane];
#pragma unroll
    for (int k = 1; k < PW; ++k) t += red[k][lane];
    out[transpose ? c * rows + r : i] = t;
  }
}

// out[b][n] = sum over groups g (ascending) with gb[g] == b of
//             sum over chunks ch < ceil(gm[g] / chunk) of ws[(g*maxch + ch)*N + n]
// (chunks split over the PW warps like sum_parts)
__global__ void __launch_bounds__(RT) seg_colsum_kernel(uint32_t groups, const int32_t* __restrict__ gm,
                                                        const int32_t* __restrict__ gb, uint32_t N,
                                                        uint32_t chunk, uint32_t maxch,
                                                        const float* __restrict__ ws,
                                                        float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_nch[1024];
  __shared__ int s_b[1024];
  __shared__ float red[PW][32];
  const int b = blockIdx.x;
  for (uint32_t g = threadIdx.x; g < groups; g += RT) {
    s_b[g] = gb[g];
    s_nch[g] = min((int)maxch, (gm[g] + (int)chunk - 1) / (int)chunk);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t n = blockIdx.y * 32 + lane;
  float s = 0.f;
  if (n < N) {
    for (uint32_t g = 0; g < groups; ++g) {
      if (s_b[g] != b) continue;
      const float* p = ws + (uint64_t)g * maxch * N + n;
      for (int ch = w; ch < s_nch[g]; ch += PW) s += __ldcg(p + (uint64_t)ch * N);
    }
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && n < N) {
    float t = red[0][lane];
#pragma unroll
    for (int k = 1; k < PW; ++k) t += red[k][lane];
    out[(uint64_t)b * N + n] = t;
  }
}

}  // namespace

void sum_parts(const float* part, uint32_t nparts, uint64_t part_stride, uint64_t rows,
               uint64_t cols, uint64_t ldp, bool transpose, float* out, cudaStream_t st) {
  const uint64_t n = rows * cols;
  if (!n) return;
  launch_pdl(sum_parts_kernel, (unsigned)ceil_div(n, (uint64_t)32), RT, 0, st, part, nparts,
             part_stride, rows, cols, ldp, transpose ? 1 : 0, out);
  MOE_LAUNCH_CHECK("sum_parts_kernel");
  count_launch();
}

void seg_colsum(uint32_t groups, const int32_t* gm, const int32_t* gb, uint32_t num_b, uint32_t N,
                uint32_t chunk, uint32_t maxch, const float* ws, float* out, cudaStream_t st) {
  arg_check(groups >= 1 && groups <= 1024, "colsum.groups: must be in [1, 1024]");
  if (!num_b || !N) return;
  launch_pdl(seg_colsum_kernel, dim3(num_b, (unsigned)ceil_div((uint64_t)N, (uint64_t)32)), RT, 0, st,
             groups, gm, gb, N, chunk, maxch, ws, out);
  MOE_LAUNCH_CHECK("seg_colsum_kernel");
  count_launch();
}

}  // namespace moe
