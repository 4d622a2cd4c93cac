// Fixed-order reductions for the gradient paths.
//
// Every gradient that used to be accumulated with float atomics (split-K dWg,
// db1 in the DGELU epilogue, dbg in the routing backward, db2 column sums of
// several groups, the fp32 gate wgrad) now writes per-block partials with
// plain stores and is summed here in a fixed order, so a training step's
// gradients are bitwise reproducible run to run — the reference's simulator
// is deterministic by construction (acceptance_main.cpp:442-486).
//
// Both kernels are HBM/L2-bound streaming reductions: one thread per output
// element walks the partials in index order; adjacent threads read adjacent
// columns (coalesced 128-byte lines per warp).
#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace {

constexpr int RT = 256;

// out[r*cols + c] (transpose: out[c*rows + r]) = sum_{p < nparts} part[p*pstride + r*ldp + c]
__global__ void __launch_bounds__(RT) sum_parts_kernel(const float* __restrict__ part,
                                                       uint32_t nparts, uint64_t pstride,
                                                       uint64_t rows, uint64_t cols, uint64_t ldp,
                                                       int transpose, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const uint64_t i = (uint64_t)blockIdx.x * RT + threadIdx.x;
  if (i >= rows * cols) return;
  const uint64_t r = i / cols, c = i % cols;
  const float* p = part + r * ldp + c;
  float s = 0.f;
  uint32_t q = 0;
  for (; q + 4 <= nparts; q += 4) {  // 4 loads in flight, summed in index order
    const float a0 = __ldcg(p + (uint64_t)q * pstride), a1 = __ldcg(p + (uint64_t)(q + 1) * pstride);
    const float a2 = __ldcg(p + (uint64_t)(q + 2) * pstride), a3 = __ldcg(p + (uint64_t)(q + 3) * pstride);
    s += a0;
    s += a1;
    s += a2;
    s += a3;
  }
  for (; q < nparts; ++q) s += __ldcg(p + (uint64_t)q * pstride);
  out[transpose ? c * rows + r : i] = s;
}

// out[b][n] = sum over groups g (ascending) with gb[g] == b of
//             sum over chunks ch < ceil(gm[g] / chunk) of ws[(g*maxch + ch)*N + n]
__global__ void __launch_bounds__(RT) seg_colsum_kernel(uint32_t groups, const int32_t* __restrict__ gm,
                                                        const int32_t* __restrict__ gb, uint32_t N,
                                                        uint32_t chunk, uint32_t maxch,
                                                        const float* __restrict__ ws,
                                                        float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_nch[1024];
  __shared__ int s_b[1024];
  const int b = blockIdx.x;
  for (uint32_t g = threadIdx.x; g < groups; g += RT) {
    s_b[g] = gb[g];
    s_nch[g] = min((int)maxch, (gm[g] + (int)chunk - 1) / (int)chunk);
  }
  __syncthreads();
  const uint32_t n = blockIdx.y * RT + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (uint32_t g = 0; g < groups; ++g) {
    if (s_b[g] != b) continue;
    const float* p = ws + (uint64_t)g * maxch * N + n;
    const int nch = s_nch[g];
    int ch = 0;
    for (; ch + 4 <= nch; ch += 4) {
      const float a0 = __ldcg(p + (uint64_t)ch * N), a1 = __ldcg(p + (uint64_t)(ch + 1) * N);
      const float a2 = __ldcg(p + (uint64_t)(ch + 2) * N), a3 = __ldcg(p + (uint64_t)(ch + 3) * N);
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; ch < nch; ++ch) s += __ldcg(p + (uint64_t)ch * N);
  }
  out[(uint64_t)b * N + n] = s;
}

}  // namespace

void sum_parts(const float* part, uint32_t nparts, uint64_t part_stride, uint64_t rows,
               uint64_t cols, uint64_t ldp, bool transpose, float* out, cudaStream_t st) {
  const uint64_t n = rows * cols;
  if (!n) return;
  launch_pdl(sum_parts_kernel, (unsigned)ceil_div(n, (uint64_t)RT), RT, 0, st, part, nparts,
             part_stride, rows, cols, ldp, transpose ? 1 : 0, out);
  MOE_LAUNCH_CHECK("sum_parts_kernel");
  count_launch();
}

void seg_colsum(uint32_t groups, const int32_t* gm, const int32_t* gb, uint32_t num_b, uint32_t N,
                uint32_t chunk, uint32_t maxch, const float* ws, float* out, cudaStream_t st) {
  arg_check(groups >= 1 && groups <= 1024, "colsum.groups: must be in [1, 1024]");
  if (!num_b || !N) return;
  launch_pdl(seg_colsum_kernel, dim3(num_b, (unsigned)ceil_div((uint64_t)N, (uint64_t)RT)), RT, 0, st,
             groups, gm, gb, N, chunk, maxch, ws, out);
  MOE_LAUNCH_CHECK("seg_colsum_kernel");
  count_launch();
}

}  // namespace moe
