// Fixed-order reductions for the gradient paths.
//
// Every gradient that used to be accumulated with float atomics (split-K dWg,
// db1 in the DGELU epilogue, dbg in the routing backward, db2 column sums of
// several groups, the fp32 gate wgrad) now writes per-block partials with
// plain stores and is summed here in a fixed order, so a training step's
// gradients are bitwise reproducible run to run — the reference's simulator
// is deterministic by construction (acceptance_main.cpp:442-486).
//
// Both kernels are HBM/L2-bound streaming reductions: a warp reads 128
// adjacent outputs of one partial (512 contiguous bytes, float4 per lane),
// eight warps split the partials and are combined in a fixed order.
#include "common.cuh"
#include "kernels.h"

namespace moe {
namespace {

// Block = 32 lanes x PW part-groups: lane = 4 adjacent outputs (one float4,
// a warp covers 512 contiguous bytes of a partial row), warp w sums the
// partials p = w, w + PW, ... with every load of its loop in flight, then
// warp 0 adds the PW group sums in order -- a fixed summation order.
constexpr int PW = 8;
constexpr int RT = 32 * PW;

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// out[r*cols + c] (transpose: out[c*rows + r]) = sum_{p < nparts} part[p*pstride + r*ldp + c]
// VEC: cols % 4 == 0, ldp % 4 == 0, pstride % 4 == 0 (float4 loads)
template <bool VEC>
__global__ void __launch_bounds__(RT) sum_parts_kernel(const float* __restrict__ part,
                                                       uint32_t nparts, uint64_t pstride,
                                                       uint64_t rows, uint64_t cols, uint64_t ldp,
                                                       int transpose, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int V = VEC ? 4 : 1;
  __shared__ float4 red[PW][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t i = ((uint64_t)blockIdx.x * 32 + lane) * V;  // first of this lane's outputs
  const bool ok = i < rows * cols;
  const uint64_t r = ok ? i / cols : 0, c = ok ? i % cols : 0;
  const float* p = part + r * ldp + c;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (ok) {
    auto ld = [&](uint32_t q) -> float4 {
      if (VEC) return __ldcg(reinterpret_cast<const float4*>(p + (uint64_t)q * pstride));
      return make_float4(__ldcg(p + (uint64_t)q * pstride), 0.f, 0.f, 0.f);
    };
    uint32_t q = w;
    for (; q + 3 * PW < nparts; q += 4 * PW) {  // four loads in flight, summed in order
      const float4 a0 = ld(q), a1 = ld(q + PW), a2 = ld(q + 2 * PW), a3 = ld(q + 3 * PW);
      s = add4(add4(add4(add4(s, a0), a1), a2), a3);
    }
    for (; q < nparts; q += PW) s = add4(s, ld(q));
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && ok) {
    float4 t = red[0][lane];
#pragma unroll
    for (int k = 1; k < PW; ++k) t = add4(t, red[k][lane]);
    const float tv[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
    for (int v = 0; v < V; ++v) out[transpose ? (c + v) * rows + r : i + v] = tv[v];
  }
}

// out[b][n] = sum over groups g (ascending) with gb[g] == b of
//             sum over chunks ch < ceil(gm[g] / chunk) of ws[(g*maxch + ch)*N + n]
// (chunks split over the PW warps like sum_parts; VEC: N % 4 == 0)
template <bool VEC>
__global__ void __launch_bounds__(RT) seg_colsum_kernel(uint32_t groups, const int32_t* __restrict__ gm,
                                                        const int32_t* __restrict__ gb, uint32_t N,
                                                        uint32_t chunk, uint32_t maxch,
                                                        const float* __restrict__ ws,
                                                        float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int V = VEC ? 4 : 1;
  __shared__ float4 red[PW][32];
  __shared__ int glist[1024];  // this output's groups, ascending
  __shared__ int wcnt[PW], gtotal;
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // ordered compaction of {g : gb[g] == b} by the whole block (ballots + a
  // prefix over the warps per 256-group slice) instead of every warp walking
  // all groups (c2: 64 dependent checks per warp, ~90% of this kernel's
  // instructions); the summation order below is unchanged (ascending g)
  if (threadIdx.x == 0) gtotal = 0;
  __syncthreads();
  for (uint32_t g0 = 0; g0 < groups; g0 += RT) {
    const uint32_t g = g0 + threadIdx.x;
    const bool mine = g < groups && __ldg(gb + g) == b;
    const uint32_t bal = __ballot_sync(0xffffffffu, mine);
    if (lane == 0) wcnt[w] = __popc(bal);
    __syncthreads();
    int base = gtotal;
    for (int k = 0; k < w; ++k) base += wcnt[k];
    if (mine) glist[base + __popc(bal & ((1u << lane) - 1u))] = (int)g;
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int k = 0; k < PW; ++k) t += wcnt[k];
      gtotal += t;
    }
    __syncthreads();
  }
  const int ng = gtotal;
  const uint32_t n = (blockIdx.y * 32 + lane) * V;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  if (n < N) {
    for (int gi = 0; gi < ng; ++gi) {
      const uint32_t g = (uint32_t)glist[gi];
      const int nch = min((int)maxch, (__ldg(gm + g) + (int)chunk - 1) / (int)chunk);
      const float* p = ws + (uint64_t)g * maxch * N + n;
      auto ld = [&](int ch) -> float4 {
        if (VEC) return __ldcg(reinterpret_cast<const float4*>(p + (uint64_t)ch * N));
        return make_float4(__ldcg(p + (uint64_t)ch * N), 0.f, 0.f, 0.f);
      };
      int ch = w;
      for (; ch + 3 * PW < nch; ch += 4 * PW) {  // four loads in flight, summed in order
        const float4 a0 = ld(ch), a1 = ld(ch + PW), a2 = ld(ch + 2 * PW), a3 = ld(ch + 3 * PW);
        s = add4(add4(add4(add4(s, a0), a1), a2), a3);
      }
      for (; ch < nch; ch += PW) s = add4(s, ld(ch));
    }
  }
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && n < N) {
    float4 t = red[0][lane];
#pragma unroll
    for (int k = 1; k < PW; ++k) t = add4(t, red[k][lane]);
    if (VEC) *reinterpret_cast<float4*>(out + (uint64_t)b * N + n) = t;
    else out[(uint64_t)b * N + n] = t.x;
  }
}

// Few partials over many outputs (the split-fp32 weight gradients): one
// float4 of outputs per thread, grid-stride, partials summed in index order.
__global__ void __launch_bounds__(256) sum_few_parts_kernel(const float4* __restrict__ part,
                                                            uint32_t nparts, uint64_t pstride4,
                                                            uint64_t n4, float4* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (uint64_t)gridDim.x * blockDim.x) {
    float4 s = __ldcg(part + i);
    for (uint32_t q = 1; q < nparts; ++q) s = add4(s, __ldcg(part + (uint64_t)q * pstride4 + i));
    out[i] = s;
  }
}

}  // namespace

void sum_parts(const float* part, uint32_t nparts, uint64_t part_stride, uint64_t rows,
               uint64_t cols, uint64_t ldp, bool transpose, float* out, cudaStream_t st) {
  const uint64_t n = rows * cols;
  if (!n) return;
  const bool vec = cols % 4 == 0 && ldp % 4 == 0 && part_stride % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(part) & 15) == 0;
  if (vec && nparts <= 8 && !transpose && ldp == cols && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    const uint64_t n4 = n / 4;
    const unsigned blocks = (unsigned)std::min<uint64_t>(ceil_div(n4, (uint64_t)256), (uint64_t)num_sms() * 16);
    launch_pdl(sum_few_parts_kernel, blocks, 256, 0, st, reinterpret_cast<const float4*>(part),
               nparts, part_stride / 4, n4, reinterpret_cast<float4*>(out));
  } else if (vec)
    launch_pdl(sum_parts_kernel<true>, (unsigned)ceil_div(n, (uint64_t)128), RT, 0, st, part,
               nparts, part_stride, rows, cols, ldp, transpose ? 1 : 0, out);
  else
    launch_pdl(sum_parts_kernel<false>, (unsigned)ceil_div(n, (uint64_t)32), RT, 0, st, part,
               nparts, part_stride, rows, cols, ldp, transpose ? 1 : 0, out);
  MOE_LAUNCH_CHECK("sum_parts_kernel");
  count_launch();
}

void seg_colsum(uint32_t groups, const int32_t* gm, const int32_t* gb, uint32_t num_b, uint32_t N,
                uint32_t chunk, uint32_t maxch, const float* ws, float* out, cudaStream_t st) {
  arg_check(groups >= 1 && groups <= 1024, "colsum.groups: must be in [1, 1024]");
  if (!num_b || !N) return;
  const bool vec = N % 4 == 0 && (reinterpret_cast<uintptr_t>(ws) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (vec)
    launch_pdl(seg_colsum_kernel<true>, dim3(num_b, (unsigned)ceil_div((uint64_t)N, (uint64_t)128)),
               RT, 0, st, groups, gm, gb, N, chunk, maxch, ws, out);
  else
    launch_pdl(seg_colsum_kernel<false>, dim3(num_b, (unsigned)ceil_div((uint64_t)N, (uint64_t)32)),
               RT, 0, st, groups, gm, gb, N, chunk, maxch, ws, out);
  MOE_LAUNCH_CHECK("seg_colsum_kernel");
  count_launch();
}

}  // namespace moe
