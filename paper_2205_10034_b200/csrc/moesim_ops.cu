// Device implementations of the reference's data-plane functions on the path
// plus the synthetic-input generator.
//
//   gen_trace        workload.cpp:19-53   one SplitMix64 draw per token,
//                                         upper_bound into the Zipf CDF
//   imbalance_ratio  workload.cpp:55-66   max / mean expert total
//   alltoall_flat    collectives.cpp:10-21 out[i][j] = in[j][i]
//   fuse/split       collectives.cpp:88-118 concatenation + SliceIndex
//
// SplitMix64 is counter-based (state_i = seed + i*golden), so draw i of a
// substream is computed independently per thread and the device results are
// bit-identical to the reference's sequential loop (rng.hpp:19-42).
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace moe {

namespace {

__global__ void fill_uniform_kernel(void* out, uint64_t n, int dt, uint64_t seed, double lo,
                                    double span) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double u = (double)(splitmix64_at(seed, i) >> 11) * 0x1.0p-53;
    const float f = __double2float_rn(__dadd_rn(lo, __dmul_rn(span, u)));  // no FMA contraction
    if (dt == MOE_DTYPE_BF16) reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(f);
    else reinterpret_cast<float*>(out)[i] = f;
  }
}

__global__ void convert_kernel(const float* in, void* out, uint64_t n, int dt) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (dt == MOE_DTYPE_BF16) reinterpret_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(in[i]);
    else reinterpret_cast<float*>(out)[i] = in[i];
  }
}

__device__ __forceinline__ uint64_t substream(uint64_t seed, uint64_t step, uint64_t rank) {
  return seed ^ (0x9E3779B97F4A7C15ull * (step + 1)) ^ (0xC2B2AE3D27D4EB4Full * (rank + 1));
}

constexpr int TRACE_TOKENS_PER_THREAD = 16;
constexpr int TRACE_MAX_E = 4096;

// grid.x: token blocks; grid.y: step*ranks + rank
__global__ void gen_trace_kernel(uint64_t seed, uint32_t ranks, uint32_t E, uint64_t tokens,
                                 const double* __restrict__ cdf, unsigned long long* counts) {
  __shared__ unsigned int hist[TRACE_MAX_E];
  __shared__ double scdf[TRACE_MAX_E];
  for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
    hist[e] = 0;
    scdf[e] = cdf[e];
  }
  __syncthreads();
  const uint32_t sr = blockIdx.y;
  const uint64_t st = substream(seed, sr / ranks, sr % ranks);
  const uint64_t base = (uint64_t)blockIdx.x * blockDim.x * TRACE_TOKENS_PER_THREAD;
  for (int j = 0; j < TRACE_TOKENS_PER_THREAD; ++j) {
    const uint64_t t = base + (uint64_t)j * blockDim.x + threadIdx.x;
    if (t >= tokens) break;
    const double u = (double)(splitmix64_at(st, t) >> 11) * 0x1.0p-53;
    uint32_t lo = 0, hi = E;  // upper_bound
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (scdf[mid] > u) hi = mid; else lo = mid + 1;
    }
    atomicAdd(&hist[lo < E - 1 ? lo : E - 1], 1u);
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < E; e += blockDim.x)
    if (hist[e]) atomicAdd(counts + (uint64_t)sr * E + e, (unsigned long long)hist[e]);
}

// per-expert totals over [rows][E] counts, then max and sum (single block)
__global__ void imbalance_kernel(uint64_t rows, uint32_t E, const uint64_t* __restrict__ counts,
                                 unsigned long long* out /* [2]: max, total */) {
  __shared__ unsigned long long smax, ssum;
  if (threadIdx.x == 0) { smax = 0; ssum = 0; }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < E; e += blockDim.x) {
    unsigned long long t = 0;
    for (uint64_t r = 0; r < rows; ++r) t += counts[r * E + e];
    atomicMax(&smax, t);
    atomicAdd(&ssum, t);
  }
  __syncthreads();
  if (threadIdx.x == 0) { out[0] = smax; out[1] = ssum; }
}

__device__ void copy_bytes(uint8_t* dst, const uint8_t* src, uint64_t len) {
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  uint64_t done = 0;
  if (vec) {
    const uint64_t nv = len / 16;
    for (uint64_t i = threadIdx.x; i < nv; i += blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    done = nv * 16;
  }
  for (uint64_t i = done + threadIdx.x; i < len; i += blockDim.x) dst[i] = src[i];
}

// one block (x) per chunk (src, dst) -> out chunk (dst, src); y splits long chunks
__global__ void a2a_flat_kernel(uint64_t R, const uint64_t* __restrict__ lens,
                                const uint64_t* __restrict__ in_off, const uint8_t* __restrict__ in,
                                const uint64_t* __restrict__ out_off, uint8_t* __restrict__ out) {
  const uint64_t c = blockIdx.x;
  const uint64_t s = c / R, d = c % R;
  const uint64_t len = lens[c];
  const uint64_t part = (len + gridDim.y - 1) / gridDim.y;
  const uint64_t p0 = min(len, ((part + 15) / 16) * 16 * blockIdx.y);
  const uint64_t p1 = min(len, p0 + ((part + 15) / 16) * 16);
  if (p0 >= p1) return;
  copy_bytes(out + out_off[d * R + s] + p0, in + in_off[c] + p0, p1 - p0);
}

// generic chunk permutation: chunk i of `in` (in_off[i], len[i]) -> out at out_off[i]
__global__ void chunk_copy_kernel(const uint64_t* __restrict__ lens,
                                  const uint64_t* __restrict__ in_off, const uint8_t* __restrict__ in,
                                  const uint64_t* __restrict__ out_off, uint8_t* __restrict__ out) {
  const uint64_t c = blockIdx.x;
  const uint64_t len = lens[c];
  const uint64_t part = (len + gridDim.y - 1) / gridDim.y;
  const uint64_t p0 = min(len, ((part + 15) / 16) * 16 * blockIdx.y);
  const uint64_t p1 = min(len, p0 + ((part + 15) / 16) * 16);
  if (p0 >= p1) return;
  copy_bytes(out + out_off[c] + p0, in + in_off[c] + p0, p1 - p0);
}

__global__ void fuse_index_kernel(uint64_t n, const uint64_t* __restrict__ lens,
                                  moe_slice_index_entry_t* __restrict__ index) {
  if (threadIdx.x != 0) return;
  uint64_t off = 0;
  for (uint64_t i = 0; i < n; ++i) {
    index[i].slice_id = i;
    index[i].offset = off;
    index[i].length = lens[i];
    off += lens[i];
  }
}

__global__ void fuse_copy_kernel(const uint8_t* const* __restrict__ slices,
                                 const moe_slice_index_entry_t* __restrict__ index, uint8_t* blob) {
  const moe_slice_index_entry_t e = index[blockIdx.x];
  const uint64_t part = (e.length + gridDim.y - 1) / gridDim.y;
  const uint64_t step = ((part + 15) / 16) * 16;
  const uint64_t p0 = min(e.length, step * blockIdx.y), p1 = min(e.length, p0 + step);
  if (p0 < p1) copy_bytes(blob + e.offset + p0, slices[blockIdx.x] + p0, p1 - p0);
}

// collectives.cpp:101-110: 1 = not contiguous, 2 = does not cover the blob
__global__ void split_validate_kernel(uint64_t blob_len, uint64_t n,
                                      const moe_slice_index_entry_t* __restrict__ index, int32_t* bad) {
  if (threadIdx.x != 0) return;
  uint64_t expect = 0;
  int32_t b = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (index[i].offset != expect) { b = 1; break; }
    expect += index[i].length;
  }
  if (!b && expect != blob_len) b = 2;
  *bad = b;
}

__global__ void split_copy_kernel(const uint8_t* __restrict__ blob,
                                  const moe_slice_index_entry_t* __restrict__ index,
                                  uint8_t* const* __restrict__ out, const int32_t* __restrict__ bad) {
  if (*bad) return;
  const moe_slice_index_entry_t e = index[blockIdx.x];
  const uint64_t part = (e.length + gridDim.y - 1) / gridDim.y;
  const uint64_t step = ((part + 15) / 16) * 16;
  const uint64_t p0 = min(e.length, step * blockIdx.y), p1 = min(e.length, p0 + step);
  if (p0 < p1) copy_bytes(out[blockIdx.x] + p0, blob + e.offset + p0, p1 - p0);
}

unsigned grid_for(uint64_t n) { return (unsigned)std::min<uint64_t>(ceil_div(n, 256), 148ull * 16); }

}  // namespace

void fill_uniform(void* out, uint64_t n, moe_dtype_t dt, uint64_t seed, double lo, double hi,
                  cudaStream_t st) {
  if (!n) return;
  fill_uniform_kernel<<<grid_for(n), 256, 0, st>>>(out, n, (int)dt, seed, lo, hi - lo);
  MOE_LAUNCH_CHECK("fill_uniform_kernel");
  count_launch();
}

void convert_f32_to(const float* in, void* out, uint64_t n, moe_dtype_t dt, cudaStream_t st) {
  if (!n) return;
  convert_kernel<<<grid_for(n), 256, 0, st>>>(in, out, n, (int)dt);
  MOE_LAUNCH_CHECK("convert_kernel");
  count_launch();
}

void gen_trace_device(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                      uint64_t tokens, double skew, uint64_t* counts, cudaStream_t st) {
  config_check(experts != 0, "workload.experts: must be >= 1");
  config_check(!(skew < 0.0), "workload.skew: must be >= 0");
  config_check(experts <= (uint32_t)TRACE_MAX_E, "workload.experts: must be <= 4096 on the device");
  // Cumulative expert weights, shared by all substreams (workload.cpp:32-39);
  // computed on the host with the same std::pow so the CDF is bit-identical.
  std::vector<double> cdf(experts);
  double acc = 0.0;
  for (uint32_t e = 0; e < experts; ++e) {
    acc += std::pow(static_cast<double>(e + 1), -skew);
    cdf[e] = acc;
  }
  for (uint32_t e = 0; e < experts; ++e) cdf[e] /= acc;
  cdf[experts - 1] = 1.0;
  const uint64_t n = (uint64_t)steps * ranks * experts;
  if (n) MOE_CUDA(cudaMemsetAsync(counts, 0, n * sizeof(uint64_t), st));
  if (!n || !tokens) return;
  double* dcdf = nullptr;
  MOE_CUDA(cudaMallocAsync(&dcdf, experts * sizeof(double), st));
  MOE_CUDA(cudaMemcpyAsync(dcdf, cdf.data(), experts * sizeof(double), cudaMemcpyHostToDevice, st));
  const uint64_t per_block = 256ull * TRACE_TOKENS_PER_THREAD;
  dim3 grid((unsigned)ceil_div(tokens, per_block), steps * ranks);
  gen_trace_kernel<<<grid, 256, 0, st>>>(seed, ranks, experts, tokens, dcdf,
                                         reinterpret_cast<unsigned long long*>(counts));
  MOE_LAUNCH_CHECK("gen_trace_kernel");
  count_launch();
  MOE_CUDA(cudaFreeAsync(dcdf, st));
}

void imbalance_device(uint64_t rows, uint32_t experts, const uint64_t* counts,
                      unsigned long long* out2, cudaStream_t st) {
  imbalance_kernel<<<1, 256, 0, st>>>(rows, experts, counts, out2);
  MOE_LAUNCH_CHECK("imbalance_kernel");
  count_launch();
}

void alltoall_flat_device(uint64_t R, const uint64_t* lens, const uint64_t* in_off,
                          const uint8_t* in, const uint64_t* out_off, uint8_t* out,
                          uint64_t max_len, cudaStream_t st) {
  if (!R) return;
  const unsigned split = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(max_len, 1 << 20), 64));
  dim3 grid((unsigned)(R * R), split);
  a2a_flat_kernel<<<grid, 256, 0, st>>>(R, lens, in_off, in, out_off, out);
  MOE_LAUNCH_CHECK("a2a_flat_kernel");
  count_launch();
}

void copy_chunks_device(uint64_t n, const uint64_t* lens, const uint64_t* in_off,
                        const uint8_t* in, const uint64_t* out_off, uint8_t* out, uint64_t max_len,
                        cudaStream_t st) {
  if (!n) return;
  const unsigned split = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(max_len, 1 << 20), 64));
  dim3 grid((unsigned)n, split);
  chunk_copy_kernel<<<grid, 256, 0, st>>>(lens, in_off, in, out_off, out);
  MOE_LAUNCH_CHECK("chunk_copy_kernel");
  count_launch();
}

void fuse_slices_device(uint64_t n, const uint8_t* const* slices, const uint64_t* lens,
                        uint8_t* blob, moe_slice_index_entry_t* index, uint64_t max_len,
                        cudaStream_t st) {
  fuse_index_kernel<<<1, 32, 0, st>>>(n, lens, index);
  MOE_LAUNCH_CHECK("fuse_index_kernel");
  const unsigned split = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(max_len, 1 << 20), 64));
  fuse_copy_kernel<<<dim3((unsigned)n, split), 256, 0, st>>>(slices, index, blob);
  MOE_LAUNCH_CHECK("fuse_copy_kernel");
  count_launch(2);
}

void split_blob_device(uint64_t blob_len, const uint8_t* blob, uint64_t n,
                       const moe_slice_index_entry_t* index, uint8_t* const* out, int32_t* bad,
                       uint64_t max_len, cudaStream_t st) {
  split_validate_kernel<<<1, 32, 0, st>>>(blob_len, n, index, bad);
  MOE_LAUNCH_CHECK("split_validate_kernel");
  count_launch();
  if (!n) return;
  const unsigned split = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(max_len, 1 << 20), 64));
  split_copy_kernel<<<dim3((unsigned)n, split), 256, 0, st>>>(blob, index, out, bad);
  MOE_LAUNCH_CHECK("split_copy_kernel");
  count_launch();
}

}  // namespace moe
