// K2 (gating: softmax, top-k, capacity scan, aux loss, histograms), K3
// (dispatch), K6 (combine) and their backward passes.
//
// Semantics: DESIGN.md Appendix A (builder-owned; the reference has no gating —
// SPEC.md:15,153,156).  Integer outputs (experts, positions, drops, counts) are
// bit-exact against oracle/moe_oracle.c:oracle_route given identical logits:
// selection compares fp32 logits (never exp'd values), ties go to the lowest
// expert, NaN reads as -inf, and positions come from an order-preserving scan
// (warp match + per-warp histograms inside a 256-token chunk, then a per-expert
// scan over chunks) so the token order of Appendix A §6 is kept exactly.
//
// The reference's only "routing" is the count sampler gen_trace
// (workload.cpp:19-53); the dataflow of dispatch/combine mirrors its
// embed_forward/backward route->exchange->reassemble pattern
// (embed_partition.cpp:58-169), with experts in place of shard owners.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace moe {

namespace {

// tokens per routing block (a thread per token); A/B on c2: 128-token blocks
// (4 per SM instead of 2) are slower, 27.5 vs 24.5 us forward, 30.8 vs 28.7 backward
#ifndef MOE_ROUTE_CHUNK
#define MOE_ROUTE_CHUNK 256
#endif
constexpr int CHUNK = MOE_ROUTE_CHUNK;
constexpr int RT_THREADS = CHUNK;
constexpr int NW = RT_THREADS / 32;  // warps per routing block
constexpr int MAX_E = 256;
constexpr int SLAB = 64;        // experts per shared-memory slab of logits
constexpr int TS = SLAB + 1;    // padded row stride (floats): row and column reads conflict-free
constexpr int SLAB_SMEM = CHUNK * TS * 4;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float nan_to_ninf(float v) { return isnan(v) ? -INFINITY : v; }

// Stage logits[t0, t0 + CHUNK) x [e0, e0 + ne) into tile[CHUNK][TS] (NaN read
// as -inf, missing rows/columns -inf): each warp instruction reads 128
// contiguous bytes of one row, so the thread-per-token passes below read
// shared memory instead of issuing 32-row-wide scattered global loads.
__device__ __forceinline__ void load_slab(const float* __restrict__ logits, uint64_t t0, uint64_t T,
                                          int E, int e0, int ne, float* tile) {
  const int tid = threadIdx.x;
  if ((E & 3) == 0) {
    // all 16 float4 loads of a thread in flight before the first store; a
    // warp instruction covers two 256-byte row pieces
    constexpr int Q = SLAB / 4;
    constexpr int PER = CHUNK * Q / RT_THREADS;
    float4 v[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int x = i * RT_THREADS + tid, r = x / Q, q = x % Q;
      const uint64_t t = t0 + r;
      v[i] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
      if (t < T && 4 * q < ne) v[i] = __ldg(reinterpret_cast<const float4*>(logits + t * E + e0) + q);
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int x = i * RT_THREADS + tid, r = x / Q, q = x % Q;
      float* d = tile + r * TS + 4 * q;
      d[0] = nan_to_ninf(v[i].x);
      d[1] = nan_to_ninf(v[i].y);
      d[2] = nan_to_ninf(v[i].z);
      d[3] = nan_to_ninf(v[i].w);
    }
    return;
  }
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll 4
  for (int r = warp; r < CHUNK; r += RT_THREADS / 32) {
    const uint64_t t = t0 + r;
    const float* L = logits + t * E + e0;
#pragma unroll
    for (int j = lane; j < SLAB; j += 32) {
      float v = -INFINITY;
      if (t < T && j < ne) v = nan_to_ninf(__ldg(L + j));
      tile[r * TS + j] = v;
    }
  }
}

// exp(x) as one FMUL + MUFU.EX2 (against libdevice expf's ~10 instructions);
// exp(-inf) = 0, NaN stays NaN.  Relative error: ex2.approx's ~2^-22 plus the
// rounding of x * log2(e), ~|x| * log2(e) * 2^-24 (about 1e-6 at x = -20,
// 5e-6 at x = -80), and .ftz flushes results below 2^-126 to zero -- only
// the softmax normaliser and the aux-loss column sums use it, where those
// terms are negligible tails.  The top-2 gates (the compared outputs) use the
// precise expf of l2 - l1 and do not depend on the normaliser.
__device__ __forceinline__ float exp_f(float x) { return ex2_approx(x * 1.44269504088896341f); }

// Phase A: thread per token (the block is one 256-token chunk): top-k on the
// fp32 logits, softmax, gates; per chunk: histograms (expert-major
// [i][E][nchunks]), in-chunk ranks (warp match over 32 consecutive tokens +
// per-warp histograms), and softmax column partial sums reduced in a fixed
// order (deterministic aux loss), written expert-major [E][nchunks].
__global__ void __launch_bounds__(RT_THREADS) route_topk_kernel(
    uint64_t T, int E, int k, const float* __restrict__ logits, int32_t* __restrict__ expert,
    float* __restrict__ gate, int32_t* __restrict__ rank_local, int32_t* __restrict__ chunk_cnt,
    float* __restrict__ psum_part, uint64_t nchunks) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float tile[];  // [CHUNK][TS]
  __shared__ int hist[2][NW][MAX_E];
  __shared__ float pw[NW][MAX_E];
  __shared__ float mrow[CHUNK], irow[CHUNK];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const uint64_t chunk = blockIdx.x;
  const uint64_t t0 = chunk * CHUNK;
  const uint64_t t = t0 + tid;
  const bool valid = t < T;
  const int nslab = (E + SLAB - 1) / SLAB;

  for (int i = tid; i < 2 * NW * MAX_E; i += RT_THREADS) (&hist[0][0][0])[i] = 0;

  // pass 1: top-1 / top-2 on logits (NaN read as -inf, ties to the lowest index)
  float v1 = -INFINITY, v2 = -INFINITY;
  int i1 = 0x7fffffff, i2 = 0x7fffffff;
  for (int sl = 0; sl < nslab; ++sl) {
    const int e0 = sl * SLAB, ne = min(SLAB, E - e0);
    __syncthreads();
    load_slab(logits, t0, T, E, e0, ne, tile);
    __syncthreads();
    if (valid) {
      // experts arrive in index order, so a tie can only displace the
      // sentinel: (v > v1 || (v == v1 && e < i1)) == (v > v1 || i1 unset).
      // Branchless selects instead of the divergent if / else-if chain.
      const float* row = tile + tid * TS;
#pragma unroll 4
      for (int j = 0; j < ne; ++j) {
        const float v = row[j];
        const int e = e0 + j;
        const bool c1 = v > v1 || i1 == 0x7fffffff;
        const bool c2 = !c1 && (v > v2 || i2 == 0x7fffffff);
        const float nv2 = c1 ? v1 : v;
        const int ni2 = c1 ? i1 : e;
        v2 = (c1 || c2) ? nv2 : v2;
        i2 = (c1 || c2) ? ni2 : i2;
        v1 = c1 ? v : v1;
        i1 = c1 ? e : i1;
      }
    }
  }
  // pass 2: softmax denominator (max = v1), experts in index order
  float z = 0.f;
  for (int sl = 0; sl < nslab; ++sl) {
    const int e0 = sl * SLAB, ne = min(SLAB, E - e0);
    if (nslab > 1) {
      __syncthreads();
      load_slab(logits, t0, T, E, e0, ne, tile);
      __syncthreads();
    }
    if (valid) {  // one slab: keep exp(l - max) in the tile for pass 3
      float* row = tile + tid * TS;
      for (int j = 0; j < ne; ++j) {
        const float ex = exp_f(row[j] - v1);
        if (nslab == 1) row[j] = ex;
        z += ex;
      }
    }
  }
  const float inv = valid ? 1.0f / z : 0.f;
  if (valid) {
    if (k == 1) {
      expert[t] = i1;
      gate[t] = inv;  // p[e1] = exp(0) / z
    } else {
      const float p2 = expf(v2 - v1);
      const float sden = 1.0f + p2;
      expert[2 * t] = i1;
      expert[2 * t + 1] = i2;
      gate[2 * t] = 1.0f / sden;
      gate[2 * t + 1] = p2 / sden;
    }
  }
  mrow[tid] = v1;
  irow[tid] = inv;
  // pass 3: softmax column sums over the warp's 32 tokens (lane = expert
  // column), then a fixed-order sum over the 8 warps (deterministic aux)
  for (int sl = 0; sl < nslab; ++sl) {
    const int e0 = sl * SLAB, ne = min(SLAB, E - e0);
    __syncthreads();
    if (nslab > 1) {
      load_slab(logits, t0, T, E, e0, ne, tile);
      __syncthreads();
    }
    float acc[SLAB / 32];
#pragma unroll
    for (int q = 0; q < SLAB / 32; ++q) acc[q] = 0.f;
    for (int j = 0; j < 32; ++j) {
      const int r = warp * 32 + j;
      if (t0 + r >= T) break;
      const float mj = mrow[r], ij = irow[r];
#pragma unroll
      for (int q = 0; q < SLAB / 32; ++q) {
        const float tv = tile[r * TS + lane + 32 * q];
        acc[q] += (nslab == 1 ? tv : exp_f(tv - mj)) * ij;
      }
    }
#pragma unroll
    for (int q = 0; q < SLAB / 32; ++q)
      if (lane + 32 * q < ne) pw[warp][e0 + lane + 32 * q] = acc[q];
  }
  __syncthreads();
  // in-chunk ranks: thread = token, warp = 32 consecutive tokens in order
  int ech[2] = {valid ? i1 : -1, (valid && k == 2) ? i2 : -1};
  int r_in[2] = {0, 0};
  for (int i = 0; i < k; ++i) {
    const int e = ech[i];
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const unsigned lt = (1u << lane) - 1u;
    r_in[i] = __popc(peers & lt);
    if (e >= 0 && (peers & lt) == 0) hist[i][warp][e] = __popc(peers);
  }
  __syncthreads();
  for (int x = tid; x < k * E; x += RT_THREADS) {
    const int i = x / E, e = x % E;
    int run = 0;
    for (int w = 0; w < NW; ++w) {
      const int c = hist[i][w][e];
      hist[i][w][e] = run;
      run += c;
    }
    chunk_cnt[((uint64_t)i * E + e) * nchunks + chunk] = run;
  }
  for (int e = tid; e < E; e += RT_THREADS) {
    float sp = 0.f;
    for (int w = 0; w < NW; ++w) sp += pw[w][e];
    psum_part[(uint64_t)e * nchunks + chunk] = sp;
  }
  __syncthreads();
  if (valid) {
    for (int i = 0; i < k; ++i) rank_local[t * k + i] = hist[i][warp][ech[i]] + r_in[i];
  }
}

// Exclusive scan of one expert's chunk counts by one warp: lane l owns the
// contiguous chunk range [l*per, (l+1)*per); all loads of a pass are
// independent.  Returns the total.
__device__ __forceinline__ int warp_chunk_scan(const int32_t* __restrict__ cc,
                                               int32_t* __restrict__ co, uint64_t nchunks,
                                               int base) {
  const int lane = threadIdx.x & 31;
  const uint64_t per = (nchunks + 31) / 32;
  const uint64_t c0 = lane * per, c1 = min(nchunks, c0 + per);
  int mine = 0;
  for (uint64_t c = c0; c < c1; ++c) mine += cc[c];
  int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  int run = base + incl - mine;
  for (uint64_t c = c0; c < c1; ++c) {
    const int v = cc[c];
    co[c] = run;
    run += v;
  }
  return base + __shfl_sync(0xffffffffu, incl, 31);
}

// Phase B: per-expert exclusive scan over chunks (one warp per expert),
// counts, kept, per-expert softmax mass (fixed-order sum).
__global__ void __launch_bounds__(256) route_scan_kernel(
    uint64_t T, int E, int k, uint64_t C, const int32_t* __restrict__ chunk_cnt,
    int32_t* __restrict__ chunk_off, const float* __restrict__ psum_part, uint64_t nchunks,
    int32_t* __restrict__ count1, int32_t* __restrict__ count2, int32_t* __restrict__ kept,
    float* __restrict__ psum_e) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (e >= E) return;
  const int c1 = warp_chunk_scan(chunk_cnt + (uint64_t)e * nchunks,
                                 chunk_off + (uint64_t)e * nchunks, nchunks, 0);
  int c2 = 0;
  if (k == 2)  // top-2 positions start after all (pre-drop) top-1 tokens
    c2 = warp_chunk_scan(chunk_cnt + ((uint64_t)E + e) * nchunks,
                         chunk_off + ((uint64_t)E + e) * nchunks, nchunks, c1) - c1;
  const uint64_t per = (nchunks + 31) / 32;
  const uint64_t q0 = lane * per, q1 = min(nchunks, q0 + per);
  float ps = 0.f;
  for (uint64_t c = q0; c < q1; ++c) ps += psum_part[(uint64_t)e * nchunks + c];
  ps = warp_sum(ps);
  if (lane == 0) {
    count1[e] = c1;
    count2[e] = c2;
    const uint64_t tot = (uint64_t)c1 + (uint64_t)c2;
    kept[e] = (int32_t)(tot < C ? tot : C);
    psum_e[e] = ps;
  }
}

// Phase C: positions and keep flags; block 0 / warp 0 also forms the aux loss
// E * sum_e (psum_e / T) (count1_e / T) in a fixed order.
__global__ void route_finalize_kernel(uint64_t T, int E, int k, uint64_t C, uint64_t nchunks,
                                      const int32_t* __restrict__ expert,
                                      const int32_t* __restrict__ rank_local,
                                      const int32_t* __restrict__ chunk_off,
                                      int32_t* __restrict__ position, uint8_t* __restrict__ keep,
                                      const float* __restrict__ psum_e,
                                      const int32_t* __restrict__ count1, float* __restrict__ aux) {
  pdl_wait();
  pdl_trigger();
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    const double invT = T ? 1.0 / (double)T : 0.0;
    double a = 0.0;
    for (int e = threadIdx.x; e < E; e += 32)
      a += ((double)psum_e[e] * invT) * ((double)count1[e] * invT);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x == 0) aux[0] = (float)((double)E * a);
  }
  const uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= T * k) return;
  const uint64_t t = x / k;
  const int i = (int)(x % k);
  const int e = expert[x];
  const uint64_t chunk = t / CHUNK;
  const int p = chunk_off[((uint64_t)i * E + e) * nchunks + chunk] + rank_local[x];
  position[x] = p;
  if (keep) keep[x] = (uint64_t)p < C ? 1 : 0;
}

}  // namespace

uint64_t route_chunks(uint64_t T) { return (T + CHUNK - 1) / CHUNK; }

void route_forward(uint64_t T, uint32_t E, uint32_t k, uint64_t C, const float* logits,
                   const moe_routing_out_t& out, const RouteWorkspace& ws, cudaStream_t st) {
  config_check(E >= 1 && E <= (uint32_t)MAX_E, "routing.experts: must be in [1, 256]");
  config_check(k == 1 || k == 2, "routing.top_k: must be 1 or 2");
  config_check(k == 1 || E >= 2, "routing.experts: top-2 needs >= 2 experts");
  if (T == 0) {
    MOE_CUDA(cudaMemsetAsync(out.count1, 0, sizeof(int32_t) * E, st));
    MOE_CUDA(cudaMemsetAsync(out.count2, 0, sizeof(int32_t) * E, st));
    MOE_CUDA(cudaMemsetAsync(out.kept, 0, sizeof(int32_t) * E, st));
    MOE_CUDA(cudaMemsetAsync(out.aux_loss, 0, sizeof(float), st));
    return;
  }
  MOE_CUDA(cudaFuncSetAttribute(route_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                SLAB_SMEM));
  const uint64_t nch = route_chunks(T);
  float* psum_e = ws.psum_part + nch * E;
  launch_pdl(route_topk_kernel, (unsigned)nch, RT_THREADS, SLAB_SMEM, st, 
      T, (int)E, (int)k, logits, out.expert, out.gate, ws.rank_local, ws.chunk_cnt, ws.psum_part,
      nch);
  MOE_LAUNCH_CHECK("route_topk_kernel");
  launch_pdl(route_scan_kernel, (E + 7) / 8, 256, 0, st, T, (int)E, (int)k, C, ws.chunk_cnt, ws.chunk_off,
                                                 ws.psum_part, nch, out.count1, out.count2,
                                                 out.kept, psum_e);
  MOE_LAUNCH_CHECK("route_scan_kernel");
  const uint64_t n = T * k;
  launch_pdl(route_finalize_kernel, (unsigned)((n + 255) / 256), 256, 0, st, 
      T, (int)E, (int)k, C, nch, out.expert, ws.rank_local, ws.chunk_off, out.position, out.keep,
      psum_e, out.count1, out.aux_loss);
  MOE_LAUNCH_CHECK("route_finalize_kernel");
  count_launch(3);
}

// ---------------------------------------------------------------- K3 -------
namespace {

// Row copy helpers: a row of d elements of type dt viewed as 16B vectors.
template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
};

// Zero rows [kept_e, round_up(kept_e, pad)) of expert e's slot region (the
// weight-gradient GEMM runs whole K blocks); block-strided over experts.
template <typename T>
__device__ __forceinline__ void zero_pad_rows(int d, int E, uint64_t Cs, uint32_t pad,
                                              const int32_t* __restrict__ kept, T* __restrict__ buf) {
  if (pad <= 1) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nv = d / Vec<T>::N;
  for (int e = blockIdx.x; e < E; e += gridDim.x) {
    const int n = kept[e];
    const int end = (int)min((uint64_t)((n + pad - 1) / pad) * pad, Cs);
    for (int r = n + warp; r < end; r += nw) {
      uint4* row = reinterpret_cast<uint4*>(buf + ((uint64_t)e * Cs + r) * d);
      for (int v = lane; v < nv; v += 32) row[v] = make_uint4(0, 0, 0, 0);
    }
  }
}

template <typename T>
__global__ void dispatch_kernel(uint64_t T_, int d, int E, int k, uint64_t Cs, uint64_t C,
                                const T* __restrict__ x, const int32_t* __restrict__ expert,
                                const int32_t* __restrict__ position, T* __restrict__ buf,
                                int32_t* __restrict__ slot, uint32_t pad,
                                const int32_t* __restrict__ kept) {
  pdl_wait();
  pdl_trigger();
  zero_pad_rows(d, E, Cs, pad, kept, buf);
  const int lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T_;
       t += nwarps) {
    int64_t dst[2] = {-1, -1};
    for (int i = 0; i < k; ++i) {
      const int e = expert[t * k + i];
      const int p = position[t * k + i];
      const int64_t s = ((uint64_t)p < C) ? (int64_t)e * (int64_t)Cs + p : -1;
      dst[i] = s;
      if (lane == 0) slot[t * k + i] = (int32_t)s;
    }
    if (dst[0] < 0 && dst[1] < 0) continue;
    const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
    const int nv = d / Vec<T>::N;
    constexpr int B = 4;  // 16-byte pieces per lane in flight
    for (int v0 = 0; v0 < nv; v0 += 32 * B) {
      uint4 val[B];
#pragma unroll
      for (int q = 0; q < B; ++q)
        if (v0 + lane + 32 * q < nv) val[q] = __ldg(src + v0 + lane + 32 * q);
#pragma unroll
      for (int q = 0; q < B; ++q) {
        const int v = v0 + lane + 32 * q;
        if (v >= nv) continue;
        for (int i = 0; i < k; ++i)
          if (dst[i] >= 0) reinterpret_cast<uint4*>(buf + dst[i] * d)[v] = val[q];
      }
    }
  }
}

// Zero rows [kept_e, round_up(kept_e, pad)) of each expert slot: one block per
// expert, rows strided over warps.
template <typename T>
__global__ void zero_pad_kernel(int d, uint64_t Cs, uint32_t pad, const int32_t* __restrict__ kept,
                                T* __restrict__ buf) {
  pdl_wait();
  pdl_trigger();
  const int e = blockIdx.x;
  const int n = kept[e];
  const int end = (int)min((uint64_t)((n + pad - 1) / pad) * pad, Cs);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int nv = d / Vec<T>::N;
  for (int r = n + warp; r < end; r += nw) {
    uint4* row = reinterpret_cast<uint4*>(buf + ((uint64_t)e * Cs + r) * d);
    for (int v = lane; v < nv; v += 32) row[v] = make_uint4(0, 0, 0, 0);
  }
}

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&f)[8]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(h[i]);
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&f)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
template <typename T>
__device__ __forceinline__ void store8(T* p, const float (&f)[8]);
template <>
__device__ __forceinline__ void store8<__nv_bfloat16>(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 o;
  o.x = pack_bf16x2(f[0], f[1]);
  o.y = pack_bf16x2(f[2], f[3]);
  o.z = pack_bf16x2(f[4], f[5]);
  o.w = pack_bf16x2(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = o;
}
template <>
__device__ __forceinline__ void store8<float>(float* p, const float (&f)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}

// y[t] = sum_i g_i Y[slot_i]; one warp per token, 8 elements per lane step.
template <typename T>
__global__ void combine_kernel(uint64_t T_, int d, int k, const T* __restrict__ Y,
                               const int32_t* __restrict__ slot, const float* __restrict__ gate,
                               T* __restrict__ y) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T_) return;
  int32_t s[2] = {-1, -1};
  float g[2] = {0.f, 0.f};
  for (int i = 0; i < k; ++i) {
    s[i] = slot[t * k + i];
    g[i] = gate[t * k + i];
  }
  for (int c = lane * 8; c < d; c += 256) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < k; ++i) {
      if (s[i] < 0) continue;
      float f[8];
      load8<T>(Y + (uint64_t)s[i] * d + c, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = fmaf(g[i], f[q], acc[q]);
    }
    store8<T>(y + t * d + c, acc);
  }
}

// dgate[t,i] = <dy_t, Y[slot_i]>, dY[slot_i] = g_i dy_t.
template <typename T>
__global__ void combine_bwd_kernel(uint64_t T_, int d, int k, const T* __restrict__ dy,
                                   const T* __restrict__ Y, const int32_t* __restrict__ slot,
                                   const float* __restrict__ gate, T* __restrict__ dY,
                                   float* __restrict__ dgate, int E, uint64_t Cs, uint32_t pad,
                                   const int32_t* __restrict__ kept) {
  pdl_wait();
  pdl_trigger();
  zero_pad_rows(d, E, Cs, pad, kept, dY);
  const int lane = threadIdx.x & 31;
  const uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T_) return;
  for (int i = 0; i < k; ++i) {
    const int32_t s = slot[t * k + i];
    if (s < 0) {
      if (lane == 0) dgate[t * k + i] = 0.f;
      continue;
    }
    const float g = gate[t * k + i];
    float dot = 0.f;
    for (int c = lane * 8; c < d; c += 256) {
      float a[8], b[8], o[8];
      load8<T>(dy + t * d + c, a);
      load8<T>(Y + (uint64_t)s * d + c, b);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        dot = fmaf(a[q], b[q], dot);
        o[q] = g * a[q];
      }
      store8<T>(dY + (uint64_t)s * d + c, o);
    }
    dot = warp_sum(dot);
    if (lane == 0) dgate[t * k + i] = dot;
  }
}

template <typename T>
__global__ void gather_dx_kernel(uint64_t T_, int d, int k, const T* __restrict__ dXe,
                                 const int32_t* __restrict__ slot, const float* __restrict__ dxg,
                                 T* __restrict__ dx) {
  pdl_wait();
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T_) return;
  int32_t s[2] = {-1, -1};
  for (int i = 0; i < k; ++i) s[i] = slot[t * k + i];
  for (int c = lane * 8; c < d; c += 256) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (dxg) {
      const float4 a = *reinterpret_cast<const float4*>(dxg + t * d + c);
      const float4 b = *reinterpret_cast<const float4*>(dxg + t * d + c + 4);
      acc[0] = a.x; acc[1] = a.y; acc[2] = a.z; acc[3] = a.w;
      acc[4] = b.x; acc[5] = b.y; acc[6] = b.z; acc[7] = b.w;
    }
    for (int i = 0; i < k; ++i) {
      if (s[i] < 0) continue;
      float f[8];
      load8<T>(dXe + (uint64_t)s[i] * d + c, f);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += f[q];
    }
    store8<T>(dx + t * d + c, acc);
  }
}

// Routing backward (DESIGN.md Appendix A §9), thread per token on a staged
// 256-token slab of logits: recompute the softmax, add the aux-loss term and
// the gate term, put the dlogits row back into the slab, then write the slab
// out row-coalesced (fp32 and/or the bf16 GEMM operand, pad columns zero) and
// reduce its columns into the gate-bias gradient.
template <typename LP>
__global__ void __launch_bounds__(RT_THREADS) route_bwd_kernel(
    uint64_t T_, int E, int k, const float* __restrict__ logits,
    const int32_t* __restrict__ expert, const float* __restrict__ gate,
    const uint8_t* __restrict__ keep, const int32_t* __restrict__ count1,
    const float* __restrict__ dgate, float d_aux, float* __restrict__ dl_f32,
    LP* __restrict__ dl_lp, int ld, float* __restrict__ dbg) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float tile[];  // [CHUNK][TS]
  __shared__ float a_s[MAX_E];
  __shared__ float cs[NW][SLAB];
  const float invT = 1.0f / (float)T_;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  for (int e = tid; e < E; e += blockDim.x) a_s[e] = (float)E * (float)count1[e] * invT * invT;
  const uint64_t t0 = (uint64_t)blockIdx.x * CHUNK;
  const uint64_t t = t0 + tid;
  const bool valid = t < T_;
  const int nslab = (E + SLAB - 1) / SLAB;
  float m = -INFINITY, z = 0.f, pnum = 0.f;
  for (int sl = 0; sl < nslab; ++sl) {
    const int e0 = sl * SLAB, ne = min(SLAB, E - e0);
    __syncthreads();
    load_slab(logits, t0, T_, E, e0, ne, tile);
    __syncthreads();
    if (valid)
      for (int j = 0; j < ne; ++j) m = fmaxf(m, tile[tid * TS + j]);
  }
  for (int sl = 0; sl < nslab; ++sl) {
    const int e0 = sl * SLAB, ne = min(SLAB, E - e0);
    if (nslab > 1) {
      __syncthreads();
      load_slab(logits, t0, T_, E, e0, ne, tile);
      __syncthreads();
    }
    if (valid)  // one slab: keep exp(l - max) in the tile for the next pass
      for (int j = 0; j < ne; ++j) {
        const float ex = exp_f(tile[tid * TS + j] - m);
        if (nslab == 1) tile[tid * TS + j] = ex;
        z += ex;
        pnum = fmaf(ex, a_s[e0 + j], pnum);
      }
  }
  const float inv = valid ? 1.0f / z : 0.f;
  const float pa = pnum * inv;
  int e1 = -1, e2 = -1;
  float gterm = 0.f, p1 = 0.f;
  if (valid) {
    e1 = expert[t * k];
    const float dg1 = keep[t * k] ? dgate[t * k] : 0.f;
    if (k == 2) {
      e2 = expert[t * k + 1];
      const float dg2 = keep[t * k + 1] ? dgate[t * k + 1] : 0.f;
      gterm = (dg1 - dg2) * gate[t * k] * gate[t * k + 1];  // +/- on e1/e2
    } else {
      gterm = dg1;
      p1 = gate[t];  // = p[e1]
    }
  }
  for (int sl = 0; sl < nslab; ++sl) {
    const int e0 = sl * SLAB, ne = min(SLAB, E - e0);
    if (nslab > 1) {
      __syncthreads();
      load_slab(logits, t0, T_, E, e0, ne, tile);
      __syncthreads();
    }
    // own row: logits -> dlogits in place (invalid rows -> 0)
    for (int j = 0; j < ne; ++j) {
      const int e = e0 + j;
      float v = 0.f;
      if (valid) {
        const float tv = tile[tid * TS + j];
        const float pe = (nslab == 1 ? tv : exp_f(tv - m)) * inv;
        v = d_aux * pe * (a_s[e] - pa);
        if (k == 1) v += gterm * p1 * ((e == e1 ? 1.f : 0.f) - pe);
        else v += (e == e1 ? gterm : 0.f) - (e == e2 ? gterm : 0.f);
      }
      tile[tid * TS + j] = v;
    }
    __syncthreads();
    // row-coalesced write-out; the last slab also zeroes pad columns [E, ld)
    const int wl = (sl == nslab - 1 && dl_lp) ? max(ne, ld - e0) : ne;
    for (int r = warp; r < CHUNK; r += RT_THREADS / 32) {
      const uint64_t tr = t0 + r;
      if (tr >= T_) break;
      for (int j = lane; j < wl; j += 32) {
        const float v = j < ne ? tile[r * TS + j] : 0.f;
        if (dl_f32 && j < ne) dl_f32[tr * E + e0 + j] = v;
        if (dl_lp) dl_lp[tr * ld + e0 + j] = (LP)v;
      }
    }
    if (dbg) {
      // column sums: warp w over its 32 rows, then a fixed order over warps
#pragma unroll
      for (int q = 0; q < SLAB / 32; ++q) {
        float a = 0.f;
        for (int j = 0; j < 32; ++j) a += tile[(warp * 32 + j) * TS + lane + 32 * q];
        cs[warp][lane + 32 * q] = a;
      }
      __syncthreads();
      if (tid < ne) {  // this block's partial row; summed over blocks in order (sum_parts)
        float a = 0.f;
        for (int w = 0; w < NW; ++w) a += cs[w][tid];
        dbg[(uint64_t)blockIdx.x * E + e0 + tid] = a;
      }
    }
  }
}

template <typename T>
__global__ void colsum_kernel(const int32_t* __restrict__ gm, const int32_t* __restrict__ ga,
                              const int32_t* __restrict__ gb, int N, const T* __restrict__ X,
                              float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x;
  const int rows = gm[g];
  constexpr int CH = 32;  // rows per block (partials reduced by seg_colsum)
  const int r0 = blockIdx.y * CH;
  if (r0 >= rows) return;
  const int n = blockIdx.z * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int r1 = min(rows, r0 + CH);
  const T* base = X + ((uint64_t)ga[g] + r0) * N + n;
  float s = 0.f;
  for (int r = r0; r < r1; ++r, base += N) s += (float)*base;
  out[((uint64_t)g * gridDim.y + blockIdx.y) * N + n] = s;  // chunk partial (seg_colsum)
}

// bf16, 8 columns per thread (16-byte loads), 64 rows per block, 8 rows in flight
__global__ void colsum_bf16x8_kernel(const int32_t* __restrict__ gm, const int32_t* __restrict__ ga,
                                     const int32_t* __restrict__ gb, int N,
                                     const __nv_bfloat16* __restrict__ X, float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int g = blockIdx.x;
  const int rows = gm[g];
  const int r0 = blockIdx.y * 64;
  if (r0 >= rows) return;
  const int n = (blockIdx.z * blockDim.x + threadIdx.x) * 8;
  if (n >= N) return;
  const int r1 = min(rows, r0 + 64);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const __nv_bfloat16* base = X + ((uint64_t)ga[g] + r0) * N + n;
  int r = r0;
  for (; r + 8 <= r1; r += 8, base += 8 * (uint64_t)N) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)u * N));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v[u]);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] += __bfloat162float(h[q]);
    }
  }
  for (; r < r1; ++r, base += N) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(base));
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] += __bfloat162float(h[q]);
  }
  float* o = out + ((uint64_t)g * gridDim.y + blockIdx.y) * N + n;  // chunk partial (seg_colsum)
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = acc[q];
}

// One group per output row (groups == num_b): a block per (group, 256-column
// slice) sums ALL the group's rows — 16 row lanes x 32 column threads (8 bf16
// columns each), 8 rows in flight per thread — and reduces the row lanes in a
// fixed order through shared memory: deterministic, no atomics, no memset.
constexpr int CS_LANES = 16;
// One block per (group, row chunk of CS_CHUNK rows, 256 columns): chunk
// partials go to a workspace and the last chunk block of a (group, column
// block) to finish -- an acq_rel ticket -- sums them in chunk order, so db2 is
// deterministic and a heavily loaded expert (skewed routing) is spread over
// many blocks instead of serialising on one.
#ifndef MOE_CS_CHUNK
#define MOE_CS_CHUNK 256  // A/B: c3 db2 22 -> 20 us vs 512, 1024 slower (30 us), 128 slower (c2 39 -> 43 us)
#endif
constexpr int CS_CHUNK = MOE_CS_CHUNK;

__global__ void __launch_bounds__(CS_LANES * 32) colsum_group_bf16_kernel(
    const int32_t* __restrict__ gm, const int32_t* __restrict__ ga, const int32_t* __restrict__ gb,
    int N, int maxch, const __nv_bfloat16* __restrict__ X, float* __restrict__ out,
    float* __restrict__ part_ws, int32_t* __restrict__ ticket) {
  pdl_wait();
  pdl_trigger();
  __shared__ float part[CS_LANES][256 + 8];
  __shared__ int last;
  const int g = blockIdx.x / maxch, ch = blockIdx.x % maxch;
  const int rows = gm[g];
  const int nch = max(1, (rows + CS_CHUNK - 1) / CS_CHUNK);
  if (ch >= nch) return;
  const int r_end = min(rows, (ch + 1) * CS_CHUNK);
  const int cl = threadIdx.x & 31, rl = threadIdx.x >> 5;
  const int n = blockIdx.y * 256 + cl * 8;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (n < N) {
    const __nv_bfloat16* base = X + (uint64_t)ga[g] * N + n;
    int r = ch * CS_CHUNK + rl;
    for (; r + 7 * CS_LANES < r_end; r += 8 * CS_LANES) {
      uint4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)(r + u * CS_LANES) * N));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h[q]);
          acc[2 * q] += f.x;
          acc[2 * q + 1] += f.y;
        }
      }
    }
    for (; r < r_end; r += CS_LANES) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)r * N));
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = __bfloat1622float2(h[q]);
        acc[2 * q] += f.x;
        acc[2 * q + 1] += f.y;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) part[rl][cl * 8 + q] = acc[q];
  __syncthreads();
  const int col = blockIdx.y * 256 + threadIdx.x;
  float sum = 0.f;
  if (threadIdx.x < 256) {
#pragma unroll
    for (int l = 0; l < CS_LANES; ++l) sum += part[l][threadIdx.x];
  }
  if (nch == 1) {
    if (threadIdx.x < 256 && col < N) out[(uint64_t)gb[g] * N + col] = sum;
    return;
  }
  float* const mine = part_ws + ((uint64_t)g * maxch + ch) * N;
  if (threadIdx.x < 256 && col < N) mine[col] = sum;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t* t = ticket + (uint64_t)g * gridDim.y + blockIdx.y;
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
    last = old == nch - 1;
    if (last) *t = 0;  // every chunk block has arrived: re-arm for the next launch
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < 256 && col < N) {
    const float* p = part_ws + (uint64_t)g * maxch * N + col;
    float s = 0.f;
    for (int c = 0; c < nch; ++c) s += __ldcg(p + (uint64_t)c * N);
    out[(uint64_t)gb[g] * N + col] = s;
  }
}

__global__ void build_groups_kernel(uint32_t P, uint32_t El, uint64_t Cs, const int32_t* cnt,
                                   int32_t* gm, int32_t* ga, int32_t* gb, int32_t* gm_k,
                                   int32_t* ga_k, int32_t* gb_k) {
  pdl_wait();
  pdl_trigger();
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P * El) return;
  const uint32_t s = g / El, j = g % El;
  const int32_t m = cnt[g];
  gm[g] = m;
  ga[g] = (int32_t)(g * Cs);
  gb[g] = (int32_t)j;
  const uint32_t gk = j * P + s;
  gm_k[gk] = m;
  ga_k[gk] = (int32_t)(g * Cs);
  gb_k[gk] = (int32_t)j;
}

}  // namespace

void dispatch_tokens(uint64_t T, uint32_t d, uint32_t E, uint32_t k, uint64_t C, uint32_t pad,
                     moe_dtype_t dt, const void* x, const int32_t* expert, const int32_t* position,
                     const int32_t* kept, void* buf, int32_t* slot, cudaStream_t st) {
  const uint64_t Cs = round_up(C, pad);
  const unsigned blocks = (unsigned)std::min<uint64_t>(ceil_div(T, 8), (uint64_t)num_sms() * 8);
  if (T) {
    if (dt == MOE_DTYPE_BF16)
      launch_pdl(dispatch_kernel<__nv_bfloat16>, blocks, 256, 0, st, 
          T, d, E, k, Cs, C, (const __nv_bfloat16*)x, expert, position, (__nv_bfloat16*)buf, slot,
          pad, kept);
    else
      launch_pdl(dispatch_kernel<float>, blocks, 256, 0, st, T, d, E, k, Cs, C, (const float*)x, expert,
                                                     position, (float*)buf, slot, pad, kept);
    MOE_LAUNCH_CHECK("dispatch_kernel");
    count_launch();
  } else if (pad > 1) {
    if (dt == MOE_DTYPE_BF16)
      launch_pdl(zero_pad_kernel<__nv_bfloat16>, E, 256, 0, st, d, Cs, pad, kept, (__nv_bfloat16*)buf);
    else
      launch_pdl(zero_pad_kernel<float>, E, 256, 0, st, d, Cs, pad, kept, (float*)buf);
    MOE_LAUNCH_CHECK("zero_pad_kernel");
    count_launch();
  }
}

void combine_tokens(uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt, const void* Y,
                    const int32_t* slot, const float* gate, void* y, cudaStream_t st) {
  if (!T) return;
  const unsigned blocks = (unsigned)ceil_div(T, 8);
  if (dt == MOE_DTYPE_BF16)
    launch_pdl(combine_kernel<__nv_bfloat16>, blocks, 256, 0, st, T, d, k, (const __nv_bfloat16*)Y, slot,
                                                          gate, (__nv_bfloat16*)y);
  else
    launch_pdl(combine_kernel<float>, blocks, 256, 0, st, T, d, k, (const float*)Y, slot, gate, (float*)y);
  MOE_LAUNCH_CHECK("combine_kernel");
  count_launch();
}

void combine_backward(uint64_t T, uint32_t d, uint32_t E, uint32_t k, uint64_t C, uint32_t pad,
                      moe_dtype_t dt, const void* dy, const void* Y, const int32_t* slot,
                      const float* gate, const int32_t* kept, void* dY, float* dgate,
                      cudaStream_t st) {
  const uint64_t Cs = round_up(C, pad);
  if (T) {
    const unsigned blocks = (unsigned)ceil_div(T, 8);
    if (dt == MOE_DTYPE_BF16)
      launch_pdl(combine_bwd_kernel<__nv_bfloat16>, blocks, 256, 0, st, 
          T, d, k, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)Y, slot, gate,
          (__nv_bfloat16*)dY, dgate, (int)E, Cs, pad, kept);
    else
      launch_pdl(combine_bwd_kernel<float>, blocks, 256, 0, st, T, d, k, (const float*)dy,
                                                        (const float*)Y, slot, gate, (float*)dY,
                                                        dgate, (int)E, Cs, pad, kept);
    MOE_LAUNCH_CHECK("combine_bwd_kernel");
    count_launch();
  } else if (pad > 1) {
    if (dt == MOE_DTYPE_BF16)
      launch_pdl(zero_pad_kernel<__nv_bfloat16>, E, 256, 0, st, d, Cs, pad, kept, (__nv_bfloat16*)dY);
    else
      launch_pdl(zero_pad_kernel<float>, E, 256, 0, st, d, Cs, pad, kept, (float*)dY);
    MOE_LAUNCH_CHECK("zero_pad_kernel");
    count_launch();
  }
}

void gather_dx(uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt, const void* dXe,
               const int32_t* slot, const float* dx_gate, void* dx, cudaStream_t st) {
  if (!T) return;
  const unsigned blocks = (unsigned)ceil_div(T, 8);
  if (dt == MOE_DTYPE_BF16)
    launch_pdl(gather_dx_kernel<__nv_bfloat16>, blocks, 256, 0, st, 
        T, d, k, (const __nv_bfloat16*)dXe, slot, dx_gate, (__nv_bfloat16*)dx);
  else
    launch_pdl(gather_dx_kernel<float>, blocks, 256, 0, st, T, d, k, (const float*)dXe, slot, dx_gate,
                                                    (float*)dx);
  MOE_LAUNCH_CHECK("gather_dx_kernel");
  count_launch();
}

void route_backward(uint64_t T, uint32_t E, uint32_t k, const float* logits, const int32_t* expert,
                    const float* gate, const uint8_t* keep, const int32_t* count1,
                    const float* dgate, float d_aux, float* dlogits_f32, void* dlogits_lp,
                    moe_dtype_t lp_dtype, uint32_t ld, float* dbg, float* dbg_ws,
                    cudaStream_t st) {
  if (!T) {
    if (dbg) MOE_CUDA(cudaMemsetAsync(dbg, 0, sizeof(float) * E, st));
    return;
  }
  const unsigned blocks = (unsigned)ceil_div(T, CHUNK);
  arg_check(!dbg || dbg_ws, "route_backward.dbg_ws: workspace required for the gate-bias gradient");
  float* const dbg_part = dbg ? dbg_ws : nullptr;  // [blocks][E] partials
  MOE_CUDA(cudaFuncSetAttribute(route_bwd_kernel<__nv_bfloat16>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, SLAB_SMEM));
  MOE_CUDA(cudaFuncSetAttribute(route_bwd_kernel<float>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, SLAB_SMEM));
  if (dlogits_lp && lp_dtype == MOE_DTYPE_BF16)
    launch_pdl(route_bwd_kernel<__nv_bfloat16>, blocks, RT_THREADS, SLAB_SMEM, st, 
        T, (int)E, (int)k, logits, expert, gate, keep, count1, dgate, d_aux, dlogits_f32,
        (__nv_bfloat16*)dlogits_lp, (int)ld, dbg_part);
  else
    launch_pdl(route_bwd_kernel<float>, blocks, RT_THREADS, SLAB_SMEM, st, T, (int)E, (int)k, logits, expert, gate, keep,
                                                    count1, dgate, d_aux, dlogits_f32,
                                                    (float*)dlogits_lp, (int)ld, dbg_part);
  MOE_LAUNCH_CHECK("route_bwd_kernel");
  count_launch();
  if (dbg) sum_parts(dbg_part, blocks, E, 1, E, E, false, dbg, st);
}

uint64_t colsum_ws_floats(uint32_t groups, uint32_t N, uint64_t max_rows) {
  // the finest chunking of any colsum path (32 rows, colsum_kernel)
  return (uint64_t)groups * std::max<uint64_t>(1, ceil_div(max_rows, (uint64_t)32)) * N;
}
uint64_t colsum_ticket_ints(uint32_t groups, uint32_t N) {
  return (uint64_t)groups * ceil_div((uint64_t)N, (uint64_t)256);
}

void group_colsum(uint32_t groups, const int32_t* gm, const int32_t* ga, const int32_t* gb,
                  uint32_t num_b, uint32_t N, moe_dtype_t dt, const void* X, float* out,
                  cudaStream_t st, uint64_t max_rows, float* part_ws, int32_t* ticket) {
  if (dt == MOE_DTYPE_BF16 && N % 8 == 0 && groups == num_b && part_ws && ticket) {
    // one group per expert (N = 1 and the P2P exchange): gb is a permutation
    const int maxch = (int)std::max<uint64_t>(1, ceil_div(max_rows, (uint64_t)CS_CHUNK));
    launch_pdl(colsum_group_bf16_kernel, dim3(groups * maxch, (unsigned)ceil_div(N, 256)), CS_LANES * 32, 0,
                               st, gm, ga, gb, (int)N, maxch, (const __nv_bfloat16*)X, out,
                                     part_ws, ticket);
    MOE_LAUNCH_CHECK("colsum_group_bf16_kernel");
    count_launch();
    return;
  }
  // several groups per output (or fp32): chunk partials into part_ws, then a
  // fixed-order segmented sum over (group, chunk) -- deterministic
  arg_check(part_ws != nullptr, "colsum.part_ws: workspace required");
  const uint32_t chunk = dt == MOE_DTYPE_BF16 && N % 8 == 0 ? 64 : 32;
  const uint32_t maxch = (uint32_t)std::max<uint64_t>(1, ceil_div(max_rows, (uint64_t)chunk));
  if (chunk == 64) {
    dim3 grid(groups, maxch, (unsigned)ceil_div(N / 8, 128));
    launch_pdl(colsum_bf16x8_kernel, grid, 128, 0, st, gm, ga, gb, (int)N, (const __nv_bfloat16*)X,
               part_ws);
  } else {
    dim3 grid(groups, maxch, (unsigned)ceil_div(N, 256));
    if (dt == MOE_DTYPE_BF16)
      launch_pdl(colsum_kernel<__nv_bfloat16>, grid, 256, 0, st, gm, ga, gb, (int)N,
                                                         (const __nv_bfloat16*)X, part_ws);
    else
      launch_pdl(colsum_kernel<float>, grid, 256, 0, st, gm, ga, gb, (int)N, (const float*)X, part_ws);
  }
  MOE_LAUNCH_CHECK("colsum_kernel");
  count_launch();
  seg_colsum(groups, gm, gb, num_b, N, chunk, maxch, part_ws, out, st);
}

// Round-robin expert placement: physical expert id pi(e) = (e % P) * El + e / P
// (rank e % P, local expert e / P), so the contiguous-placement exchange and
// slot layout downstream serve it unchanged.  pexpert = pi(expert) (-1 kept),
// pkept[pi(e)] = kept[e].
__global__ void relabel_experts_kernel(uint64_t n, uint32_t E, uint32_t P,
                                       const int32_t* __restrict__ expert,
                                       const int32_t* __restrict__ kept,
                                       int32_t* __restrict__ pexpert, int32_t* __restrict__ pkept) {
  pdl_wait();
  pdl_trigger();
  const uint32_t El = E / P;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < E) pkept[(i % P) * El + i / P] = kept[i];
  if (i < n) {
    const int32_t e = expert[i];
    pexpert[i] = e < 0 ? e : (int32_t)((e % P) * El + e / P);
  }
}

void relabel_experts(uint64_t T, uint32_t k, uint32_t E, uint32_t P, const int32_t* expert,
                     const int32_t* kept, int32_t* pexpert, int32_t* pkept, cudaStream_t st) {
  const uint64_t n = std::max<uint64_t>(T * k, E);
  launch_pdl(relabel_experts_kernel, (unsigned)ceil_div(n, 256), 256, 0, st, T * k, E, P, expert,
             kept, pexpert, pkept);
  MOE_LAUNCH_CHECK("relabel_experts_kernel");
  count_launch();
}

void build_groups(uint32_t P, uint32_t El, uint64_t Cs, const int32_t* cnt, int32_t* gm,
                  int32_t* ga, int32_t* gb, int32_t* gm_k, int32_t* ga_k, int32_t* gb_k,
                  cudaStream_t st) {
  const uint32_t n = P * El;
  launch_pdl(build_groups_kernel, (n + 255) / 256, 256, 0, st, P, El, Cs, cnt, gm, ga, gb, gm_k, ga_k,
                                                       gb_k);
  MOE_LAUNCH_CHECK("build_groups_kernel");
  count_launch();
}

}  // namespace moe
