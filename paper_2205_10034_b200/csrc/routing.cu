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

constexpr int CHUNK = 256;  // tokens per routing block (8 warps x 32)
constexpr int RT_THREADS = 256;
constexpr int MAX_E = 256;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float nan_to_ninf(float v) { return isnan(v) ? -INFINITY : v; }

// Phase A: thread per token (the block is one 256-token chunk): top-k on the
// fp32 logits, softmax, gates; per chunk: histograms (expert-major
// [i][E][nchunks]), in-chunk ranks (warp match over 32 consecutive tokens +
// per-warp histograms), and softmax column partial sums reduced in a fixed
// order (deterministic aux loss).
__global__ void __launch_bounds__(RT_THREADS) route_topk_kernel(
    uint64_t T, int E, int k, const float* __restrict__ logits, int32_t* __restrict__ expert,
    float* __restrict__ gate, int32_t* __restrict__ rank_local, int32_t* __restrict__ chunk_cnt,
    float* __restrict__ psum_part, uint64_t nchunks) {
  __shared__ int hist[2][8][MAX_E];
  __shared__ float pw[8][MAX_E];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t chunk = blockIdx.x;
  const uint64_t t = chunk * CHUNK + threadIdx.x;
  const bool valid = t < T;

  for (int i = threadIdx.x; i < 2 * 8 * MAX_E; i += RT_THREADS) (&hist[0][0][0])[i] = 0;

  // pass 1: top-1 / top-2 on logits (NaN read as -inf, ties to the lowest index)
  const float4* L4 = reinterpret_cast<const float4*>(logits + t * E);
  const float* L = logits + t * E;
  float v1 = -INFINITY, v2 = -INFINITY;
  int i1 = 0x7fffffff, i2 = 0x7fffffff;
  auto consider = [&](float v, int e) {
    v = nan_to_ninf(v);
    if (v > v1 || (v == v1 && e < i1)) {
      v2 = v1; i2 = i1; v1 = v; i1 = e;
    } else if (v > v2 || (v == v2 && e < i2)) {
      v2 = v; i2 = e;
    }
  };
  const bool vec = (E % 4) == 0;
  if (valid) {
    if (vec) {
      for (int q = 0; q < E / 4; ++q) {
        const float4 f = __ldg(L4 + q);
        consider(f.x, 4 * q);
        consider(f.y, 4 * q + 1);
        consider(f.z, 4 * q + 2);
        consider(f.w, 4 * q + 3);
      }
    } else {
      for (int e = 0; e < E; ++e) consider(__ldg(L + e), e);
    }
  }
  // pass 2: softmax denominator (max = v1)
  float z = 0.f;
  if (valid) {
    if (vec) {
      for (int q = 0; q < E / 4; ++q) {
        const float4 f = __ldg(L4 + q);
        z += expf(nan_to_ninf(f.x) - v1) + expf(nan_to_ninf(f.y) - v1) +
             expf(nan_to_ninf(f.z) - v1) + expf(nan_to_ninf(f.w) - v1);
      }
    } else {
      for (int e = 0; e < E; ++e) z += expf(nan_to_ninf(__ldg(L + e)) - v1);
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
  // pass 3: softmax column sums over the warp's 32 tokens: lane l owns experts
  // l, l+32, ...; token j's (max, 1/z) broadcast from lane j; rows read
  // coalesced.  Then a fixed-order sum over the 8 warps (deterministic aux).
  {
    float acc[MAX_E / 32];
#pragma unroll
    for (int q = 0; q < MAX_E / 32; ++q) acc[q] = 0.f;
    const uint64_t t0w = chunk * CHUNK + warp * 32;
    for (int j = 0; j < 32; ++j) {
      const float mj = __shfl_sync(0xffffffffu, v1, j);
      const float ij = __shfl_sync(0xffffffffu, inv, j);
      if (t0w + j >= T) break;
      const float* Lj = logits + (t0w + j) * E;
#pragma unroll
      for (int q = 0; q < MAX_E / 32; ++q) {
        const int e = lane + 32 * q;
        if (e < E) acc[q] += expf(nan_to_ninf(__ldg(Lj + e)) - mj) * ij;
      }
    }
#pragma unroll
    for (int q = 0; q < MAX_E / 32; ++q) {
      const int e = lane + 32 * q;
      if (e < E) pw[warp][e] = acc[q];
    }
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
  for (int x = threadIdx.x; x < k * E; x += RT_THREADS) {
    const int i = x / E, e = x % E;
    int run = 0;
    for (int w = 0; w < 8; ++w) {
      const int c = hist[i][w][e];
      hist[i][w][e] = run;
      run += c;
    }
    chunk_cnt[((uint64_t)i * E + e) * nchunks + chunk] = run;
  }
  for (int e = threadIdx.x; e < E; e += RT_THREADS) {
    float sp = 0.f;
    for (int w = 0; w < 8; ++w) sp += pw[w][e];
    psum_part[chunk * E + e] = sp;
  }
  __syncthreads();
  if (valid) {
    for (int i = 0; i < k; ++i) rank_local[t * k + i] = hist[i][warp][ech[i]] + r_in[i];
  }
}

// Phase B: per-expert exclusive scan over chunks (one warp per expert),
// counts, kept, aux loss.  Single block.
__global__ void __launch_bounds__(1024) route_scan_kernel(
    uint64_t T, int E, int k, uint64_t C, const int32_t* __restrict__ chunk_cnt,
    int32_t* __restrict__ chunk_off, const float* __restrict__ psum_part, uint64_t nchunks,
    int32_t* __restrict__ count1, int32_t* __restrict__ count2, int32_t* __restrict__ kept,
    float* __restrict__ aux) {
  __shared__ float auxe[MAX_E];
  __shared__ int c1s[MAX_E];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int e = warp; e < E; e += nw) {
    // top-1
    const int32_t* cc = chunk_cnt + (uint64_t)e * nchunks;
    int32_t* co = chunk_off + (uint64_t)e * nchunks;
    int carry = 0;
    float ps = 0.f;
    for (uint64_t base = 0; base < nchunks; base += 32) {
      const uint64_t c = base + lane;
      const int v = c < nchunks ? cc[c] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (c < nchunks) co[c] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
      if (c < nchunks) ps += psum_part[c * E + e];
    }
    ps = warp_sum(ps);
    const int c1 = carry;
    int c2 = 0;
    if (k == 2) {
      const int32_t* cc2 = chunk_cnt + ((uint64_t)E + e) * nchunks;
      int32_t* co2 = chunk_off + ((uint64_t)E + e) * nchunks;
      int carry2 = c1;  // top-2 positions start after all (pre-drop) top-1 tokens
      for (uint64_t base = 0; base < nchunks; base += 32) {
        const uint64_t c = base + lane;
        const int v = c < nchunks ? cc2[c] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        if (c < nchunks) co2[c] = carry2 + incl - v;
        carry2 += __shfl_sync(0xffffffffu, incl, 31);
      }
      c2 = carry2 - c1;
    }
    if (lane == 0) {
      count1[e] = c1;
      count2[e] = c2;
      const uint64_t tot = (uint64_t)c1 + (uint64_t)c2;
      kept[e] = (int32_t)(tot < C ? tot : C);
      auxe[e] = ps;
      c1s[e] = c1;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    const double invT = T ? 1.0 / (double)T : 0.0;
    for (int e = 0; e < E; ++e) a += ((double)auxe[e] * invT) * ((double)c1s[e] * invT);
    aux[0] = (float)((double)E * a);
  }
}

// Phase C: positions and keep flags.
__global__ void route_finalize_kernel(uint64_t T, int E, int k, uint64_t C, uint64_t nchunks,
                                      const int32_t* __restrict__ expert,
                                      const int32_t* __restrict__ rank_local,
                                      const int32_t* __restrict__ chunk_off,
                                      int32_t* __restrict__ position, uint8_t* __restrict__ keep) {
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
  const uint64_t nch = route_chunks(T);
  route_topk_kernel<<<(unsigned)nch, RT_THREADS, 0, st>>>(T, (int)E, (int)k, logits, out.expert,
                                                          out.gate, ws.rank_local, ws.chunk_cnt,
                                                          ws.psum_part, nch);
  MOE_LAUNCH_CHECK("route_topk_kernel");
  route_scan_kernel<<<1, 1024, 0, st>>>(T, (int)E, (int)k, C, ws.chunk_cnt, ws.chunk_off,
                                        ws.psum_part, nch, out.count1, out.count2, out.kept,
                                        out.aux_loss);
  MOE_LAUNCH_CHECK("route_scan_kernel");
  const uint64_t n = T * k;
  route_finalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      T, (int)E, (int)k, C, nch, out.expert, ws.rank_local, ws.chunk_off, out.position, out.keep);
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

template <typename T>
__global__ void dispatch_kernel(uint64_t T_, int d, int E, int k, uint64_t Cs, uint64_t C,
                                const T* __restrict__ x, const int32_t* __restrict__ expert,
                                const int32_t* __restrict__ position, T* __restrict__ buf,
                                int32_t* __restrict__ slot) {
  const int lane = threadIdx.x & 31;
  const uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= T_) return;
  int64_t dst[2] = {-1, -1};
  for (int i = 0; i < k; ++i) {
    const int e = expert[t * k + i];
    const int p = position[t * k + i];
    const int64_t s = ((uint64_t)p < C) ? (int64_t)e * (int64_t)Cs + p : -1;
    dst[i] = s;
    if (lane == 0) slot[t * k + i] = (int32_t)s;
  }
  if (dst[0] < 0 && dst[1] < 0) return;
  const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
  const int nv = d / Vec<T>::N;
  for (int v = lane; v < nv; v += 32) {
    const uint4 val = __ldg(src + v);
    for (int i = 0; i < k; ++i)
      if (dst[i] >= 0) reinterpret_cast<uint4*>(buf + dst[i] * d)[v] = val;
  }
}

// Zero rows [kept_e, round_up(kept_e, pad)) of each expert slot: one block per
// expert, rows strided over warps.
template <typename T>
__global__ void zero_pad_kernel(int d, uint64_t Cs, uint32_t pad, const int32_t* __restrict__ kept,
                                T* __restrict__ buf) {
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
                                   float* __restrict__ dgate) {
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

// Routing backward (DESIGN.md Appendix A §9), thread per token: recompute the
// softmax from the stored logits, add the aux-loss term and the gate term, and
// write the dlogits row (fp32 and/or the bf16 GEMM operand, pad columns zero).
template <typename LP>
__global__ void __launch_bounds__(256) route_bwd_kernel(
    uint64_t T_, int E, int k, const float* __restrict__ logits,
    const int32_t* __restrict__ expert, const float* __restrict__ gate,
    const uint8_t* __restrict__ keep, const int32_t* __restrict__ count1,
    const float* __restrict__ dgate, float d_aux, float* __restrict__ dl_f32,
    LP* __restrict__ dl_lp, int ld, float* __restrict__ dbg) {
  __shared__ float a_s[MAX_E];
  __shared__ float dbg_s[MAX_E];
  const float invT = 1.0f / (float)T_;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    a_s[e] = (float)E * (float)count1[e] * invT * invT;
    dbg_s[e] = 0.f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = t < T_;
  const float* L = logits + (valid ? t : 0) * E;
  float m = -INFINITY, z = 0.f, pnum = 0.f;
  if (valid) {
    for (int e = 0; e < E; ++e) m = fmaxf(m, nan_to_ninf(__ldg(L + e)));
    for (int e = 0; e < E; ++e) {
      const float ex = expf(nan_to_ninf(__ldg(L + e)) - m);
      z += ex;
      pnum = fmaf(ex, a_s[e], pnum);
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
  for (int e0 = 0; e0 < E; e0 += 8) {
    float dl[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u;
      float v = 0.f;
      if (valid && e < E) {
        const float pe = expf(nan_to_ninf(__ldg(L + e)) - m) * inv;
        v = d_aux * pe * (a_s[e] - pa);
        if (k == 1) v += gterm * p1 * ((e == e1 ? 1.f : 0.f) - pe);
        else v += (e == e1 ? gterm : 0.f) - (e == e2 ? gterm : 0.f);
      }
      dl[u] = v;
    }
    if (valid) {
      if (dl_f32) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u < E) dl_f32[t * E + e0 + u] = dl[u];
      }
      if (dl_lp) {
        if (sizeof(LP) == 2 && (ld % 8) == 0 && e0 + 8 <= ld) {
          uint4 o;
          o.x = pack_bf16x2(dl[0], dl[1]);
          o.y = pack_bf16x2(dl[2], dl[3]);
          o.z = pack_bf16x2(dl[4], dl[5]);
          o.w = pack_bf16x2(dl[6], dl[7]);
          *reinterpret_cast<uint4*>(dl_lp + t * ld + e0) = o;
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (e0 + u < ld) dl_lp[t * ld + e0 + u] = (LP)dl[u];
        }
      }
    }
    if (dbg) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        float v = dl[u];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0 && e0 + u < E) atomicAdd(&dbg_s[e0 + u], v);
      }
    }
  }
  if (valid && dl_lp) {
    const int from = ((E + 7) / 8) * 8;
    for (int e = from; e < ld; ++e) dl_lp[t * ld + e] = (LP)0.f;
  }
  __syncthreads();
  if (dbg)
    for (int e = threadIdx.x; e < E; e += blockDim.x) atomicAdd(&dbg[e], dbg_s[e]);
}

template <typename T>
__global__ void colsum_kernel(const int32_t* __restrict__ gm, const int32_t* __restrict__ ga,
                              const int32_t* __restrict__ gb, int N, const T* __restrict__ X,
                              float* __restrict__ out) {
  const int g = blockIdx.x;
  const int rows = gm[g];
  const int r0 = blockIdx.y * 128;
  if (r0 >= rows) return;
  const int n = blockIdx.z * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int r1 = min(rows, r0 + 128);
  const T* base = X + ((uint64_t)ga[g] + r0) * N + n;
  float s = 0.f;
  for (int r = r0; r < r1; ++r, base += N) s += (float)*base;
  atomicAdd(out + (uint64_t)gb[g] * N + n, s);
}

// bf16, 8 columns per thread (16-byte loads), 64 rows per block, 4 rows in flight
__global__ void colsum_bf16x8_kernel(const int32_t* __restrict__ gm, const int32_t* __restrict__ ga,
                                     const int32_t* __restrict__ gb, int N,
                                     const __nv_bfloat16* __restrict__ X, float* __restrict__ out) {
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
  for (; r + 4 <= r1; r += 4, base += 4 * (uint64_t)N) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const uint4*>(base + (uint64_t)u * N));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
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
  float* o = out + (uint64_t)gb[g] * N + n;
#pragma unroll
  for (int q = 0; q < 8; ++q) atomicAdd(o + q, acc[q]);
}

__global__ void build_groups_kernel(uint32_t P, uint32_t El, uint64_t Cs, const int32_t* cnt,
                                   int32_t* gm, int32_t* ga, int32_t* gb, int32_t* gm_k,
                                   int32_t* ga_k, int32_t* gb_k) {
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
  const unsigned blocks = (unsigned)ceil_div(T, 8);
  if (T) {
    if (dt == MOE_DTYPE_BF16)
      dispatch_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
          T, d, E, k, Cs, C, (const __nv_bfloat16*)x, expert, position, (__nv_bfloat16*)buf, slot);
    else
      dispatch_kernel<float><<<blocks, 256, 0, st>>>(T, d, E, k, Cs, C, (const float*)x, expert,
                                                     position, (float*)buf, slot);
    MOE_LAUNCH_CHECK("dispatch_kernel");
    count_launch();
  }
  if (pad > 1) {
    if (dt == MOE_DTYPE_BF16)
      zero_pad_kernel<__nv_bfloat16><<<E, 256, 0, st>>>(d, Cs, pad, kept, (__nv_bfloat16*)buf);
    else
      zero_pad_kernel<float><<<E, 256, 0, st>>>(d, Cs, pad, kept, (float*)buf);
    MOE_LAUNCH_CHECK("zero_pad_kernel");
    count_launch();
  }
}

void combine_tokens(uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt, const void* Y,
                    const int32_t* slot, const float* gate, void* y, cudaStream_t st) {
  if (!T) return;
  const unsigned blocks = (unsigned)ceil_div(T, 8);
  if (dt == MOE_DTYPE_BF16)
    combine_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(T, d, k, (const __nv_bfloat16*)Y, slot,
                                                          gate, (__nv_bfloat16*)y);
  else
    combine_kernel<float><<<blocks, 256, 0, st>>>(T, d, k, (const float*)Y, slot, gate, (float*)y);
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
      combine_bwd_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
          T, d, k, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)Y, slot, gate,
          (__nv_bfloat16*)dY, dgate);
    else
      combine_bwd_kernel<float><<<blocks, 256, 0, st>>>(T, d, k, (const float*)dy,
                                                        (const float*)Y, slot, gate, (float*)dY,
                                                        dgate);
    MOE_LAUNCH_CHECK("combine_bwd_kernel");
    count_launch();
  }
  if (pad > 1) {
    if (dt == MOE_DTYPE_BF16)
      zero_pad_kernel<__nv_bfloat16><<<E, 256, 0, st>>>(d, Cs, pad, kept, (__nv_bfloat16*)dY);
    else
      zero_pad_kernel<float><<<E, 256, 0, st>>>(d, Cs, pad, kept, (float*)dY);
    MOE_LAUNCH_CHECK("zero_pad_kernel");
    count_launch();
  }
}

void gather_dx(uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt, const void* dXe,
               const int32_t* slot, const float* dx_gate, void* dx, cudaStream_t st) {
  if (!T) return;
  const unsigned blocks = (unsigned)ceil_div(T, 8);
  if (dt == MOE_DTYPE_BF16)
    gather_dx_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        T, d, k, (const __nv_bfloat16*)dXe, slot, dx_gate, (__nv_bfloat16*)dx);
  else
    gather_dx_kernel<float><<<blocks, 256, 0, st>>>(T, d, k, (const float*)dXe, slot, dx_gate,
                                                    (float*)dx);
  MOE_LAUNCH_CHECK("gather_dx_kernel");
  count_launch();
}

void route_backward(uint64_t T, uint32_t E, uint32_t k, const float* logits, const int32_t* expert,
                    const float* gate, const uint8_t* keep, const int32_t* count1,
                    const float* dgate, float d_aux, float* dlogits_f32, void* dlogits_lp,
                    moe_dtype_t lp_dtype, uint32_t ld, float* dbg, cudaStream_t st) {
  if (!T) return;
  const unsigned blocks = (unsigned)ceil_div(T, 256);
  if (dlogits_lp && lp_dtype == MOE_DTYPE_BF16)
    route_bwd_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
        T, (int)E, (int)k, logits, expert, gate, keep, count1, dgate, d_aux, dlogits_f32,
        (__nv_bfloat16*)dlogits_lp, (int)ld, dbg);
  else
    route_bwd_kernel<float><<<blocks, 256, 0, st>>>(T, (int)E, (int)k, logits, expert, gate, keep,
                                                    count1, dgate, d_aux, dlogits_f32,
                                                    (float*)dlogits_lp, (int)ld, dbg);
  MOE_LAUNCH_CHECK("route_bwd_kernel");
  count_launch();
}

void group_colsum(uint32_t groups, const int32_t* gm, const int32_t* ga, const int32_t* gb,
                  uint32_t num_b, uint32_t N, moe_dtype_t dt, const void* X, float* out,
                  cudaStream_t st, uint64_t max_rows) {
  MOE_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * (uint64_t)num_b * N, st));
  if (dt == MOE_DTYPE_BF16 && N % 8 == 0) {
    dim3 grid(groups, (unsigned)ceil_div(max_rows, 64), (unsigned)ceil_div(N / 8, 128));
    colsum_bf16x8_kernel<<<grid, 128, 0, st>>>(gm, ga, gb, (int)N, (const __nv_bfloat16*)X, out);
  } else {
    dim3 grid(groups, (unsigned)ceil_div(max_rows, 128), (unsigned)ceil_div(N, 256));
    if (dt == MOE_DTYPE_BF16)
      colsum_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(gm, ga, gb, (int)N,
                                                         (const __nv_bfloat16*)X, out);
    else
      colsum_kernel<float><<<grid, 256, 0, st>>>(gm, ga, gb, (int)N, (const float*)X, out);
  }
  MOE_LAUNCH_CHECK("colsum_kernel");
  count_launch();
}

void build_groups(uint32_t P, uint32_t El, uint64_t Cs, const int32_t* cnt, int32_t* gm,
                  int32_t* ga, int32_t* gb, int32_t* gm_k, int32_t* ga_k, int32_t* gb_k,
                  cudaStream_t st) {
  const uint32_t n = P * El;
  build_groups_kernel<<<(n + 255) / 256, 256, 0, st>>>(P, El, Cs, cnt, gm, ga, gb, gm_k, ga_k,
                                                       gb_k);
  MOE_LAUNCH_CHECK("build_groups_kernel");
  count_launch();
}

}  // namespace moe
