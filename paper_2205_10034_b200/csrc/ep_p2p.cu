// K4 over NVLink peer memory: the dispatch and combine-backward kernels store
// token rows straight into the owning rank's receive buffer (CUDA IPC mapping
// of one window per rank), and expert outputs are pushed back the same way —
// the exchange is fused into the kernels that produce the rows, moves exactly
// the kept rows (no capacity padding on the wire) and needs no host sync.
//
// Per phase the kept counts are all-gathered first (E int32 per rank, one
// tiny peer-store kernel) so every sender knows where its rows start inside
// the receiver's per-expert region: rows of source s for expert e land at
// offset sum_{s' < s} cnt[s'][e].  Each local expert is then ONE contiguous
// GEMM group for any number of ranks (no per-(source, expert) tile quantisation).
//
// Ordering: every producing kernel ends with a grid-wide "last block" step that
// publishes `epoch` into each destination's flags[slot][me] with a
// system-scope release store after all its remote stores are fenced
// (fence.sc.sys per thread, then an atomic ticket); consumers spin on
// ld.acquire.sys in a one-block wait kernel.  Reuse safety: a phase (forward or
// backward) starts only after every peer has finished its previous phase
// (SLOT_PHASE), which is when it last read the buffers this phase overwrites.
// Spins time out after a configurable limit (MOE_P2P_TIMEOUT_S, default 600 s,
// 0 = never) by recording an error code instead of trapping; teardown is a
// flag handshake so no peer store can land in a freed window.
//
// Receive order: alltoall_flat's source rank order (collectives.cpp:10-21)
// rotated to start at the receiver (its own rows first, then r+1, ..., r-1),
// so the receiver's expert GEMM can start on its local rows before any peer
// row lands.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

#include "common.cuh"
#include "ep_p2p.h"
#include "kernels.h"

namespace moe {

namespace {

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Kernel-side view of the window (by value).
struct Win {
  uint8_t** peers;
  uint64_t off_xr, off_dyr, off_cnt, off_flags;
  uint32_t P, me, E, El;
  uint64_t Cs, Rmax, row_bytes;
};

__device__ __forceinline__ uint64_t* flag_at(uint8_t* base, const Win& w, int slot, uint32_t src) {
  return reinterpret_cast<uint64_t*>(base + w.off_flags) + (uint64_t)slot * w.P + src;
}
__device__ __forceinline__ const int32_t* cnt_of(const Win& w) {
  return reinterpret_cast<const int32_t*>(w.peers[w.me] + w.off_cnt);
}

// All threads of every block call this exactly once at the end of a producing
// kernel; the last block to arrive publishes the epoch to every peer.
__device__ void grid_done_signal(const Win& w, uint32_t* ctr, int slot, uint64_t value) {
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    const unsigned prev = atomicAdd(ctr, 1u);
    if (prev == nb - 1) {
      __threadfence_system();
      for (uint32_t p = 0; p < w.P; ++p)
        if (p != w.me) st_release_sys(flag_at(w.peers[p], w, slot, w.me), value);
      atomicExch(ctr, 0u);
    }
  }
}

// Spin until every peer's flag reaches `target`.  timeout_ns == 0 waits
// forever (NCCL's behaviour); otherwise a late peer sets *err = 1000 +
// 16*slot + peer and the wait gives up WITHOUT trapping, so the context
// survives and the host can read the code (moe_layer_comm_status) and recover
// or abort.  Once *err is set every later wait returns at once (fail fast).
__global__ void p2p_wait_kernel(const uint64_t* flags, uint32_t P, uint32_t me, int slot,
                                uint64_t target, int32_t* err, uint64_t timeout_ns,
                                int fail_fast = 1) {
  const uint32_t p = threadIdx.x;
  if (p < P && p != me) {
    const uint64_t* f = flags + (uint64_t)slot * P + p;
    const uint64_t t0 = globaltimer();
    volatile int32_t* verr = err;
    while (ld_acquire_sys(f) < target) {
      if (fail_fast && *verr != 0) break;
      if (timeout_ns && globaltimer() - t0 > timeout_ns) {
        atomicCAS(err, 0, 1000 + slot * 16 + (int)p);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

__global__ void p2p_signal_kernel(Win w, int slot, uint64_t value) {
  __threadfence_system();
  const uint32_t p = threadIdx.x;
  if (p < w.P && p != w.me) st_release_sys(flag_at(w.peers[p], w, slot, w.me), value);
}

// kept[E] -> cnt[me][:] on every rank (including this one)
__global__ void p2p_counts_kernel(Win w, uint32_t* ctr, const int32_t* __restrict__ kept,
                                  uint64_t epoch) {
  for (uint32_t e = threadIdx.x; e < w.E; e += blockDim.x) {
    const int32_t n = kept[e];
    for (uint32_t p = 0; p < w.P; ++p)
      reinterpret_cast<int32_t*>(w.peers[p] + w.off_cnt)[(uint64_t)w.me * w.E + e] = n;
  }
  grid_done_signal(w, ctr, SLOT_CNT, epoch);
}

// offset of source `me`'s rows inside expert e's region on its owner
// Receive order inside a region: the receiver's own rows first, then the
// other sources in rank order from there (receiver r: r, r+1, ..., r-1), so a
// receiver can run its local rows before any peer row has landed.
// Offset of source `src`'s rows of expert e in receiver `recv`'s region:
__device__ __forceinline__ int rot_offset(const int32_t* cnt, uint32_t E, uint32_t P,
                                          uint32_t recv, uint32_t src, int e) {
  int off = 0;
  const uint32_t n = (src + P - recv) % P;
  for (uint32_t i = 0; i < n; ++i) off += cnt[(uint64_t)((recv + i) % P) * E + e];
  return off;
}
// offset of this rank's rows in the region of expert e (owner e / El)
__device__ __forceinline__ int src_offset(const int32_t* cnt, uint32_t E, uint32_t P, uint32_t El,
                                          uint32_t me, int e) {
  return rot_offset(cnt, E, P, (uint32_t)e / El, me, e);
}

constexpr int MAXE = 256;

// Persistent grid (a few blocks per SM), warp per token, grid-stride: the
// count-matrix prologue and the system-scope fence of the completion signal
// are paid once per block instead of once per 8 tokens, and each lane has all
// 16-byte pieces of its row in flight before the first (remote) store.
template <typename T, int NV>
__global__ void __launch_bounds__(256) p2p_dispatch_kernel(
    Win w, uint32_t* ctr, uint64_t T_, int d, int k, uint64_t C, const T* __restrict__ x,
    const int32_t* __restrict__ expert, const int32_t* __restrict__ position,
    int32_t* __restrict__ slot, uint64_t epoch) {
  __shared__ int off_s[MAXE];
  const int32_t* cnt = cnt_of(w);
  for (uint32_t e = threadIdx.x; e < w.E; e += blockDim.x) off_s[e] = src_offset(cnt, w.E, w.P, w.El, w.me, e);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nv = (int)(w.row_bytes / 16);
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T_;
       t += nwarps) {
    uint4* dst[2] = {nullptr, nullptr};
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      if (i >= k) break;
      const int e = expert[t * k + i];
      const int p = position[t * k + i];
      const bool keep = (uint64_t)p < C;
      if (lane == 0) slot[t * k + i] = keep ? (int32_t)(e * w.Cs + p) : -1;
      if (keep) {
        const int r = e / (int)w.El, j = e % (int)w.El;
        const uint64_t row = (uint64_t)j * w.Rmax + off_s[e] + p;
        dst[i] = reinterpret_cast<uint4*>(w.peers[r] + w.off_xr + row * w.row_bytes);
      }
    }
    const uint4* src = reinterpret_cast<const uint4*>(x + t * d);
    if constexpr (NV > 0) {
      uint4 val[NV];
#pragma unroll
      for (int q = 0; q < NV; ++q) val[q] = __ldg(src + lane + 32 * q);
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        if (dst[0]) dst[0][lane + 32 * q] = val[q];
        if (dst[1]) dst[1][lane + 32 * q] = val[q];
      }
    } else {  // any row size
      for (int v = lane; v < nv; v += 32) {
        const uint4 val = __ldg(src + v);
        if (dst[0]) dst[0][v] = val;
        if (dst[1]) dst[1][v] = val;
      }
    }
  }
  grid_done_signal(w, ctr, SLOT_DISPATCH, epoch);
}

// one block per local expert: group tables + zero pad rows [m, round64(m))
__global__ void p2p_local_groups_kernel(Win w, int32_t* gm, int32_t* ga, int32_t* gb,
                                        uint8_t* buf) {
  const int j = blockIdx.x;
  const int e = (int)(w.me * w.El) + j;
  const int32_t* cnt = cnt_of(w);
  int m = 0;
  for (uint32_t s = 0; s < w.P; ++s) m += cnt[(uint64_t)s * w.E + e];
  if (threadIdx.x == 0) {
    gm[j] = m;
    ga[j] = (int32_t)(j * w.Rmax);
    gb[j] = j;
  }
  const int end = (int)min((uint64_t)((m + 63) / 64) * 64, w.Rmax);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nv = (int)(w.row_bytes / 16);
  for (int r = m + warp; r < end; r += nw) {
    uint4* row = reinterpret_cast<uint4*>(buf + ((uint64_t)j * w.Rmax + r) * w.row_bytes);
    for (int v = lane; v < nv; v += 32) row[v] = make_uint4(0, 0, 0, 0);
  }
}

template <typename T>
__device__ __forceinline__ void ld8(const T* p, float (&f)[8]);
template <>
__device__ __forceinline__ void ld8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(h[i]);
}
template <>
__device__ __forceinline__ void ld8<float>(const float* p, float (&f)[8]) {
  const float4 a = reinterpret_cast<const float4*>(p)[0];
  const float4 b = reinterpret_cast<const float4*>(p)[1];
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
template <typename T>
__device__ __forceinline__ void st8(T* p, const float (&f)[8]);
template <>
__device__ __forceinline__ void st8<__nv_bfloat16>(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 o;
  o.x = pack_bf16x2(f[0], f[1]);
  o.y = pack_bf16x2(f[2], f[3]);
  o.z = pack_bf16x2(f[4], f[5]);
  o.w = pack_bf16x2(f[6], f[7]);
  *reinterpret_cast<uint4*>(p) = o;
}
template <>
__device__ __forceinline__ void st8<float>(float* p, const float (&f)[8]) {
  reinterpret_cast<float4*>(p)[0] = make_float4(f[0], f[1], f[2], f[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(f[4], f[5], f[6], f[7]);
}

template <typename T>
__global__ void __launch_bounds__(256) p2p_combine_bwd_kernel(
    Win w, uint64_t off_yh, uint32_t* ctr, uint64_t T_, int d, int k, const T* __restrict__ dy,
    const int32_t* __restrict__ slot, const float* __restrict__ gate,
    const int32_t* __restrict__ expert, const int32_t* __restrict__ position,
    float* __restrict__ dgate, uint64_t epoch) {
  __shared__ int off_s[MAXE];
  const int32_t* cnt = cnt_of(w);
  for (uint32_t e = threadIdx.x; e < w.E; e += blockDim.x) off_s[e] = src_offset(cnt, w.E, w.P, w.El, w.me, e);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const T* Yh = reinterpret_cast<const T*>(w.peers[w.me] + off_yh);
  const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < T_;
       t += nwarps) {
    for (int i = 0; i < k; ++i) {
      const int32_t s = slot[t * k + i];
      if (s < 0) {
        if (lane == 0) dgate[t * k + i] = 0.f;
        continue;
      }
      const int e = expert[t * k + i], p = position[t * k + i];
      const int r = e / (int)w.El, j = e % (int)w.El;
      T* dst = reinterpret_cast<T*>(w.peers[r] + w.off_dyr) +
               ((uint64_t)j * w.Rmax + off_s[e] + p) * d;
      const float g = gate[t * k + i];
      float dot = 0.f;
      for (int c = lane * 8; c < d; c += 256) {
        float a[8], b[8], o[8];
        ld8<T>(dy + t * d + c, a);
        ld8<T>(Yh + (uint64_t)s * d + c, b);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          dot = fmaf(a[q], b[q], dot);
          o[q] = g * a[q];
        }
        st8<T>(dst + c, o);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      if (lane == 0) dgate[t * k + i] = dot;
    }
  }
  grid_done_signal(w, ctr, SLOT_DY, epoch);
}

// grid (El * P, row chunks of 64): (j, s) = (blockIdx.x / P, blockIdx.x % P)
__global__ void __launch_bounds__(256) p2p_push_kernel(Win w, uint64_t home_off, uint32_t* ctr,
                                                       const uint8_t* __restrict__ src,
                                                       int slot_id, uint64_t epoch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x / w.P, s = blockIdx.x % w.P;
  const int e = (int)(w.me * w.El) + j;
  const int32_t* cnt = cnt_of(w);
  const int off = rot_offset(cnt, w.E, w.P, w.me, (uint32_t)s, e);
  const int n = cnt[(uint64_t)s * w.E + e];
  const int r0 = blockIdx.y * 64;
  const uint64_t nv = w.row_bytes / 16;
  for (int r = r0 + warp; r < min(n, r0 + 64); r += 8) {
    const uint4* from =
        reinterpret_cast<const uint4*>(src + ((uint64_t)j * w.Rmax + off + r) * w.row_bytes);
    uint4* to = reinterpret_cast<uint4*>(w.peers[s] + home_off +
                                         ((uint64_t)e * w.Cs + r) * w.row_bytes);
    for (uint64_t v = lane; v < nv; v += 32) to[v] = __ldg(from + v);
  }
  grid_done_signal(w, ctr, slot_id, epoch);
}

// red[me] of every window := a ++ b (float4 stores over NVLink for a)
__global__ void p2p_red_push_kernel(Win w, uint64_t off_red, uint64_t n_red, uint32_t* ctr,
                                    const float* __restrict__ a, uint64_t na,
                                    const float* __restrict__ b, uint64_t nb, uint64_t epoch) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < na / 4; i += nt) {
    const float4 v = reinterpret_cast<const float4*>(a)[i];
    for (uint32_t p = 0; p < w.P; ++p)
      reinterpret_cast<float4*>(w.peers[p] + off_red + (uint64_t)w.me * n_red * 4)[i] = v;
  }
  for (uint64_t i = tid; i < nb; i += nt) {
    const float v = b[i];
    for (uint32_t p = 0; p < w.P; ++p)
      reinterpret_cast<float*>(w.peers[p] + off_red + (uint64_t)w.me * n_red * 4)[na + i] = v;
  }
  grid_done_signal(w, ctr, SLOT_GRAD, epoch);
}

// a ++ b := sum over sources of red[s], in source order (identical on all ranks)
__global__ void p2p_red_sum_kernel(const float* __restrict__ red, uint32_t P, uint64_t n_red,
                                   float* __restrict__ a, uint64_t na, float* __restrict__ b,
                                   uint64_t nb) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < na / 4; i += nt) {
    float4 acc = reinterpret_cast<const float4*>(red)[i];
    for (uint32_t s = 1; s < P; ++s) {
      const float4 v = reinterpret_cast<const float4*>(red + s * n_red)[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(a)[i] = acc;
  }
  for (uint64_t i = tid; i < nb; i += nt) {
    float acc = red[na + i];
    for (uint32_t s = 1; s < P; ++s) acc += red[s * n_red + na + i];
    b[i] = acc;
  }
}

uint64_t a256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

Win win_of(const P2PWindow& w) {
  return Win{w.peer_dev, w.off_xr, w.off_dyr, w.off_cnt, w.off_flags, w.P, w.me, w.E, w.El,
             w.Cs, w.Rmax, w.row_bytes};
}
uint32_t* ctr_of(const P2PWindow& w, int i) {
  return reinterpret_cast<uint32_t*>(w.base + w.off_ctr) + i;
}

}  // namespace

#define P2P_NCCL(expr)                                                                \
  do {                                                                                \
    ncclResult_t _r = (expr);                                                         \
    if (_r != ncclSuccess)                                                            \
      ::moe::fail(MOE_ERR_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));  \
  } while (0)

uint64_t p2p_default_timeout_ns() {
  const char* v = std::getenv("MOE_P2P_TIMEOUT_S");
  const double s = v && *v ? std::atof(v) : 600.0;
  return s <= 0 ? 0 : (uint64_t)(s * 1e9);
}

void p2p_setup(P2PWindow& w, void* nccl_comm, uint32_t P, uint32_t me, uint32_t E, uint64_t Cs,
               uint64_t row_bytes, uint64_t n_red, cudaStream_t st) {
  config_check(P <= 8, "layer.ep_size: P2P exchange supports up to 8 GPUs of one box");
  config_check(E <= (uint32_t)MAXE, "layer.num_experts: P2P exchange supports up to 256");
  config_check(row_bytes % 16 == 0, "layer.d_model: rows must be a multiple of 16 bytes");
  w.P = P;
  w.me = me;
  w.E = E;
  w.El = E / P;
  w.Cs = Cs;
  w.Rmax = (uint64_t)P * Cs;
  w.row_bytes = row_bytes;
  w.n_red = (n_red + 3) / 4 * 4;
  w.timeout_ns = p2p_default_timeout_ns();
  const uint64_t region = (uint64_t)w.El * w.Rmax * row_bytes;  // == E * Cs rows
  const uint64_t home = (uint64_t)E * Cs * row_bytes;
  w.off_xr = 0;
  w.off_dyr = a256(w.off_xr + region);
  w.off_yh = a256(w.off_dyr + region);
  w.off_dxh = a256(w.off_yh + home);
  w.off_cnt = a256(w.off_dxh + home);
  w.off_flags = a256(w.off_cnt + (uint64_t)P * E * 4);
  w.off_ctr = a256(w.off_flags + (uint64_t)NSLOT * P * 8);
  w.off_red = a256(w.off_ctr + 256);
  w.bytes = w.off_red + (uint64_t)P * w.n_red * 4;
  MOE_CUDA(cudaMalloc(&w.base, w.bytes));
  MOE_CUDA(cudaMemsetAsync(w.base, 0, w.bytes, st));
  MOE_CUDA(cudaMalloc(&w.err, sizeof(int32_t)));
  MOE_CUDA(cudaMemsetAsync(w.err, 0, sizeof(int32_t), st));
  cudaIpcMemHandle_t h;
  MOE_CUDA(cudaIpcGetMemHandle(&h, w.base));
  uint8_t* dh = nullptr;
  MOE_CUDA(cudaMalloc(&dh, (uint64_t)P * sizeof(h)));
  MOE_CUDA(cudaMemcpyAsync(dh + me * sizeof(h), &h, sizeof(h), cudaMemcpyHostToDevice, st));
  P2P_NCCL(ncclAllGather(dh + me * sizeof(h), dh, sizeof(h), ncclUint8, (ncclComm_t)nccl_comm, st));
  std::vector<cudaIpcMemHandle_t> all(P);
  MOE_CUDA(cudaMemcpyAsync(all.data(), dh, (uint64_t)P * sizeof(h), cudaMemcpyDeviceToHost, st));
  MOE_CUDA(cudaStreamSynchronize(st));
  MOE_CUDA(cudaFree(dh));
  for (uint32_t p = 0; p < P; ++p) {
    if (p == me) {
      w.peer_host[p] = w.base;
      continue;
    }
    void* ptr = nullptr;
    MOE_CUDA(cudaIpcOpenMemHandle(&ptr, all[p], cudaIpcMemLazyEnablePeerAccess));
    w.peer_host[p] = static_cast<uint8_t*>(ptr);
  }
  MOE_CUDA(cudaMalloc(&w.peer_dev, P * sizeof(uint8_t*)));
  MOE_CUDA(cudaMemcpy(w.peer_dev, w.peer_host, P * sizeof(uint8_t*), cudaMemcpyHostToDevice));
  // every rank has mapped every window before anyone writes into one
  int32_t* one = nullptr;
  MOE_CUDA(cudaMalloc(&one, 4));
  P2P_NCCL(ncclAllReduce(one, one, 1, ncclInt32, ncclSum, (ncclComm_t)nccl_comm, st));
  MOE_CUDA(cudaStreamSynchronize(st));
  MOE_CUDA(cudaFree(one));
}

int32_t p2p_status(const P2PWindow& w) {
  if (!w.err) return 0;
  int32_t e = 0;
  MOE_CUDA(cudaMemcpy(&e, w.err, 4, cudaMemcpyDeviceToHost));
  return e;
}

void p2p_teardown(P2PWindow& w) {
  if (w.P > 1 && w.base) {
    // Handshake before unmapping: after this rank's device work is done it
    // stores BYE into every peer's window (its last store into any of them)
    // and waits for every peer's BYE in its own.  Once all have arrived no
    // peer will write here again, so the window can be freed.
    cudaStream_t st = nullptr;
    if (cudaDeviceSynchronize() == cudaSuccess &&
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess) {
      p2p_signal_kernel<<<1, 32, 0, st>>>(win_of(w), SLOT_BYE, 1);
      // the BYE wait does not fail fast on an earlier error: a late peer
      // still gets the full timeout to stop writing before the window goes
      p2p_wait_kernel<<<1, 32, 0, st>>>(reinterpret_cast<const uint64_t*>(w.base + w.off_flags),
                                         w.P, w.me, SLOT_BYE, 1, w.err, w.timeout_ns, 0);
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
  for (uint32_t p = 0; p < w.P; ++p)
    if (p != w.me && w.peer_host[p]) cudaIpcCloseMemHandle(w.peer_host[p]);
  if (w.peer_dev) cudaFree(w.peer_dev);
  if (w.base) cudaFree(w.base);
  if (w.err) cudaFree(w.err);
  w = P2PWindow{};
}

void p2p_wait(const P2PWindow& w, int slot, uint64_t target, cudaStream_t st) {
  if (w.P <= 1) return;
  p2p_wait_kernel<<<1, 32, 0, st>>>(reinterpret_cast<const uint64_t*>(w.base + w.off_flags), w.P,
                                     w.me, slot, target, w.err, w.timeout_ns);
  MOE_LAUNCH_CHECK("p2p_wait_kernel");
  count_launch();
}

void p2p_signal(const P2PWindow& w, int slot, uint64_t value, cudaStream_t st) {
  if (w.P <= 1) return;
  p2p_signal_kernel<<<1, 32, 0, st>>>(win_of(w), slot, value);
  MOE_LAUNCH_CHECK("p2p_signal_kernel");
  count_launch();
}

void p2p_counts(const P2PWindow& w, const int32_t* kept, uint64_t epoch, cudaStream_t st) {
  p2p_counts_kernel<<<1, 256, 0, st>>>(win_of(w), ctr_of(w, 4), kept, epoch);
  MOE_LAUNCH_CHECK("p2p_counts_kernel");
  count_launch();
}

static unsigned red_grid(uint64_t na, uint64_t nb) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(na / 4 + nb, 256),
                                                            (uint64_t)num_sms()));
}

void p2p_allreduce_push(const P2PWindow& w, const float* a, uint64_t na, const float* b,
                        uint64_t nb, uint64_t epoch, cudaStream_t st) {
  if (w.P <= 1) return;
  arg_check(na % 4 == 0 && na + nb <= w.n_red, "p2p_allreduce: gradient does not fit the window");
  p2p_red_push_kernel<<<red_grid(na, nb), 256, 0, st>>>(win_of(w), w.off_red, w.n_red,
                                                        ctr_of(w, 5), a, na, b, nb, epoch);
  MOE_LAUNCH_CHECK("p2p_red_push_kernel");
  count_launch();
}

void p2p_allreduce_finish(const P2PWindow& w, float* a, uint64_t na, float* b, uint64_t nb,
                          uint64_t epoch, cudaStream_t st) {
  if (w.P <= 1) return;
  p2p_wait(w, SLOT_GRAD, epoch, st);
  p2p_red_sum_kernel<<<red_grid(na, nb), 256, 0, st>>>(
      reinterpret_cast<const float*>(w.base + w.off_red), w.P, w.n_red, a, na, b, nb);
  MOE_LAUNCH_CHECK("p2p_red_sum_kernel");
  count_launch();
}

void p2p_allreduce_f32(const P2PWindow& w, float* a, uint64_t na, float* b, uint64_t nb,
                       uint64_t epoch, cudaStream_t st) {
  p2p_allreduce_push(w, a, na, b, nb, epoch, st);
  p2p_allreduce_finish(w, a, na, b, nb, epoch, st);
}

unsigned persistent_grid(uint64_t T) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(T, 8), (uint64_t)num_sms() * 4));
}

void p2p_dispatch(const P2PWindow& w, uint64_t T, uint32_t d, uint32_t k, uint64_t C,
                  moe_dtype_t dt, const void* x, const int32_t* expert, const int32_t* position,
                  int32_t* slot, uint64_t epoch, cudaStream_t st) {
  const unsigned grid = persistent_grid(T);
  const bool v4 = w.row_bytes == 4 * 512;  // d = 1024 bf16 / 512 fp32: 4 pieces per lane
  if (dt == MOE_DTYPE_BF16) {
    if (v4)
      p2p_dispatch_kernel<__nv_bfloat16, 4><<<grid, 256, 0, st>>>(
          win_of(w), ctr_of(w, 0), T, d, k, C, (const __nv_bfloat16*)x, expert, position, slot, epoch);
    else
      p2p_dispatch_kernel<__nv_bfloat16, 0><<<grid, 256, 0, st>>>(
          win_of(w), ctr_of(w, 0), T, d, k, C, (const __nv_bfloat16*)x, expert, position, slot, epoch);
  } else {
    p2p_dispatch_kernel<float, 0><<<grid, 256, 0, st>>>(win_of(w), ctr_of(w, 0), T, d, k, C,
                                                        (const float*)x, expert, position, slot,
                                                        epoch);
  }
  MOE_LAUNCH_CHECK("p2p_dispatch_kernel");
  count_launch();
}

void p2p_local_groups(const P2PWindow& w, int32_t* gm, int32_t* ga, int32_t* gb, void* buf,
                      cudaStream_t st) {
  p2p_local_groups_kernel<<<w.El, 256, 0, st>>>(win_of(w), gm, ga, gb, static_cast<uint8_t*>(buf));
  MOE_LAUNCH_CHECK("p2p_local_groups_kernel");
  count_launch();
}

void p2p_combine_bwd(const P2PWindow& w, uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt,
                     const void* dy, const int32_t* slot, const float* gate,
                     const int32_t* expert, const int32_t* position, float* dgate, uint64_t epoch,
                     cudaStream_t st) {
  const unsigned grid = persistent_grid(T);
  if (dt == MOE_DTYPE_BF16)
    p2p_combine_bwd_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        win_of(w), w.off_yh, ctr_of(w, 1), T, d, k, (const __nv_bfloat16*)dy, slot, gate, expert,
        position, dgate, epoch);
  else
    p2p_combine_bwd_kernel<float><<<grid, 256, 0, st>>>(win_of(w), w.off_yh, ctr_of(w, 1), T, d, k,
                                                        (const float*)dy, slot, gate, expert,
                                                        position, dgate, epoch);
  MOE_LAUNCH_CHECK("p2p_combine_bwd_kernel");
  count_launch();
}

void p2p_push_home(const P2PWindow& w, uint64_t home_off, const void* src, int slot,
                   uint64_t epoch, cudaStream_t st) {
  dim3 grid(w.El * w.P, (unsigned)ceil_div(w.Cs, 64));
  p2p_push_kernel<<<grid, 256, 0, st>>>(win_of(w), home_off, ctr_of(w, slot == SLOT_Y ? 2 : 3),
                                        static_cast<const uint8_t*>(src), slot, epoch);
  MOE_LAUNCH_CHECK("p2p_push_kernel");
  count_launch();
}

}  // namespace moe
