// NVLink peer-memory throughput by access method, one process driving every
// GPU (cudaDeviceEnablePeerAccess).  Each GPU sends `MB` MiB to every other GPU
// at once (all-to-all pattern of the EP exchange) or to one peer (pair):
//   ce      cudaMemcpyPeerAsync per destination (copy engines)
//   st      SM stores: warp per 2 KiB row, 16 B per lane, v4 stores to the peer
//   ld      SM loads: the receiver pulls rows from the peer, stores locally
//   bulk    TMA bulk copies: global -> smem (cp.async.bulk) -> peer global
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bw p2p_bw.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

constexpr int ROW = 2048;  // bytes per token row (d = 1024 bf16)

struct Dsts {
  uint4* p[8];
};

// rows [0, n) of src go round-robin to the destinations (row r -> dst r % nd,
// slot r / nd), like tokens routed to experts on different ranks
__global__ void push_rows(const uint4* __restrict__ src, Dsts d, int nd, long n) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long r = warp; r < n; r += nw) {
    const uint4* s = src + r * (ROW / 16);
    uint4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = s[lane + 32 * i];
    uint4* t = d.p[r % nd] + (r / nd) * (ROW / 16);
#pragma unroll
    for (int i = 0; i < 4; ++i) t[lane + 32 * i] = v[i];
  }
}

// receiver pulls: rows come from the sources round-robin
__global__ void pull_rows(Dsts s, int ns, uint4* __restrict__ dst, long n) {
  const int lane = threadIdx.x & 31;
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  for (long r = warp; r < n; r += nw) {
    const uint4* src = s.p[r % ns] + (r / ns) * (ROW / 16);
    uint4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = src[lane + 32 * i];
    uint4* t = dst + r * (ROW / 16);
#pragma unroll
    for (int i = 0; i < 4; ++i) t[lane + 32 * i] = v[i];
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// TMA bulk: each warp stages NB rows in smem with one elected lane issuing
// cp.async.bulk loads (mbarrier) and bulk stores to the peer
template <int NB>
__global__ void bulk_rows(const uint8_t* __restrict__ src, Dsts d, int nd, long n) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) unsigned long long bar[32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = sm + (size_t)wid * NB * ROW;
  const unsigned b = smem_u32(&bar[wid]);
  if (lane == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
  __syncwarp();
  const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  unsigned phase = 0;
  for (long r0 = warp * NB; r0 < n; r0 += nw * NB) {
    const int cnt = (int)((n - r0) < NB ? (n - r0) : NB);
    if (lane == 0) {
      // smem reuse: previous bulk stores must have read the buffer
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(cnt * ROW)
                   : "memory");
      for (int i = 0; i < cnt; ++i)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(buf + i * ROW)),
            "l"(src + (r0 + i) * ROW), "r"(ROW), "r"(b)
            : "memory");
      asm volatile(
          "{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(b),
          "r"(phase)
          : "memory");
      for (int i = 0; i < cnt; ++i) {
        const long r = r0 + i;
        uint8_t* t = reinterpret_cast<uint8_t*>(d.p[r % nd]) + (r / nd) * ROW;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(t),
                     "r"(smem_u32(buf + i * ROW)), "r"(ROW)
                     : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    phase ^= 1;
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char** argv) {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  const int G = argc > 1 ? atoi(argv[1]) : ng;
  const long MB = argc > 2 ? atol(argv[2]) : 64;  // MiB each GPU sends in total
  if (G < 2 || G > ng) {
    printf("need >= 2 GPUs (have %d)\n", ng);
    return 0;
  }
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long bytes = MB << 20, rows = bytes / ROW;
  std::vector<uint8_t*> src(G), dst(G);
  std::vector<cudaStream_t> st(G);
  std::vector<cudaEvent_t> e0(G), e1(G);
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int h = 0; h < G; ++h)
      if (h != g) CK(cudaDeviceEnablePeerAccess(h, 0));
    CK(cudaMalloc(&src[g], bytes));
    CK(cudaMalloc(&dst[g], bytes));  // receives bytes/(G-1) from every peer
    CK(cudaMemset(src[g], g + 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
    CK(cudaFuncSetAttribute(bulk_rows<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * ROW));
  }
  // destination of (src g -> dst h): region g' of h's receive buffer
  auto region = [&](int g, int h) {
    const int slot = g < h ? g : g - 1;
    return dst[h] + (long)slot * (bytes / (G - 1));
  };
  auto run = [&](const char* name, int mode, int blocks_per_sm, int pair) {
    const int peers = pair ? 1 : G - 1;
    float worst = 0;
    for (int rep = 0; rep < 4; ++rep) {
      for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaDeviceSynchronize());
      }
      for (int g = 0; g < G; ++g) {
        if (pair && g != 0) continue;
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        Dsts d{};
        int nd = 0, dev[8];
        for (int h = 0; h < G && nd < peers; ++h)
          if (h != g) dev[nd] = h, d.p[nd++] = reinterpret_cast<uint4*>(region(g, h));
        const long n = pair ? rows / (G - 1) : rows;  // pair: one peer's share
        const int grid = sms * blocks_per_sm;
        if (mode == 0) {
          for (int i = 0; i < nd; ++i)
            CK(cudaMemcpyPeerAsync(d.p[i], dev[i], src[g] + (long)i * (bytes / (G - 1)), g,
                                   bytes / (G - 1), st[g]));
        } else if (mode == 1) {
          push_rows<<<grid, 256, 0, st[g]>>>(reinterpret_cast<uint4*>(src[g]), d, nd, n);
        } else if (mode == 2) {
          // pull: g reads its share from every peer's source
          Dsts s{};
          int ns = 0;
          for (int h = 0; h < G && ns < peers; ++h)
            if (h != g) s.p[ns++] = reinterpret_cast<uint4*>(src[h]);
          pull_rows<<<grid, 256, 0, st[g]>>>(s, ns, reinterpret_cast<uint4*>(dst[g]), n);
        } else {
          bulk_rows<4><<<grid, 256, 8 * 4 * ROW, st[g]>>>(src[g], d, nd, n);
        }
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1[g], st[g]));
      }
      for (int g = 0; g < G; ++g) {
        if (pair && g != 0) continue;
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        if (rep > 0 && ms > worst) worst = ms;
      }
    }
    const double sent = pair ? (double)bytes / (G - 1) : (double)bytes;
    printf("{\"gpus\": %d, \"pattern\": \"%s\", \"method\": \"%s\", \"blocks_per_sm\": %d, "
           "\"MiB_per_gpu\": %.0f, \"ms\": %.4f, \"GBps_per_gpu\": %.1f}\n",
           G, pair ? "pair" : "all-to-all", name, blocks_per_sm, sent / (1 << 20), worst,
           sent / worst / 1e6);
  };
  for (int pair = 1; pair >= 0; --pair) {
    run("ce", 0, 1, pair);
    for (int b : {1, 2, 4, 8}) run("st", 1, b, pair);
    for (int b : {1, 2, 4, 8}) run("ld", 2, b, pair);
    for (int b : {1, 2}) run("bulk", 3, b, pair);
  }
  return 0;
}
