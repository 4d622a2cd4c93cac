// HBM write bandwidth by store method (what bounds the write-heavy GEMM
// epilogues): 1 GiB per pass, persistent grid of SMs x blocks.
//   v4        st.global.v4 (default policy)
//   v4.cs     st.global.cs.v4 (streaming / evict-first)
//   bulk      TMA bulk store smem -> global (cp.async.bulk.global.shared::cta),
//             16 KiB per op, 4 in flight per block
//   memset    cudaMemsetAsync
//   copy      st.global.v4 of a read stream (read + write, for reference)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hbm_write hbm_write.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void st_v4(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = v;
}

__global__ void st_v4_cs(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, v);
}

__global__ void copy_v4(const uint4* __restrict__ a, uint4* __restrict__ p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = a[i];
}

constexpr int CHUNK = 16384, INFL = 4;
__global__ void bulk_store(uint8_t* p, size_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  for (int i = threadIdx.x; i < CHUNK * INFL / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  int k = 0;
  for (size_t off = (size_t)blockIdx.x * CHUNK; off < bytes; off += (size_t)gridDim.x * CHUNK) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(sm + (k % INFL) * CHUNK);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off),
                 "r"(s), "r"(CHUNK)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(INFL - 1) : "memory");
    ++k;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 1ull << 30, n = bytes / 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint8_t *p, *a;
  CK(cudaMalloc(&p, bytes));
  CK(cudaMalloc(&a, bytes));
  CK(cudaMemset(a, 1, bytes));
  CK(cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, CHUNK * INFL));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, int bps, int threads, auto fn, double traffic) {
    for (int i = 0; i < 3; ++i) fn(bps, threads);
    CK(cudaEventRecord(e0));
    const int reps = 10;
    for (int i = 0; i < reps; ++i) fn(bps, threads);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    printf("{\"method\": \"%s\", \"blocks_per_sm\": %d, \"threads\": %d, \"us\": %.1f, \"GBps\": %.0f}\n",
           name, bps, threads, ms * 1e3, traffic / ms / 1e6);
  };
  for (int bps : {1, 2, 4, 8}) {
    run("v4", bps, 512, [&](int b, int t) { st_v4<<<sms * b, t>>>((uint4*)p, n); }, bytes);
    run("v4.cs", bps, 512, [&](int b, int t) { st_v4_cs<<<sms * b, t>>>((uint4*)p, n); }, bytes);
    run("copy(r+w)", bps, 512,
        [&](int b, int t) { copy_v4<<<sms * b, t>>>((const uint4*)a, (uint4*)p, n); }, 2.0 * bytes);
  }
  for (int bps : {1, 2, 3})
    run("bulk", bps, 128,
        [&](int b, int t) { bulk_store<<<sms * b, t, CHUNK * INFL>>>(p, bytes); }, bytes);
  run("memset", 0, 0, [&](int, int) { CK(cudaMemsetAsync(p, 0, bytes)); }, bytes);
  CK(cudaGetLastError());
  return 0;
}
