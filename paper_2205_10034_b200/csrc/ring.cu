// K7 — ring-of-sections inference (§3.3 "Ring Memory"; reference
// ring_offload.hpp:16-64, ring_offload.cpp:31-117).
//
// The reference simulates the calculation-release-load rotation on an α-β
// timing model; here it runs for real: N layers' expert sections live in
// pinned host memory, K HBM slots rotate through them, loads run on a copy
// stream (PCIe H2D, copy engine — no SMs), computes on the caller's stream,
// and events enforce exactly the reference's dependencies:
//   load(i)    waits release(i-K)              (ring_offload.cpp:44-47)
//   compute(i) waits load(i)                   (ring_offload.cpp:84-87)
//   release(i) = completion of compute(i)      (ring_offload.cpp:88-91)
// The recorded event timeline gives the same metrics the reference reports
// (report.cpp:172-187): makespan, stall vs compute-only, peak vs baseline bytes.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "layer.h"
#include "ring.h"

namespace moe {

namespace {
template <typename T>
__global__ void residual_add_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                    T* __restrict__ out, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (T)((float)a[i] + (float)b[i]);
}
uint64_t align256(uint64_t x) { return (x + 255) & ~uint64_t(255); }
}  // namespace

void residual_add(moe_dtype_t dt, const void* a, const void* b, void* out, uint64_t n,
                  cudaStream_t st) {
  const unsigned grid = (unsigned)std::min<uint64_t>(ceil_div(n, 256), 148ull * 8);
  if (dt == MOE_DTYPE_BF16)
    residual_add_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
        (const __nv_bfloat16*)a, (const __nv_bfloat16*)b, (__nv_bfloat16*)out, n);
  else
    residual_add_kernel<float><<<grid, 256, 0, st>>>((const float*)a, (const float*)b,
                                                     (float*)out, n);
  MOE_LAUNCH_CHECK("residual_add_kernel");
  count_launch();
}

SectionLayout section_layout(const Layer& L) {
  SectionLayout s;
  s.w1 = 0;
  s.b1 = align256(s.w1 + (uint64_t)L.El * L.dff * L.dm * L.esz);
  s.w2 = align256(s.b1 + (uint64_t)L.El * L.dff * 4);
  s.b2 = align256(s.w2 + (uint64_t)L.El * L.dm * L.dff * L.esz);
  s.bytes = align256(s.b2 + (uint64_t)L.El * L.dm * 4);
  return s;
}

std::vector<RingOpRec> ring_schedule(uint32_t layers, uint32_t ring_slots, uint32_t* slots,
                                     bool* clamped) {
  config_check(layers >= 1, "ring.num_layers: must be >= 1");
  config_check(ring_slots != 0, "ring.ring_slots: must be >= 1");
  const uint32_t K = std::min(ring_slots, layers);
  *slots = K;
  *clamped = ring_slots > layers;
  std::vector<RingOpRec> ops;
  for (uint32_t i = 0; i < K; ++i) ops.push_back({0, i, i % K, -1});
  for (uint32_t i = 0; i < layers; ++i) {
    ops.push_back({1, i, i % K, -1});
    ops.push_back({2, i, i % K, -1});
    if (i + K < layers) ops.push_back({0, i + K, (i + K) % K, (int64_t)i});
  }
  return ops;
}

Ring::Ring(Layer* layer, const moe_ring_desc_t& d) : L(layer) {
  config_check(d.num_layers >= 1, "ring.num_layers: must be >= 1");
  config_check(d.ring_slots != 0, "ring.ring_slots: must be >= 1");
  arg_check(d.host_sections != nullptr && d.gate_weights != nullptr,
            "ring.host_sections/gate_weights: must be non-null");
  N = d.num_layers;
  ops = ring_schedule(N, d.ring_slots, &K, &clamped);
  lay = section_layout(*L);
  host.assign(d.host_sections, d.host_sections + N);
  wg.assign(d.gate_weights, d.gate_weights + N);
  bg.assign(N, nullptr);
  if (d.gate_bias) bg.assign(d.gate_bias, d.gate_bias + N);
  slots.resize(K);
  for (uint32_t s = 0; s < K; ++s) MOE_CUDA(cudaMalloc(&slots[s], lay.bytes));
  const uint64_t act = L->T * L->dm * L->esz;
  MOE_CUDA(cudaMalloc(&hbuf[0], act));
  MOE_CUDA(cudaMalloc(&hbuf[1], act));
  MOE_CUDA(cudaMalloc(&tmp, act));
  MOE_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
  ev_load0.resize(N);
  ev_load1.resize(N);
  ev_comp0.resize(N);
  ev_comp1.resize(N);
  for (uint32_t i = 0; i < N; ++i) {
    MOE_CUDA(cudaEventCreate(&ev_load0[i]));
    MOE_CUDA(cudaEventCreate(&ev_load1[i]));
    MOE_CUDA(cudaEventCreate(&ev_comp0[i]));
    MOE_CUDA(cudaEventCreate(&ev_comp1[i]));
  }
  MOE_CUDA(cudaEventCreate(&ev_start));
}

Ring::~Ring() {
  for (void* p : slots) cudaFree(p);
  cudaFree(hbuf[0]);
  cudaFree(hbuf[1]);
  cudaFree(tmp);
  for (uint32_t i = 0; i < N; ++i) {
    cudaEventDestroy(ev_load0[i]);
    cudaEventDestroy(ev_load1[i]);
    cudaEventDestroy(ev_comp0[i]);
    cudaEventDestroy(ev_comp1[i]);
  }
  cudaEventDestroy(ev_start);
  cudaStreamDestroy(copy);
}

void Ring::run(const void* x, void* y, moe_ring_timeline_t* tl, cudaStream_t st) {
  const uint64_t n = L->T * L->dm;
  const uint64_t act = n * L->esz;
  MOE_CUDA(cudaEventRecord(ev_start, st));
  MOE_CUDA(cudaStreamWaitEvent(copy, ev_start, 0));
  MOE_CUDA(cudaMemcpyAsync(hbuf[0], x, act, cudaMemcpyDeviceToDevice, st));
  int cur = 0;
  for (const RingOpRec& op : ops) {
    const uint32_t i = op.layer;
    if (op.kind == 0) {  // load
      if (op.waits >= 0) MOE_CUDA(cudaStreamWaitEvent(copy, ev_comp1[op.waits], 0));
      MOE_CUDA(cudaEventRecord(ev_load0[i], copy));
      MOE_CUDA(cudaMemcpyAsync(slots[op.slot], host[i], lay.bytes, cudaMemcpyHostToDevice, copy));
      MOE_CUDA(cudaEventRecord(ev_load1[i], copy));
    } else if (op.kind == 1) {  // compute
      MOE_CUDA(cudaStreamWaitEvent(st, ev_load1[i], 0));
      MOE_CUDA(cudaEventRecord(ev_comp0[i], st));
      const uint8_t* s = static_cast<const uint8_t*>(slots[op.slot]);
      moe_layer_params_t w;
      w.wg = wg[i];
      w.bg = bg[i];
      w.w1 = s + lay.w1;
      w.b1 = reinterpret_cast<const float*>(s + lay.b1);
      w.w2 = s + lay.w2;
      w.b2 = reinterpret_cast<const float*>(s + lay.b2);
      L->forward(w, hbuf[cur], tmp, nullptr, nullptr, nullptr, st);
      residual_add(L->dt, hbuf[cur], tmp, hbuf[cur ^ 1], n, st);
      cur ^= 1;
      MOE_CUDA(cudaEventRecord(ev_comp1[i], st));  // release(i): slot free once compute(i) ends
    }
  }
  MOE_CUDA(cudaMemcpyAsync(y, hbuf[cur], act, cudaMemcpyDeviceToDevice, st));
  if (tl) {
    MOE_CUDA(cudaStreamSynchronize(st));
    MOE_CUDA(cudaStreamSynchronize(copy));
    float mk = 0.f, comp = 0.f;
    for (uint32_t i = 0; i < N; ++i) {
      float a, b, c, e;
      MOE_CUDA(cudaEventElapsedTime(&a, ev_start, ev_load0[i]));
      MOE_CUDA(cudaEventElapsedTime(&b, ev_start, ev_load1[i]));
      MOE_CUDA(cudaEventElapsedTime(&c, ev_start, ev_comp0[i]));
      MOE_CUDA(cudaEventElapsedTime(&e, ev_start, ev_comp1[i]));
      if (tl->load_start) tl->load_start[i] = a;
      if (tl->load_end) tl->load_end[i] = b;
      if (tl->compute_start) tl->compute_start[i] = c;
      if (tl->compute_end) tl->compute_end[i] = e;
      mk = std::max(mk, std::max(b, e));
      comp += e - c;
    }
    tl->makespan_ms = mk;
    tl->compute_total_ms = comp;
    tl->peak_gpu_bytes = dense_bytes() + (uint64_t)K * lay.bytes;
    tl->baseline_gpu_bytes = dense_bytes() + (uint64_t)N * lay.bytes;
    tl->slots = K;
    tl->clamped = clamped ? 1 : 0;
  }
}

uint64_t Ring::dense_bytes() const {
  // resident dense parameters: the N gates (+ biases)
  return (uint64_t)N * ((uint64_t)L->E * L->dm * L->esz + (L->desc.has_gate_bias ? L->E * 4 : 0));
}

}  // namespace moe
