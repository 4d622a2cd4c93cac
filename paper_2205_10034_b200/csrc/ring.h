// Ring-of-sections runner (K7) behind moe_ring_t.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "moe_b200.h"

namespace moe {

struct Layer;

struct SectionLayout {
  uint64_t w1 = 0, b1 = 0, w2 = 0, b2 = 0, bytes = 0;
};
SectionLayout section_layout(const Layer& L);

// out = a + b elementwise (the residual of a stacked MoE layer)
void residual_add(moe_dtype_t dt, const void* a, const void* b, void* out, uint64_t n,
                  cudaStream_t st);

// build_schedule (ring_offload.cpp:31-50): kind 0 load, 1 compute, 2 release.
struct RingOpRec {
  int kind;
  uint32_t layer;
  uint32_t slot;
  int64_t waits;  // layer whose release frees the slot, or -1
};
std::vector<RingOpRec> ring_schedule(uint32_t layers, uint32_t ring_slots, uint32_t* slots,
                                     bool* clamped);

struct Ring {
  Ring(Layer* layer, const moe_ring_desc_t& d);
  ~Ring();
  void run(const void* x, void* y, moe_ring_timeline_t* tl, cudaStream_t st);
  uint64_t dense_bytes() const;

  Layer* L;
  uint32_t N = 0, K = 0;
  bool clamped = false;
  std::vector<RingOpRec> ops;
  SectionLayout lay;
  std::vector<const void*> host;
  std::vector<const void*> wg;
  std::vector<const float*> bg;
  std::vector<void*> slots;
  void* hbuf[2] = {nullptr, nullptr};
  void* tmp = nullptr;
  cudaStream_t copy = nullptr;
  std::vector<cudaEvent_t> ev_load0, ev_load1, ev_comp0, ev_comp1;
  cudaEvent_t ev_start = nullptr;
};

}  // namespace moe
