// 2D prefetch executor with the Algorithm-1 CPU cache (prefetch.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "moe_b200.h"
#include "ring.h"
#include "sparse_cache.h"

namespace moe {

struct Layer;

struct Prefetch2D {
  Prefetch2D(Layer* layer, const moe_prefetch_desc_t& d);
  ~Prefetch2D();
  void run(uint32_t steps, const void* x, void* y, moe_prefetch_record_t* recs,
           moe_prefetch_summary_t* sum, cudaStream_t st);

  struct Block {
    void* ptr = nullptr;            // pinned host copy of the layer's section
    cudaEvent_t last = nullptr;     // H2D that last read it (pending or done)
  };
  void read_block(uint32_t b, void* dst);
  void write_block(uint32_t b, const void* src);
  cudaEvent_t event();

  Layer* L;
  SparseCache cache;
  uint32_t N = 0, lookahead = 1, K = 2, flush_period = 1;
  SectionLayout lay;
  std::vector<const void*> wg;
  std::string path;
  int fd = -1;
  std::map<uint32_t, Block> blocks;  // CPU cache contents
  void* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_last[2] = {nullptr, nullptr};
  uint64_t stream_count = 0;
  std::vector<void*> gslots;
  void* hbuf[2] = {nullptr, nullptr};
  void* tmp = nullptr;
  cudaStream_t copy = nullptr;
  cudaEvent_t ev_start = nullptr;
  std::vector<cudaEvent_t> evs;
  uint64_t bytes_read = 0, bytes_written = 0;
};

}  // namespace moe
