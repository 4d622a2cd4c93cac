// Gradient-bucket fusion (buckets.cu): GradBucket semantics on the host,
// pack -> one ncclAllReduce -> unpack per flushed bucket on the device.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <unordered_map>
#include <utility>
#include <vector>

namespace moe {

class GradBuckets {
 public:
  // ids in layer order; grads/numel (fp32 device buffers) may both be null for
  // a host-only container (bookkeeping without device work).  comm null: one
  // rank (no all-reduce; scale still applied).
  GradBuckets(void* comm, uint32_t n, const uint64_t* ids_layer_order, void* const* grads,
              const uint64_t* numel, uint32_t capacity, float scale);
  ~GradBuckets();
  // -1: held; else the index of the bucket this push flushed (its all-reduce is
  // enqueued on st).  Duplicate / unknown ids throw invalid_argument.
  int push(uint64_t id, cudaStream_t st);
  void reset();
  uint32_t count() const { return (uint32_t)buckets_.size(); }
  const std::vector<uint64_t>& ids(uint32_t b) const { return buckets_[b].ids; }
  bool flushed(uint32_t b) const { return buckets_[b].flushed; }

 private:
  struct Bucket {
    std::vector<uint64_t> ids;  // registration order
    std::vector<char> arrived;
    size_t missing = 0;
    bool flushed = false;
    std::vector<float*> ptrs;
    std::vector<uint64_t> numel, offset;
    uint64_t total = 0;
    float* flat = nullptr;
    float** d_ptrs = nullptr;
    uint64_t *d_numel = nullptr, *d_offset = nullptr;
  };
  void flush(Bucket& b, cudaStream_t st);
  void* comm_;
  float scale_;
  bool device_ = false;
  std::vector<Bucket> buckets_;
  std::unordered_map<uint64_t, std::pair<uint32_t, uint32_t>> where_;
};

}  // namespace moe
