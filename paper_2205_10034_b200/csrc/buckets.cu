// Gradient-bucket fusion for replicated parameters (paper
// PAPER.md:347-359): the semantics of the reference's GradBucket /
// make_gradient_buckets (collectives.cpp:120-162, pinned by
// test_collectives.cpp:174-233) — parameters registered in reverse layer order
// into buckets of at most `capacity`, a bucket flushes exactly once, when its
// last gradient arrives, with its payload in registration order — executed on
// the device: the flush packs the bucket's gradients into one flat fp32 buffer
// (one kernel, registration order), issues ONE ncclAllReduce on it, and
// unpacks (optionally scaled) on the caller's stream.  No host synchronisation.
#include <nccl.h>

#include <algorithm>
#include <string>
#include <unordered_map>
#include <vector>

#include "buckets.h"
#include "common.cuh"
#include "kernels.h"
#include "nccl_check.h"

namespace moe {

namespace {

// Copy every parameter of a bucket between its own storage and the flat buffer:
// block-strided over parameters, thread-strided within (float4 when aligned).
__global__ void bucket_copy_kernel(int nparam, float* const* ptrs, const uint64_t* numel,
                                   const uint64_t* offset, float* flat, int to_flat, float scale) {
  for (int q = blockIdx.y; q < nparam; q += gridDim.y) {
    float* p = ptrs[q];
    float* f = flat + offset[q];
    const uint64_t n = numel[q];
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(f)) & 15) == 0;
    if (vec) {
      const uint64_t n4 = n / 4;
      float4* p4 = reinterpret_cast<float4*>(p);
      float4* f4 = reinterpret_cast<float4*>(f);
      for (uint64_t i = t0; i < n4; i += stride) {
        if (to_flat) {
          f4[i] = p4[i];
        } else {
          float4 v = f4[i];
          v.x *= scale;
          v.y *= scale;
          v.z *= scale;
          v.w *= scale;
          p4[i] = v;
        }
      }
      for (uint64_t i = n4 * 4 + t0; i < n; i += stride) {
        if (to_flat) f[i] = p[i];
        else p[i] = f[i] * scale;
      }
    } else {
      for (uint64_t i = t0; i < n; i += stride) {
        if (to_flat) f[i] = p[i];
        else p[i] = f[i] * scale;
      }
    }
  }
}

}  // namespace

GradBuckets::GradBuckets(void* comm, uint32_t n, const uint64_t* ids_layer_order,
                         void* const* grads, const uint64_t* numel, uint32_t capacity, float scale)
    : comm_(comm), scale_(scale) {
  arg_check(capacity >= 1, "bucket: capacity must be >= 1");
  arg_check(n == 0 || ids_layer_order != nullptr, "bucket: ids must be non-null");
  arg_check((grads == nullptr) == (numel == nullptr), "bucket: grads and numel go together");
  device_ = grads != nullptr;
  // reverse layer order: gradients arrive back to front in the backward pass
  std::vector<uint32_t> cur;
  auto close = [&] {
    Bucket b;
    for (uint32_t q : cur) {
      b.ids.push_back(ids_layer_order[q]);
      if (device_) {
        arg_check(grads[q] != nullptr, "bucket: gradient pointer must be non-null");
        b.ptrs.push_back(static_cast<float*>(grads[q]));
        b.offset.push_back(b.total);
        b.numel.push_back(numel[q]);
        b.total += (numel[q] + 3) / 4 * 4;  // 16-byte aligned slices of the flat buffer
      }
    }
    b.arrived.assign(b.ids.size(), 0);
    b.missing = b.ids.size();
    buckets_.push_back(std::move(b));
    cur.clear();
  };
  for (uint32_t r = n; r-- > 0;) {
    cur.push_back(r);
    if (cur.size() == capacity) close();
  }
  if (!cur.empty()) close();
  for (uint32_t b = 0; b < buckets_.size(); ++b)
    for (uint32_t i = 0; i < buckets_[b].ids.size(); ++i) {
      const bool fresh = where_.emplace(buckets_[b].ids[i], std::make_pair(b, i)).second;
      arg_check(fresh, "bucket: gradient " + std::to_string(buckets_[b].ids[i]) +
                           " is registered twice");
    }
  if (device_) {
    for (Bucket& b : buckets_) {
      const size_t q = b.ptrs.size();
      MOE_CUDA(cudaMalloc(&b.flat, std::max<uint64_t>(b.total, 4) * sizeof(float)));
      MOE_CUDA(cudaMalloc(&b.d_ptrs, q * sizeof(float*)));
      MOE_CUDA(cudaMalloc(&b.d_numel, q * sizeof(uint64_t)));
      MOE_CUDA(cudaMalloc(&b.d_offset, q * sizeof(uint64_t)));
      MOE_CUDA(cudaMemcpy(b.d_ptrs, b.ptrs.data(), q * sizeof(float*), cudaMemcpyHostToDevice));
      MOE_CUDA(cudaMemcpy(b.d_numel, b.numel.data(), q * sizeof(uint64_t), cudaMemcpyHostToDevice));
      MOE_CUDA(
          cudaMemcpy(b.d_offset, b.offset.data(), q * sizeof(uint64_t), cudaMemcpyHostToDevice));
    }
  }
}

GradBuckets::~GradBuckets() {
  for (Bucket& b : buckets_) {
    cudaFree(b.flat);
    cudaFree(b.d_ptrs);
    cudaFree(b.d_numel);
    cudaFree(b.d_offset);
  }
}

int GradBuckets::push(uint64_t id, cudaStream_t st) {
  const auto it = where_.find(id);
  arg_check(it != where_.end(), "bucket: gradient " + std::to_string(id) + " is not registered");
  Bucket& b = buckets_[it->second.first];
  const uint32_t i = it->second.second;
  arg_check(!b.arrived[i], "bucket: duplicate push of gradient " + std::to_string(id));
  b.arrived[i] = 1;
  if (--b.missing > 0) return -1;
  b.flushed = true;
  if (device_) flush(b, st);
  return (int)it->second.first;
}

void GradBuckets::flush(Bucket& b, cudaStream_t st) {
  const int q = (int)b.ptrs.size();
  if (q == 0) return;
  const bool reduce = comm_ != nullptr;
  const dim3 grid(148, (unsigned)std::min(q, 65535));
  if (reduce) {
    bucket_copy_kernel<<<grid, 256, 0, st>>>(q, b.d_ptrs, b.d_numel, b.d_offset, b.flat, 1, 1.0f);
    MOE_LAUNCH_CHECK("bucket_copy_kernel(pack)");
    MOE_NCCL(ncclAllReduce(b.flat, b.flat, b.total, ncclFloat32, ncclSum, (ncclComm_t)comm_, st));
    bucket_copy_kernel<<<grid, 256, 0, st>>>(q, b.d_ptrs, b.d_numel, b.d_offset, b.flat, 0,
                                             scale_);
    MOE_LAUNCH_CHECK("bucket_copy_kernel(unpack)");
    count_launch(2);
  } else if (scale_ != 1.0f) {  // single rank: only the scale
    bucket_copy_kernel<<<grid, 256, 0, st>>>(q, b.d_ptrs, b.d_numel, b.d_offset, b.flat, 1, 1.0f);
    bucket_copy_kernel<<<grid, 256, 0, st>>>(q, b.d_ptrs, b.d_numel, b.d_offset, b.flat, 0,
                                             scale_);
    MOE_LAUNCH_CHECK("bucket_copy_kernel");
    count_launch(2);
  }
}

void GradBuckets::reset() {
  for (Bucket& b : buckets_) {
    std::fill(b.arrived.begin(), b.arrived.end(), 0);
    b.missing = b.ids.size();
    b.flushed = false;
  }
}

}  // namespace moe
