// Algorithm-1 CPU cache for sparse (expert) parameter blocks — SE-MoE's
// 2D-prefetch cache policy, with the semantics of the
// reference's SparseCache (prefetch_cache.hpp:43-83, prefetch_cache.cpp:28-64,
// pinned by test_prefetch_cache.cpp:77-236 and tests/golden): on access(b)
//   resident                  -> hit count += 1                  (CacheHit)
//   occupancy + 1 < cpu_size  -> admit with count 1              (FetchedFresh)
//   coldest resident count >= threshold (ties: lowest id)
//                             -> evict it, admit b with count 1  (EvictedAndFetched)
//   otherwise                 -> serve without caching           (StreamThrough)
// and every decay_steps calls of end_step() all counts are multiplied by beta.
// Host-side policy object: it decides which expert sections the GPU prefetch
// pipeline reads from pinned host memory and which from the backing store.
#include <map>
#include <set>
#include <utility>

#include "common.cuh"
#include "sparse_cache.h"

namespace moe {

SparseCache::SparseCache(const moe_cache_params_t& p) : p_(p) {
  config_check(p.beta > 0.0 && p.beta <= 1.0, "cache.beta: must be in (0, 1]");
  config_check(p.decay_steps >= 1, "cache.decay_steps: must be >= 1");
  config_check(p.threshold >= 0.0, "cache.threshold: must be >= 0");
}

moe_cache_access_t SparseCache::access(uint64_t block) {
  auto it = count_.find(block);
  if (it != count_.end()) {
    order_.erase({it->second, block});
    it->second += 1.0;
    order_.insert({it->second, block});
    return {MOE_CACHE_HIT, 0};
  }
  if (occupancy_ + 1 < p_.cpu_size) {
    admit(block);
    ++occupancy_;
    return {MOE_CACHE_FETCHED_FRESH, 0};
  }
  if (!order_.empty() && order_.begin()->first >= p_.threshold) {
    const uint64_t victim = order_.begin()->second;
    order_.erase(order_.begin());
    count_.erase(victim);
    admit(block);
    return {MOE_CACHE_EVICTED_AND_FETCHED, victim};
  }
  return {MOE_CACHE_STREAM_THROUGH, 0};
}

void SparseCache::admit(uint64_t block) {
  count_[block] = 1.0;
  order_.insert({1.0, block});
}

void SparseCache::end_step() {
  if (++steps_ < p_.decay_steps) return;
  steps_ = 0;
  order_.clear();
  for (auto& [block, c] : count_) {
    c *= p_.beta;
    order_.insert({c, block});
  }
}

double SparseCache::hits(uint64_t block) const {
  const auto it = count_.find(block);
  return it == count_.end() ? 0.0 : it->second;
}

}  // namespace moe
