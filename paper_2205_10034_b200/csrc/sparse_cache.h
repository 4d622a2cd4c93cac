// Algorithm-1 CPU cache policy for sparse parameter blocks (sparse_cache.cu).
#pragma once

#include <cstdint>
#include <map>
#include <set>
#include <utility>

#include "moe_b200.h"

namespace moe {

class SparseCache {
 public:
  explicit SparseCache(const moe_cache_params_t& p);
  moe_cache_access_t access(uint64_t block);
  void end_step();
  double hits(uint64_t block) const;  // 0 when not resident
  uint64_t occupancy() const { return occupancy_; }
  uint32_t steps() const { return steps_; }
  const std::map<uint64_t, double>& counts() const { return count_; }  // sorted by id

 private:
  void admit(uint64_t block);
  moe_cache_params_t p_;
  std::map<uint64_t, double> count_;              // resident block -> hit count
  std::set<std::pair<double, uint64_t>> order_;   // (count, id): coldest first
  uint64_t occupancy_ = 0;                        // blocks admitted fresh
  uint32_t steps_ = 0;
};

}  // namespace moe
