// moesim_b200.hpp — C++ drop-in for the reference's hot-path API.
//
// Restores the value-type signatures and exception types of
// /root/reference/proj/core/include/moesim/{collectives,workload,ring_offload}.hpp
// on top of the C-ABI in moe_b200.h (executed by libmoe_b200.so on the GPU).
// A caller of moesim::alltoall_flat / fuse_slices / split_blob / gen_trace /
// imbalance_ratio / build_schedule recompiles against this header and links
// libmoe_b200.so instead of moesim::core.
//
//   reference                                   here
//   collectives.hpp:36   alltoall_flat          moesim::alltoall_flat
//   collectives.hpp:54-55 alltoall_hierarchical  moesim::alltoall_hierarchical (+ AlltoAllStats)
//   topology.hpp:15-60   LinkClass/GpuId/Topology moesim::Topology (shape, route; no timing)
//   collectives.hpp:78-79 fuse_slices/split_blob moesim::fuse_slices / split_blob
//   workload.hpp:41-46   gen_trace/imbalance     moesim::gen_trace / imbalance_ratio
//   ring_offload.hpp:45  build_schedule          moesim::build_schedule
//   prefetch_cache.hpp:18-83 SparseCache          moesim::SparseCache (Algorithm-1 policy)
//   types.hpp:24-26      ConfigError             moesim::ConfigError
#pragma once

#include <array>
#include <cstdint>
#include <map>
#include <numeric>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "moe_b200.h"

namespace moesim {

using Bytes = std::uint64_t;
using Count = std::uint64_t;
using Chunk = std::vector<std::uint8_t>;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(moe_status_t s) {
  if (s == MOE_OK) return;
  const std::string msg = moe_last_error();
  switch (s) {
    case MOE_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case MOE_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case MOE_ERR_CONFIG: throw ConfigError(msg);
    case MOE_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

// collectives.hpp:19-33
struct ShardedPayload {
  std::size_t ranks = 0;
  std::vector<Chunk> chunks;  // row-major [src][dst]
  static ShardedPayload make(std::size_t ranks) {
    ShardedPayload p;
    p.ranks = ranks;
    p.chunks.resize(ranks * ranks);
    return p;
  }
  Chunk& at(std::size_t s, std::size_t d) { return chunks[s * ranks + d]; }
  const Chunk& at(std::size_t s, std::size_t d) const { return chunks[s * ranks + d]; }
  friend bool operator==(const ShardedPayload&, const ShardedPayload&) = default;
};

inline ShardedPayload alltoall_flat(const ShardedPayload& payload) {
  const std::size_t n = payload.chunks.size();
  std::vector<std::uint64_t> lens(n), out_lens(n);
  Chunk data;
  for (std::size_t i = 0; i < n; ++i) {
    lens[i] = payload.chunks[i].size();
    data.insert(data.end(), payload.chunks[i].begin(), payload.chunks[i].end());
  }
  Chunk out(data.size());
  detail::check(moesim_alltoall_flat(payload.ranks, n, lens.data(), data.data(), out_lens.data(),
                                     out.data()));
  ShardedPayload res = ShardedPayload::make(payload.ranks);
  std::size_t o = 0;
  for (std::size_t i = 0; i < n; ++i) {
    res.chunks[i].assign(out.begin() + o, out.begin() + o + out_lens[i]);
    o += out_lens[i];
  }
  return res;
}

// topology.hpp:15-60 — the shape and routing half of moesim::Topology (the
// alpha-beta timing model belongs to the simulator, out of scope here).
enum class LinkClass : std::uint8_t { kNvlink, kPcie, kSsdIo, kTor, kLeaf, kSpin };
inline constexpr std::size_t kLinkClassCount = 6;
using Path = std::vector<LinkClass>;
struct LinkParams {
  Bytes bandwidth_bytes_per_sec = 0;
  std::int64_t latency_ns = 0;
};
struct GpuId {
  std::uint32_t cluster = 0, node = 0, local_rank = 0;
  friend bool operator==(const GpuId&, const GpuId&) = default;
};

class Topology {
 public:
  Topology(std::uint32_t clusters, std::uint32_t nodes_per_cluster, std::uint32_t gpus_per_node,
           const std::array<LinkParams, kLinkClassCount>& links = flat())
      : clusters_(clusters), nodes_(nodes_per_cluster), gpus_(gpus_per_node), links_(links) {
    if (!clusters_) throw ConfigError("topology.clusters: must be >= 1");
    if (!nodes_) throw ConfigError("topology.nodes_per_cluster: must be >= 1");
    if (!gpus_) throw ConfigError("topology.gpus_per_node: must be >= 1");
    static const char* names[kLinkClassCount] = {"nvlink", "pcie", "ssd_io", "tor", "leaf", "spin"};
    for (std::size_t i = 0; i < kLinkClassCount; ++i) {
      if (!links_[i].bandwidth_bytes_per_sec)
        throw ConfigError(std::string("topology.links.") + names[i] +
                          ".bandwidth_bytes_per_sec: must be > 0");
      if (links_[i].latency_ns < 0)
        throw ConfigError(std::string("topology.links.") + names[i] + ".latency_ns: must be >= 0");
    }
  }
  std::uint32_t clusters() const { return clusters_; }
  std::uint32_t nodes_per_cluster() const { return nodes_; }
  std::uint32_t gpus_per_node() const { return gpus_; }
  std::uint32_t total_gpus() const { return clusters_ * nodes_ * gpus_; }
  const LinkParams& link(LinkClass c) const { return links_[static_cast<std::size_t>(c)]; }
  std::uint32_t global_rank(const GpuId& g) const {
    return (g.cluster * nodes_ + g.node) * gpus_ + g.local_rank;
  }
  GpuId gpu(std::uint32_t r) const {
    if (r >= total_gpus()) throw std::out_of_range("topology: global rank out of range");
    const std::uint32_t ni = r / gpus_;
    return GpuId{ni / nodes_, ni % nodes_, r % gpus_};
  }
  bool valid(const GpuId& g) const {
    return g.cluster < clusters_ && g.node < nodes_ && g.local_rank < gpus_;
  }
  Path route(const GpuId& s, const GpuId& d) const {
    if (!valid(s)) throw std::out_of_range("topology.route: invalid src GPU id");
    if (!valid(d)) throw std::out_of_range("topology.route: invalid dst GPU id");
    if (s == d) return {};
    if (s.cluster == d.cluster && s.node == d.node) return {LinkClass::kNvlink};
    if (s.local_rank == d.local_rank) return {LinkClass::kTor, LinkClass::kLeaf, LinkClass::kTor};
    return {LinkClass::kTor, LinkClass::kLeaf, LinkClass::kSpin, LinkClass::kLeaf,
            LinkClass::kTor};
  }

 private:
  static std::array<LinkParams, kLinkClassCount> flat() {
    std::array<LinkParams, kLinkClassCount> l{};
    for (auto& x : l) x.bandwidth_bytes_per_sec = 1;
    return l;
  }
  std::uint32_t clusters_, nodes_, gpus_;
  std::array<LinkParams, kLinkClassCount> links_;
};

// collectives.hpp:38-47
struct AlltoAllStats {
  std::array<std::size_t, kLinkClassCount> phase1_hops{};
  std::array<std::size_t, kLinkClassCount> phase2_hops{};
  std::size_t phase1_transfers = 0;
  std::size_t phase2_transfers = 0;
  std::size_t hops(LinkClass c) const {
    return phase1_hops[static_cast<std::size_t>(c)] + phase2_hops[static_cast<std::size_t>(c)];
  }
};

// collectives.hpp:54-55; both phases execute on the GPU
inline ShardedPayload alltoall_hierarchical(const ShardedPayload& payload,
                                            const Topology& topology,
                                            AlltoAllStats* stats = nullptr) {
  const std::size_t n = payload.chunks.size();
  std::vector<std::uint64_t> lens(n), out_lens(n), st(14);
  Chunk data;
  for (std::size_t i = 0; i < n; ++i) {
    lens[i] = payload.chunks[i].size();
    data.insert(data.end(), payload.chunks[i].begin(), payload.chunks[i].end());
  }
  Chunk out(data.size());
  detail::check(moesim_alltoall_hierarchical(
      topology.clusters(), topology.nodes_per_cluster(), topology.gpus_per_node(), payload.ranks,
      n, lens.data(), data.data(), out_lens.data(), out.data(), st.data()));
  if (stats) {
    for (std::size_t i = 0; i < kLinkClassCount; ++i) {
      stats->phase1_hops[i] += st[i];
      stats->phase2_hops[i] += st[6 + i];
    }
    stats->phase1_transfers += st[12];
    stats->phase2_transfers += st[13];
  }
  ShardedPayload res = ShardedPayload::make(payload.ranks);
  std::size_t o = 0;
  for (std::size_t i = 0; i < n; ++i) {
    res.chunks[i].assign(out.begin() + o, out.begin() + o + out_lens[i]);
    o += out_lens[i];
  }
  return res;
}

// collectives.hpp:60-79
struct SliceIndexEntry {
  std::size_t slice_id = 0;
  std::size_t offset = 0;
  std::size_t length = 0;
  friend bool operator==(const SliceIndexEntry&, const SliceIndexEntry&) = default;
};
using SliceIndex = std::vector<SliceIndexEntry>;
struct FusedBlob {
  Chunk blob;
  SliceIndex index;
};

inline FusedBlob fuse_slices(const std::vector<Chunk>& slices) {
  std::vector<std::uint64_t> lens(slices.size());
  Chunk data;
  for (std::size_t i = 0; i < slices.size(); ++i) {
    lens[i] = slices[i].size();
    data.insert(data.end(), slices[i].begin(), slices[i].end());
  }
  FusedBlob f;
  f.blob.resize(data.size());
  std::vector<moe_slice_index_entry_t> idx(slices.size());
  detail::check(moesim_fuse_slices(slices.size(), lens.data(), data.data(), f.blob.data(),
                                   idx.data()));
  for (const auto& e : idx) f.index.push_back({e.slice_id, e.offset, e.length});
  return f;
}

inline std::vector<Chunk> split_blob(const Chunk& blob, const SliceIndex& index) {
  std::vector<moe_slice_index_entry_t> idx;
  for (const auto& e : index) idx.push_back({e.slice_id, e.offset, e.length});
  Chunk out(blob.size());
  detail::check(moesim_split_blob(blob.size(), blob.data(), idx.size(), idx.data(), out.data()));
  std::vector<Chunk> slices;
  std::size_t o = 0;
  for (const auto& e : index) {
    slices.emplace_back(out.begin() + o, out.begin() + o + e.length);
    o += e.length;
  }
  return slices;
}

// workload.hpp:14-46
struct RoutingTrace {
  std::uint32_t steps = 0, ranks = 0, experts = 0;
  Count tokens_per_rank = 0;
  std::vector<Count> counts;  // [step][rank][expert]
  Count at(std::uint32_t s, std::uint32_t r, std::uint32_t e) const {
    return counts[(static_cast<std::size_t>(s) * ranks + r) * experts + e];
  }
  Count expert_total(std::uint32_t e) const {
    Count t = 0;
    for (std::uint32_t s = 0; s < steps; ++s)
      for (std::uint32_t r = 0; r < ranks; ++r) t += at(s, r, e);
    return t;
  }
};

inline RoutingTrace gen_trace(std::uint64_t seed, std::uint32_t steps, std::uint32_t ranks,
                              std::uint32_t experts, Count tokens_per_rank, double skew) {
  RoutingTrace t;
  t.steps = steps;
  t.ranks = ranks;
  t.experts = experts;
  t.tokens_per_rank = tokens_per_rank;
  t.counts.assign(static_cast<std::size_t>(steps) * ranks * experts, 0);
  detail::check(moesim_gen_trace(seed, steps, ranks, experts, tokens_per_rank, skew,
                                 t.counts.data()));
  return t;
}

inline double imbalance_ratio(const RoutingTrace& trace) {
  double out = 0.0;
  detail::check(moesim_imbalance_ratio(trace.steps, trace.ranks, trace.experts,
                                       trace.counts.data(), &out));
  return out;
}

// ring_offload.hpp:16-45
struct RingOp {
  enum class Kind : std::uint8_t { kLoad, kCompute, kRelease };
  Kind kind = Kind::kLoad;
  std::uint32_t layer = 0;
  std::uint32_t slot = 0;
  std::optional<std::uint32_t> waits_release_of;
};
struct RingSchedule {
  std::vector<RingOp> ops;
  std::uint32_t slots = 0;
  bool clamped = false;
};

inline RingSchedule build_schedule(std::uint32_t num_layers, std::uint32_t ring_slots) {
  const std::uint64_t cap = 4ull * (num_layers ? num_layers : 1);
  std::vector<std::int64_t> ops(4 * cap);
  std::uint64_t n = 0;
  std::uint32_t slots = 0;
  int clamped = 0;
  detail::check(moesim_ring_build_schedule(num_layers, ring_slots, ops.data(), cap, &n, &slots,
                                           &clamped));
  RingSchedule s;
  s.slots = slots;
  s.clamped = clamped != 0;
  for (std::uint64_t i = 0; i < n; ++i) {
    RingOp op;
    op.kind = static_cast<RingOp::Kind>(ops[4 * i]);
    op.layer = static_cast<std::uint32_t>(ops[4 * i + 1]);
    op.slot = static_cast<std::uint32_t>(ops[4 * i + 2]);
    if (ops[4 * i + 3] >= 0) op.waits_release_of = static_cast<std::uint32_t>(ops[4 * i + 3]);
    s.ops.push_back(op);
  }
  return s;
}

// prefetch_cache.hpp:18-83: CachePolicyParams / AccessKind / AccessOutcome /
// SparseCache with the reference's member names; decisions come from
// moe_sparse_cache_* (identical to the reference's, tests/golden).
struct CachePolicyParams {
  std::size_t cpu_size = 0;
  double threshold = 1.0;
  double beta = 1.0;
  std::uint32_t decay_steps = 1;
};

enum class AccessKind : std::uint8_t {
  kCacheHit = 0,
  kFetchedFresh,
  kEvictedAndFetched,
  kStreamThrough,
};

struct AccessOutcome {
  AccessKind kind = AccessKind::kCacheHit;
  std::uint64_t victim = 0;
  friend bool operator==(const AccessOutcome&, const AccessOutcome&) = default;
};

class SparseCache {
 public:
  explicit SparseCache(CachePolicyParams params) : params_(params) {
    const moe_cache_params_t p{params.cpu_size, params.threshold, params.beta, params.decay_steps};
    detail::check(moe_sparse_cache_create(&p, &h_));
  }
  SparseCache(const SparseCache&) = delete;
  SparseCache& operator=(const SparseCache&) = delete;
  ~SparseCache() { moe_sparse_cache_destroy(h_); }

  AccessOutcome access(std::uint64_t block) {
    moe_cache_access_t o{};
    detail::check(moe_sparse_cache_access(h_, block, &o));
    return AccessOutcome{static_cast<AccessKind>(o.kind), o.victim};
  }
  void end_step() { detail::check(moe_sparse_cache_end_step(h_)); }

  const CachePolicyParams& params() const { return params_; }
  bool resident(std::uint64_t block) const { return hits_snapshot().count(block) != 0; }
  std::size_t acc_caches() const {
    std::uint64_t occ = 0;
    detail::check(moe_sparse_cache_state(h_, &occ, nullptr, nullptr, nullptr, 0, nullptr));
    return occ;
  }
  std::uint32_t steps() const {
    std::uint32_t st = 0;
    detail::check(moe_sparse_cache_state(h_, nullptr, &st, nullptr, nullptr, 0, nullptr));
    return st;
  }
  double hit_count(std::uint64_t block) const {
    const auto snap = hits_snapshot();
    const auto it = snap.find(block);
    return it == snap.end() ? 0.0 : it->second;
  }
  std::map<std::uint64_t, double> hits_snapshot() const {
    std::uint64_t n = 0;
    detail::check(moe_sparse_cache_state(h_, nullptr, nullptr, nullptr, nullptr, 0, &n));
    std::vector<std::uint64_t> b(n);
    std::vector<double> h(n);
    detail::check(moe_sparse_cache_state(h_, nullptr, nullptr, b.data(), h.data(), n, &n));
    std::map<std::uint64_t, double> out;
    for (std::uint64_t i = 0; i < n; ++i) out.emplace(b[i], h[i]);
    return out;
  }

 private:
  CachePolicyParams params_;
  moe_sparse_cache_t h_ = nullptr;
};

}  // namespace moesim
