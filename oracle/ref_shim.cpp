// ORACLE — TEST INFRASTRUCTURE ONLY.
// extern "C" wrappers over the reference library (moesim::core) compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/.  Used to
// pin oracle/moe_oracle.c and to generate tests/golden/ fixtures.  Never linked
// by the product.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "moesim/collectives.hpp"
#include "moesim/prefetch_cache.hpp"
#include "moesim/ring_offload.hpp"
#include "moesim/rng.hpp"
#include "moesim/sim_engine.hpp"
#include "moesim/topology.hpp"
#include "moesim/trace_export.hpp"
#include "moesim/workload.hpp"

using namespace moesim;

namespace {
int code_of(const std::exception_ptr& p) {
  try {
    std::rethrow_exception(p);
  } catch (const ConfigError&) {
    return 3;
  } catch (const std::out_of_range&) {
    return 2;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (...) {
    return 9;
  }
}
}  // namespace

extern "C" {

uint64_t ref_splitmix64_next(uint64_t* state) {
  SplitMix64 r(*state);
  const uint64_t v = r.next();
  *state += 0x9E3779B97F4A7C15ull;
  return v;
}

uint64_t ref_substream_seed(uint64_t seed, uint64_t step, uint64_t rank) {
  return substream_seed(seed, step, rank);
}

int ref_gen_trace(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                  uint64_t tokens, double skew, uint64_t* counts) {
  try {
    const RoutingTrace t = gen_trace(seed, steps, ranks, experts, tokens, skew);
    std::memcpy(counts, t.counts.data(), t.counts.size() * sizeof(uint64_t));
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_imbalance_ratio(uint32_t steps, uint32_t ranks, uint32_t experts, const uint64_t* counts,
                        double* out) {
  try {
    RoutingTrace t;
    t.steps = steps;
    t.ranks = ranks;
    t.experts = experts;
    t.counts.assign(counts, counts + static_cast<size_t>(steps) * ranks * experts);
    *out = imbalance_ratio(t);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_alltoall_flat(uint64_t ranks, uint64_t n_chunks, const uint64_t* lens, const uint8_t* data,
                      uint64_t* out_lens, uint8_t* out_data) {
  try {
    ShardedPayload p;
    p.ranks = ranks;
    p.chunks.resize(n_chunks);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      p.chunks[i].assign(data + off, data + off + lens[i]);
      off += lens[i];
    }
    const ShardedPayload out = alltoall_flat(p);
    uint64_t o = 0;
    for (uint64_t i = 0; i < out.chunks.size(); ++i) {
      out_lens[i] = out.chunks[i].size();
      std::memcpy(out_data + o, out.chunks[i].data(), out.chunks[i].size());
      o += out.chunks[i].size();
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// collectives.cpp:31-79 through a Topology with flat (positive) link params;
// stats: phase1_hops[6], phase2_hops[6], phase1_transfers, phase2_transfers
int ref_alltoall_hierarchical(uint32_t clusters, uint32_t nodes, uint32_t gpus, uint64_t ranks,
                              uint64_t n_chunks, const uint64_t* lens, const uint8_t* data,
                              uint64_t* out_lens, uint8_t* out_data, uint64_t* stats) {
  try {
    std::array<LinkParams, kLinkClassCount> links{};
    for (auto& l : links) {
      l.bandwidth_bytes_per_sec = 1000;
      l.latency_ns = 0;
    }
    const Topology topo(clusters, nodes, gpus, links);
    ShardedPayload p;
    p.ranks = ranks;
    p.chunks.resize(n_chunks);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      p.chunks[i].assign(data + off, data + off + lens[i]);
      off += lens[i];
    }
    AlltoAllStats st;
    const ShardedPayload out = alltoall_hierarchical(p, topo, &st);
    uint64_t o = 0;
    for (uint64_t i = 0; i < out.chunks.size(); ++i) {
      out_lens[i] = out.chunks[i].size();
      std::memcpy(out_data + o, out.chunks[i].data(), out.chunks[i].size());
      o += out.chunks[i].size();
    }
    for (int i = 0; i < 6; ++i) {
      stats[i] = st.phase1_hops[i];
      stats[6 + i] = st.phase2_hops[i];
    }
    stats[12] = st.phase1_transfers;
    stats[13] = st.phase2_transfers;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_fuse_slices(uint64_t n, const uint64_t* lens, const uint8_t* data, uint8_t* blob,
                    uint64_t* index) {
  try {
    std::vector<Chunk> slices(n);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; ++i) {
      slices[i].assign(data + off, data + off + lens[i]);
      off += lens[i];
    }
    const FusedBlob f = fuse_slices(slices);
    std::memcpy(blob, f.blob.data(), f.blob.size());
    for (uint64_t i = 0; i < f.index.size(); ++i) {
      index[3 * i] = f.index[i].slice_id;
      index[3 * i + 1] = f.index[i].offset;
      index[3 * i + 2] = f.index[i].length;
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_split_blob(uint64_t blob_len, const uint8_t* blob, uint64_t n, const uint64_t* index,
                   uint8_t* out) {
  try {
    Chunk b(blob, blob + blob_len);
    SliceIndex idx(n);
    for (uint64_t i = 0; i < n; ++i) idx[i] = SliceIndexEntry{index[3 * i], index[3 * i + 1], index[3 * i + 2]};
    const auto slices = split_blob(b, idx);
    uint64_t o = 0;
    for (const auto& s : slices) {
      std::memcpy(out + o, s.data(), s.size());
      o += s.size();
    }
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_ring_schedule(uint32_t layers, uint32_t ring_slots, int64_t* ops, uint64_t* n_ops,
                      uint32_t* slots_out, int* clamped) {
  try {
    RingPlan plan = RingPlan::uniform(layers, ring_slots, 1, 0, 1);
    const RingSchedule s = build_schedule(plan);
    for (size_t i = 0; i < s.ops.size(); ++i) {
      ops[4 * i] = static_cast<int64_t>(s.ops[i].kind);
      ops[4 * i + 1] = s.ops[i].layer;
      ops[4 * i + 2] = s.ops[i].slot;
      ops[4 * i + 3] = s.ops[i].waits_release_of ? static_cast<int64_t>(*s.ops[i].waits_release_of) : -1;
    }
    *n_ops = s.ops.size();
    *slots_out = s.slots;
    *clamped = s.clamped ? 1 : 0;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// simulate() with a one-GPU topology whose PCIe link is (bw, lat); every other
// link class is irrelevant to the ring timing except SSD warmup (not exported).
int ref_ring_simulate(uint32_t layers, uint32_t ring_slots, uint64_t expert_bytes,
                      uint64_t dense_bytes, const int64_t* compute_ns, uint64_t pcie_bw,
                      int64_t pcie_lat, int64_t* load_start, int64_t* load_end,
                      int64_t* comp_start, int64_t* comp_end, int64_t* makespan, int64_t* stall,
                      int64_t* copy_ns, uint64_t* peak_bytes, uint64_t* baseline_bytes) {
  try {
    RingPlan plan;
    plan.num_layers = layers;
    plan.ring_slots = ring_slots;
    plan.expert_bytes = expert_bytes;
    plan.dense_bytes = dense_bytes;
    plan.compute_ns.assign(compute_ns, compute_ns + layers);
    std::array<LinkParams, kLinkClassCount> links;
    links.fill(LinkParams{1000, 0});
    links[static_cast<size_t>(LinkClass::kPcie)] = LinkParams{pcie_bw, pcie_lat};
    const Topology topo(1, 1, 1, links);
    const RingSimResult r = simulate(plan, topo);
    for (const TaskRecord& t : r.timeline.tasks) {
      unsigned l = 0;
      if (t.label.rfind("load l", 0) == 0) {
        l = std::stoul(t.label.substr(6));
        load_start[l] = t.start;
        load_end[l] = t.end;
      } else if (t.label.rfind("compute l", 0) == 0) {
        l = std::stoul(t.label.substr(9));
        comp_start[l] = t.start;
        comp_end[l] = t.end;
      }
    }
    *makespan = r.makespan;
    *stall = r.stall_ns;
    *copy_ns = r.copy_ns_per_layer;
    *peak_bytes = r.peak_gpu_bytes;
    *baseline_bytes = r.baseline_gpu_bytes;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// workload.cpp:68-85 trace_to_json(...).dump() into out (cap bytes); *len = size.
int ref_trace_to_json(uint32_t steps, uint32_t ranks, uint32_t experts, uint64_t tokens,
                      const uint64_t* counts, char* out, uint64_t cap, uint64_t* len) {
  try {
    RoutingTrace t;
    t.steps = steps;
    t.ranks = ranks;
    t.experts = experts;
    t.tokens_per_rank = tokens;
    t.counts.assign(counts, counts + static_cast<size_t>(steps) * ranks * experts);
    const std::string s = trace_to_json(t).dump();
    *len = s.size();
    if (s.size() + 1 > cap) return 8;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// workload.cpp:87-119 trace_from_json(parse(text)); error text into err.
int ref_trace_from_json(const char* text, uint32_t* steps, uint32_t* ranks, uint32_t* experts,
                        uint64_t* tokens, uint64_t* counts, uint64_t counts_cap, char* err,
                        uint64_t err_cap) {
  try {
    const RoutingTrace t = trace_from_json(nlohmann::json::parse(text));
    *steps = t.steps;
    *ranks = t.ranks;
    *experts = t.experts;
    *tokens = t.tokens_per_rank;
    if (t.counts.size() > counts_cap) return 8;
    std::memcpy(counts, t.counts.data(), t.counts.size() * sizeof(uint64_t));
    return 0;
  } catch (const std::exception& e) {
    std::strncpy(err, e.what(), err_cap - 1);
    err[err_cap - 1] = 0;
    return code_of(std::current_exception());
  }
}

// prefetch_cache.cpp:28-64 SparseCache over an op list (ops[i] < 0: end_step,
// else access(ops[i])); outcome kinds / victims per op (-1 for end_step) and
// the final hits snapshot.
int ref_sparse_cache_run(uint64_t cpu_size, double threshold, double beta, uint32_t decay_steps,
                         const int64_t* ops, uint64_t n, int32_t* kinds, uint64_t* victims,
                         uint64_t* snap_blocks, double* snap_hits, uint64_t snap_cap,
                         uint64_t* snap_n, uint64_t* acc, uint32_t* steps) {
  try {
    SparseCache cache(CachePolicyParams{cpu_size, threshold, beta, decay_steps});
    for (uint64_t i = 0; i < n; ++i) {
      if (ops[i] < 0) {
        cache.end_step();
        kinds[i] = -1;
        victims[i] = 0;
        continue;
      }
      const AccessOutcome o = cache.access(static_cast<uint64_t>(ops[i]));
      kinds[i] = static_cast<int32_t>(o.kind);
      victims[i] = o.victim;
    }
    uint64_t k = 0;
    for (const auto& [b, h] : cache.hits_snapshot()) {
      if (k < snap_cap) {
        snap_blocks[k] = b;
        snap_hits[k] = h;
      }
      ++k;
    }
    *snap_n = k;
    *acc = cache.acc_caches();
    *steps = cache.steps();
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

// trace_export.cpp:28-50 timeline_to_trace_json(...).dump() of a Timeline
// built from n tasks (labels / streams as NUL-separated strings, start/end in
// ns); validate_trace_json of the parsed text into err ("" = valid).
int ref_timeline_trace_json(uint64_t n, const char* labels, const char* streams,
                            const int64_t* start, const int64_t* end, char* out, uint64_t cap,
                            uint64_t* len) {
  try {
    Timeline tl;
    const char* lp = labels;
    const char* sp = streams;
    for (uint64_t i = 0; i < n; ++i) {
      TaskRecord t;
      t.id = i;
      t.label = lp;
      t.stream = sp;
      lp += t.label.size() + 1;
      sp += t.stream.size() + 1;
      t.start = start[i];
      t.end = end[i];
      tl.streams[t.stream];
      tl.makespan = std::max<TimeNs>(tl.makespan, t.end);
      tl.tasks.push_back(std::move(t));
    }
    const std::string s = timeline_to_trace_json(tl).dump(2);
    *len = s.size();
    if (s.size() + 1 > cap) return 8;
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

int ref_validate_trace_json(const char* text, char* err, uint64_t err_cap) {
  try {
    const std::string e = validate_trace_json(nlohmann::json::parse(text));
    std::strncpy(err, e.c_str(), err_cap - 1);
    err[err_cap - 1] = 0;
    return 0;
  } catch (...) {
    return code_of(std::current_exception());
  }
}

}  // extern "C"
