// C++ host program over the drop-in API (include/moesim_b200.hpp) and the
// C-ABI (include/moe_b200.h).  Re-expresses, against libmoe_b200.so, the
// assertions the reference's own suites make for the functions on the path
// (test_collectives.cpp:35-171, test_workload.cpp:59-139,
// test_ring_offload.cpp:29-68, acceptance_main.cpp criteria 3-4), then drives
// one MoE layer forward+backward from C++ through the C-ABI.  Prints one
// PASS/FAIL line per criterion; exit status 1 if any failed.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "moe_b200.h"
#include "moesim_b200.hpp"

using namespace moesim;

namespace {

struct Fail : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void check(bool c, const std::string& what) {
  if (!c) throw Fail(what);
}
template <typename E, typename F>
void expect_throw(F&& f, const std::string& what) {
  try {
    f();
  } catch (const E&) {
    return;
  }
  throw Fail("expected exception: " + what);
}

// SplitMix64 written from the rng.hpp description (independent of the library)
struct Sm {
  std::uint64_t s;
  std::uint64_t operator()() {
    s += 0x9E3779B97F4A7C15ull;
    std::uint64_t z = s;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
};

ShardedPayload random_payload(std::size_t ranks, std::uint64_t seed, std::size_t max_len = 16) {
  Sm rng{seed};
  ShardedPayload p = ShardedPayload::make(ranks);
  for (auto& c : p.chunks) {
    c.resize(rng() % (max_len + 1));
    for (auto& b : c) b = static_cast<std::uint8_t>(rng());
  }
  return p;
}

void alltoall_cases() {
  ShardedPayload one = ShardedPayload::make(1);
  one.at(0, 0) = {1, 2, 3};
  check(alltoall_flat(one) == one, "R=1 identity");
  ShardedPayload p = ShardedPayload::make(2);
  p.at(0, 0) = {'a'};
  p.at(0, 1) = {'b'};
  p.at(1, 0) = {'c'};
  p.at(1, 1) = {'d'};
  const ShardedPayload o = alltoall_flat(p);
  check(o.at(0, 1) == Chunk{'c'} && o.at(1, 0) == Chunk{'b'}, "R=2 transpose");
  const ShardedPayload r = random_payload(4, 99);
  const ShardedPayload ro = alltoall_flat(r);
  for (std::size_t i = 0; i < 4; ++i)
    for (std::size_t j = 0; j < 4; ++j) check(ro.at(i, j) == r.at(j, i), "R=4 direct transpose");
  ShardedPayload bad;
  bad.ranks = 2;
  bad.chunks.resize(3);
  expect_throw<std::invalid_argument>([&] { alltoall_flat(bad); }, "non-square payload");
  // acceptance criterion 3 shape sweep (flat part): random payloads, 1..16 ranks
  Sm rng{0xC0113C7};
  for (int cs = 0; cs < 200; ++cs) {
    const std::size_t R = 1 + rng() % 16;
    ShardedPayload q = ShardedPayload::make(R);
    for (auto& c : q.chunks) {
      c.resize(rng() % 9);
      for (auto& b : c) b = static_cast<std::uint8_t>(rng());
    }
    const ShardedPayload qo = alltoall_flat(q);
    for (std::size_t i = 0; i < R; ++i)
      for (std::size_t j = 0; j < R; ++j) check(qo.at(i, j) == q.at(j, i), "sweep transpose");
  }
}

// test_collectives.cpp:69-110 through the drop-in Topology / AlltoAllStats
void hierarchical_cases() {
  {
    const Topology topo(1, 1, 4);
    const ShardedPayload p = random_payload(4, 5);
    AlltoAllStats st;
    check(alltoall_hierarchical(p, topo, &st) == alltoall_flat(p), "one node = flat");
    check(st.phase2_transfers == 0, "one node: no phase 2");
  }
  {
    const Topology topo(1, 2, 2);
    ShardedPayload p = ShardedPayload::make(4);
    for (std::uint8_t s = 0; s < 4; ++s)
      for (std::uint8_t d = 0; d < 4; ++d) p.at(s, d) = {s, d};
    AlltoAllStats st;
    check(alltoall_hierarchical(p, topo, &st) == alltoall_flat(p), "2x2 tagged");
    check(st.hops(LinkClass::kSpin) == 0, "2x2 no spin");
  }
  std::uint64_t seed = 1;
  for (std::uint32_t c = 1; c <= 2; ++c)
    for (std::uint32_t n = 1; n <= 2; ++n)
      for (std::uint32_t g = 1; g <= 4; ++g) {
        const Topology topo(c, n, g);
        for (int rep = 0; rep < 5; ++rep) {
          const ShardedPayload p = random_payload(topo.total_gpus(), seed++);
          AlltoAllStats st;
          check(alltoall_hierarchical(p, topo, &st) == alltoall_flat(p), "random topology");
          check(st.phase2_hops[5] == 0 && st.phase1_hops[3] == 0 && st.phase1_hops[5] == 0,
                "rails only");
        }
      }
  const Topology topo(1, 2, 2);
  expect_throw<std::invalid_argument>([&] { alltoall_hierarchical(random_payload(3, 1), topo); },
                                      "rank mismatch");
  expect_throw<ConfigError>([&] { Topology(0, 1, 1); }, "zero clusters");
  check(topo.route(topo.gpu(0), topo.gpu(3)).size() == 5, "cross-rail route via spin");
}

void fusion_cases() {
  const std::vector<Chunk> one = {{1, 2, 3}};
  const FusedBlob f = fuse_slices(one);
  check(f.blob == one[0] && f.index.size() == 1 && f.index[0] == SliceIndexEntry{0, 0, 3},
        "single slice");
  check(split_blob(f.blob, f.index) == one, "single round trip");
  const std::vector<Chunk> z = {{1, 2, 3}, {}, {4, 5, 6, 7, 8}};
  const FusedBlob fz = fuse_slices(z);
  check(fz.blob.size() == 8 && split_blob(fz.blob, fz.index) == z, "zero-length slices");
  Sm rng{0xF05105};
  for (int rep = 0; rep < 200; ++rep) {
    std::vector<Chunk> s(1 + rng() % 16);
    for (auto& c : s) {
      c.resize(rng() % 32);
      for (auto& b : c) b = static_cast<std::uint8_t>(rng());
    }
    check(split_blob(fuse_slices(s).blob, fuse_slices(s).index) == s, "random round trip");
  }
  expect_throw<std::invalid_argument>([] { fuse_slices({}); }, "empty slice list");
  const FusedBlob two = fuse_slices({{1, 2}});
  Chunk longer = two.blob;
  longer.push_back(0);
  expect_throw<std::invalid_argument>([&] { split_blob(longer, two.index); }, "longer blob");
  SliceIndex gap = two.index;
  gap[0].offset = 1;
  expect_throw<std::invalid_argument>([&] { split_blob(two.blob, gap); }, "gap");
}

std::vector<Count> sampler(std::uint64_t seed, std::uint32_t steps, std::uint32_t ranks,
                           std::uint32_t experts, Count tokens, double skew) {
  std::vector<double> cdf(experts);
  double acc = 0;
  for (std::uint32_t e = 0; e < experts; ++e) cdf[e] = (acc += std::pow(e + 1.0, -skew));
  for (auto& c : cdf) c /= acc;
  cdf[experts - 1] = 1.0;
  std::vector<Count> out(static_cast<std::size_t>(steps) * ranks * experts, 0);
  for (std::uint32_t s = 0; s < steps; ++s)
    for (std::uint32_t r = 0; r < ranks; ++r) {
      Sm rng{seed ^ (0x9E3779B97F4A7C15ull * (s + 1ull)) ^ (0xC2B2AE3D27D4EB4Full * (r + 1ull))};
      for (Count t = 0; t < tokens; ++t) {
        const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        std::uint32_t e = 0;
        while (e + 1 < experts && u >= cdf[e]) ++e;
        out[(static_cast<std::size_t>(s) * ranks + r) * experts + e] += 1;
      }
    }
  return out;
}

void workload_cases() {
  const RoutingTrace one = gen_trace(7, 2, 3, 1, 50, 1.5);
  for (Count c : one.counts) check(c == 50, "single expert takes every token");
  const RoutingTrace zero = gen_trace(7, 2, 2, 4, 0, 0.0);
  for (Count c : zero.counts) check(c == 0, "zero tokens");
  check(gen_trace(7, 1, 2, 4, 100, 0.0).counts == sampler(7, 1, 2, 4, 100, 0.0), "sampler seed 7");
  check(gen_trace(11, 3, 2, 8, 64, 1.2).counts == sampler(11, 3, 2, 8, 64, 1.2), "sampler seed 11");
  check(gen_trace(42, 4, 4, 16, 256, 0.9).counts == gen_trace(42, 4, 4, 16, 256, 0.9).counts,
        "determinism");
  check(gen_trace(42, 4, 4, 16, 256, 0.9).counts != gen_trace(43, 4, 4, 16, 256, 0.9).counts,
        "seed sensitivity");
  const RoutingTrace c = gen_trace(5, 3, 5, 7, 129, 2.0);
  for (std::uint32_t s = 0; s < 3; ++s)
    for (std::uint32_t r = 0; r < 5; ++r) {
      Count sum = 0;
      for (std::uint32_t e = 0; e < 7; ++e) sum += c.at(s, r, e);
      check(sum == 129, "conservation");
    }
  expect_throw<ConfigError>([] { gen_trace(1, 1, 1, 0, 10, 0.0); }, "experts = 0");
  RoutingTrace t;
  t.steps = t.ranks = 1;
  t.experts = 2;
  t.counts = {90, 10};
  check(std::fabs(imbalance_ratio(t) - 1.8) < 1e-12, "imbalance 1.8");
  t.counts = {50, 50};
  check(imbalance_ratio(t) == 1.0, "imbalance 1.0");
  t.counts = {0, 0};
  expect_throw<ConfigError>([&] { imbalance_ratio(t); }, "zero-token imbalance");
  check(imbalance_ratio(gen_trace(3, 2, 4, 8, 512, 2.0)) >
            imbalance_ratio(gen_trace(3, 2, 4, 8, 512, 0.0)),
        "skew raises imbalance");
}

void ring_cases() {
  const RingSchedule s1 = build_schedule(1, 1);
  check(s1.ops.size() == 3 && s1.ops[0].kind == RingOp::Kind::kLoad &&
            s1.ops[1].kind == RingOp::Kind::kCompute && s1.ops[2].kind == RingOp::Kind::kRelease,
        "N=1 K=1 shape");
  for (const RingOp& op : build_schedule(3, 1).ops)
    if (op.kind == RingOp::Kind::kLoad && op.layer > 0)
      check(op.waits_release_of && *op.waits_release_of == op.layer - 1, "N=3 K=1 chain");
  int loads = 0;
  for (const RingOp& op : build_schedule(4, 2).ops)
    if (op.kind == RingOp::Kind::kLoad) {
      ++loads;
      check(op.slot == op.layer % 2, "slot arithmetic");
      if (op.layer >= 2) check(*op.waits_release_of == op.layer - 2, "waits release(i-K)");
    }
  check(loads == 4, "N=4 K=2 loads");
  expect_throw<ConfigError>([] { build_schedule(4, 0); }, "K = 0");
  const RingSchedule cl = build_schedule(3, 10);
  check(cl.clamped && cl.slots == 3, "K > N clamps");
}

// One MoE layer forward+backward from C++ through the C-ABI.
void layer_case() {
  const uint32_t E = 8, k = 2, d = 256, f = 512;
  const uint64_t T = 1000;
  moe_layer_desc_t desc{E, k, d, f, 1.25, T, MOE_DTYPE_BF16, 0, 1, 0, nullptr};
  moe_layer_t L = nullptr;
  moe_status_t st = moe_layer_create(&desc, &L);
  check(st == MOE_OK, std::string("create: ") + moe_last_error());
  void *x, *y, *dy, *dx, *wg, *w1, *w2;
  float *b1, *b2, *g[6];
  cudaMalloc(&x, T * d * 2);
  cudaMalloc(&y, T * d * 2);
  cudaMalloc(&dy, T * d * 2);
  cudaMalloc(&dx, T * d * 2);
  cudaMalloc(&wg, E * d * 2);
  cudaMalloc(&w1, E * f * d * 2);
  cudaMalloc(&w2, E * d * f * 2);
  cudaMalloc(&b1, E * f * 4);
  cudaMalloc(&b2, E * d * 4);
  const uint64_t gsz[6] = {E * d, E, E * f * d, E * f, E * d * f, E * d};
  for (int i = 0; i < 6; ++i) cudaMalloc(&g[i], gsz[i] * 4);
  const double bd = 1.0 / std::sqrt(double(d)), bf = 1.0 / std::sqrt(double(f));
  check(moe_fill_uniform(x, T * d, MOE_DTYPE_BF16, 1, -1, 1, nullptr) == MOE_OK, "fill");
  moe_fill_uniform(dy, T * d, MOE_DTYPE_BF16, 2, -1, 1, nullptr);
  moe_fill_uniform(wg, E * d, MOE_DTYPE_BF16, 3, -bd, bd, nullptr);
  moe_fill_uniform(w1, E * f * d, MOE_DTYPE_BF16, 4, -bd, bd, nullptr);
  moe_fill_uniform(w2, E * d * f, MOE_DTYPE_BF16, 5, -bf, bf, nullptr);
  moe_fill_uniform(b1, E * f, MOE_DTYPE_F32, 6, -bd, bd, nullptr);
  moe_fill_uniform(b2, E * d, MOE_DTYPE_F32, 7, -bf, bf, nullptr);
  moe_layer_params_t p{wg, nullptr, w1, b1, w2, b2};
  moe_layer_grads_t gr{g[0], g[1], g[2], g[3], g[4], g[5]};
  int32_t *cnt1, *cnt2, *kept;
  cudaMalloc(&cnt1, E * 4);
  cudaMalloc(&cnt2, E * 4);
  cudaMalloc(&kept, E * 4);
  int32_t *ex, *pos;
  float *gate, *aux;
  uint8_t* keep;
  cudaMalloc(&ex, T * k * 4);
  cudaMalloc(&pos, T * k * 4);
  cudaMalloc(&gate, T * k * 4);
  cudaMalloc(&keep, T * k);
  cudaMalloc(&aux, 4);
  moe_routing_out_t ro{ex, gate, pos, keep, cnt1, cnt2, kept, aux};
  st = moe_layer_forward(L, &p, x, y, nullptr, nullptr, &ro, nullptr);
  check(st == MOE_OK, std::string("forward: ") + moe_last_error());
  st = moe_layer_backward(L, &p, dy, 0.01f, dx, &gr, nullptr);
  check(st == MOE_OK, std::string("backward: ") + moe_last_error());
  check(cudaDeviceSynchronize() == cudaSuccess, "sync");
  std::vector<int32_t> c1(E), c2(E), kp(E);
  cudaMemcpy(c1.data(), cnt1, E * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(c2.data(), cnt2, E * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(kp.data(), kept, E * 4, cudaMemcpyDeviceToHost);
  const uint64_t C = moe_layer_capacity(L);
  int64_t s1 = 0, s2 = 0;
  for (uint32_t e = 0; e < E; ++e) {
    s1 += c1[e];
    s2 += c2[e];
    check(kp[e] == std::min<int64_t>(c1[e] + c2[e], C), "kept = min(count1+count2, C)");
  }
  check(s1 == (int64_t)T && s2 == (int64_t)T, "every token routed twice (top-2)");
  std::vector<uint16_t> hy(T * d), hdx(T * d);
  cudaMemcpy(hy.data(), y, T * d * 2, cudaMemcpyDeviceToHost);
  cudaMemcpy(hdx.data(), dx, T * d * 2, cudaMemcpyDeviceToHost);
  for (uint16_t v : hy) check((v & 0x7f80) != 0x7f80, "finite y");
  for (uint16_t v : hdx) check((v & 0x7f80) != 0x7f80, "finite dx");
  check(moe_layer_destroy(L) == MOE_OK, "destroy");
}

// test_prefetch_cache.cpp:77-158 assertions against the drop-in SparseCache
void sparse_cache_cases() {
  using moesim::AccessKind;
  using moesim::CachePolicyParams;
  using moesim::SparseCache;
  {
    SparseCache cache(CachePolicyParams{4, 1.0, 1.0, 1});
    check(cache.access(100).kind == AccessKind::kFetchedFresh, "fresh admission");
    check(cache.hit_count(100) == 1.0 && cache.acc_caches() == 1, "fresh count");
    check(cache.access(100).kind == AccessKind::kCacheHit && cache.hit_count(100) == 2.0, "hit");
  }
  {
    SparseCache cache(CachePolicyParams{3, 1.0, 1.0, 1});
    for (int b : {1, 1, 1, 2}) cache.access(b);
    const auto out = cache.access(3);
    check(out.kind == AccessKind::kEvictedAndFetched && out.victim == 2, "evict coldest");
    check(!cache.resident(2) && cache.resident(3) && cache.hit_count(3) == 1.0, "readmit");
  }
  {
    SparseCache cache(CachePolicyParams{3, 5.0, 1.0, 1});
    for (int b : {1, 1, 1, 2}) cache.access(b);
    check(cache.access(3).kind == AccessKind::kStreamThrough && cache.hit_count(1) == 3.0,
          "no warm-enough victim streams through");
  }
  for (std::size_t size : {0u, 1u}) {
    SparseCache cache(CachePolicyParams{size, 1.0, 1.0, 1});
    for (int i = 0; i < 10; ++i)
      check(cache.access(i % 3).kind == AccessKind::kStreamThrough, "cpu_size 0/1 never caches");
    check(cache.acc_caches() == 0, "no occupancy");
  }
  {
    SparseCache cache(CachePolicyParams{4, 1.0, 0.5, 2});
    for (int i = 0; i < 4; ++i) cache.access(7);
    cache.end_step();
    check(cache.hit_count(7) == 4.0, "no decay before K");
    cache.end_step();
    check(cache.hit_count(7) == 2.0 && cache.steps() == 0, "decay after K steps");
  }
  bool threw = false;
  try {
    SparseCache bad(CachePolicyParams{4, 1.0, 0.0, 1});
  } catch (const moesim::ConfigError& e) {
    threw = std::string(e.what()) == "cache.beta: must be in (0, 1]";
  }
  check(threw, "beta 0 -> ConfigError");
}

}  // namespace

int main() {
  const std::vector<std::pair<std::string, std::function<void()>>> crit = {
      {"alltoall_flat = chunk transpose (collectives.cpp:10-21)", alltoall_cases},
      {"alltoall_hierarchical = flat, rails only (collectives.cpp:31-79)", hierarchical_cases},
      {"fuse_slices/split_blob exact inverses + errors (collectives.cpp:88-118)", fusion_cases},
      {"gen_trace = independent sampler, conservation, imbalance (workload.cpp:19-66)",
       workload_cases},
      {"build_schedule shapes, chains, clamping (ring_offload.cpp:31-50)", ring_cases},
      {"SparseCache branches, eviction, decay, errors (prefetch_cache.cpp:28-64)",
       sparse_cache_cases},
      {"MoE layer fwd+bwd from C++ through the C-ABI", layer_case},
  };
  int failed = 0;
  for (const auto& [name, fn] : crit) {
    try {
      fn();
      std::printf("PASS %s\n", name.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAIL %s: %s\n", name.c_str(), e.what());
    }
  }
  std::printf(failed ? "%d criteria failed\n" : "all criteria passed\n", failed);
  return failed ? 1 : 0;
}
