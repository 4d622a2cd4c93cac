// extern "C" boundary (include/moe_b200.h): converts moe::Error / C++
// exceptions into moe_status_t + a thread-local "<field>: <reason>" message,
// mirroring the reference's exception taxonomy.
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "buckets.h"
#include "prefetch.h"
#include "sparse_cache.h"
#include "common.cuh"
#include "kernels.h"
#include "layer.h"
#include "ring.h"

namespace moe {
static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MOE_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace moe

namespace {

thread_local std::string g_last_error;

template <typename F>
moe_status_t guard(F&& f) {
  try {
    f();
    return MOE_OK;
  } catch (const moe::Error& e) {
    g_last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host: out of memory";
    return MOE_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MOE_ERR_LOGIC;
  }
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

// RAII device buffer for the host-buffer compatibility entry points.
struct DBuf {
  void* p = nullptr;
  explicit DBuf(uint64_t n) { MOE_CUDA(cudaMalloc(&p, n ? n : 16)); }
  ~DBuf() { cudaFree(p); }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct PrivStream {
  cudaStream_t s = nullptr;
  PrivStream() { MOE_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~PrivStream() { cudaStreamDestroy(s); }
};

}  // namespace

extern "C" {

const char* moe_last_error(void) { return g_last_error.c_str(); }
int moe_abi_version(void) { return MOE_ABI_VERSION; }
uint64_t moe_kernel_launch_count(void) { return moe::g_launches.load(); }

uint64_t moe_abi_sizeof(const char* n) {
  if (!n) return 0;
  const std::string s(n);
  if (s == "moe_slice_index_entry_t") return sizeof(moe_slice_index_entry_t);
  if (s == "moe_routing_out_t") return sizeof(moe_routing_out_t);
  if (s == "moe_gemm_problem_t") return sizeof(moe_gemm_problem_t);
  if (s == "moe_layer_desc_t") return sizeof(moe_layer_desc_t);
  if (s == "moe_layer_params_t") return sizeof(moe_layer_params_t);
  if (s == "moe_layer_grads_t") return sizeof(moe_layer_grads_t);
  if (s == "moe_ring_desc_t") return sizeof(moe_ring_desc_t);
  if (s == "moe_ring_timeline_t") return sizeof(moe_ring_timeline_t);
  if (s == "moe_cache_params_t") return sizeof(moe_cache_params_t);
  if (s == "moe_cache_access_t") return sizeof(moe_cache_access_t);
  if (s == "moe_prefetch_desc_t") return sizeof(moe_prefetch_desc_t);
  if (s == "moe_prefetch_record_t") return sizeof(moe_prefetch_record_t);
  if (s == "moe_prefetch_summary_t") return sizeof(moe_prefetch_summary_t);
  return 0;
}

// ------------------------------------------------------- moesim compat ----
namespace {
// topology.cpp route(): hop classes between two GPU ids (cluster, node, local)
struct GpuPos {
  uint32_t cluster, node, local;
};
void add_route(const GpuPos& a, const GpuPos& b, uint64_t* hops) {
  enum { NVL = 0, TOR = 3, LEAF = 4, SPIN = 5 };
  if (a.cluster == b.cluster && a.node == b.node) {
    if (a.local != b.local) hops[NVL] += 1;
    return;
  }
  hops[TOR] += 2;
  hops[LEAF] += a.local == b.local ? 1 : 2;
  if (a.local != b.local) hops[SPIN] += 1;
}
bool same_gpu(const GpuPos& a, const GpuPos& b) {
  return a.cluster == b.cluster && a.node == b.node && a.local == b.local;
}
}  // namespace

moe_status_t moesim_alltoall_hierarchical(uint32_t clusters, uint32_t nodes_per_cluster,
                                          uint32_t gpus_per_node, uint64_t ranks,
                                          uint64_t n_chunks, const uint64_t* lens,
                                          const uint8_t* data, uint64_t* out_lens,
                                          uint8_t* out_data, uint64_t* stats) {
  return guard([&] {
    moe::config_check(clusters >= 1, "topology.clusters: must be >= 1");
    moe::config_check(nodes_per_cluster >= 1, "topology.nodes_per_cluster: must be >= 1");
    moe::config_check(gpus_per_node >= 1, "topology.gpus_per_node: must be >= 1");
    moe::arg_check(n_chunks == ranks * ranks, "alltoall: payload is not a square rank matrix");
    moe::arg_check(ranks == (uint64_t)clusters * nodes_per_cluster * gpus_per_node,
                   "alltoall: payload rank count does not match topology GPU count");
    auto pos = [&](uint64_t r) {
      const uint64_t node_index = r / gpus_per_node;
      return GpuPos{(uint32_t)(node_index / nodes_per_cluster),
                    (uint32_t)(node_index % nodes_per_cluster), (uint32_t)(r % gpus_per_node)};
    };
    auto rank_of = [&](const GpuPos& g) {
      return ((uint64_t)g.cluster * nodes_per_cluster + g.node) * gpus_per_node + g.local;
    };
    std::vector<uint64_t> st(14, 0);
    // phase 1: chunk (src, dst) -> holder (src node, dst local rank), in
    // (src, dst) order; phase 2: holder -> dst, in per-holder arrival order
    std::vector<std::vector<uint64_t>> staged(ranks);
    for (uint64_t s = 0; s < ranks; ++s)
      for (uint64_t d = 0; d < ranks; ++d) {
        const GpuPos ps = pos(s), pd = pos(d);
        const GpuPos h{ps.cluster, ps.node, pd.local};
        if (!same_gpu(ps, h)) {
          add_route(ps, h, st.data());
          st[12] += 1;
        }
        staged[rank_of(h)].push_back(s * ranks + d);
      }
    std::vector<uint64_t> in_off(n_chunks), stage_off(n_chunks), out_off(n_chunks);
    uint64_t total = 0, mx = 0;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      in_off[i] = total;
      total += lens[i];
      mx = std::max(mx, lens[i]);
    }
    uint64_t o = 0;
    for (uint64_t h = 0; h < ranks; ++h)
      for (uint64_t c : staged[h]) {
        stage_off[c] = o;
        o += lens[c];
        const GpuPos ph = pos(h), pd = pos(c % ranks);
        if (!same_gpu(ph, pd)) {
          add_route(ph, pd, st.data() + 6);
          st[13] += 1;
        }
      }
    o = 0;
    for (uint64_t d = 0; d < ranks; ++d)
      for (uint64_t s = 0; s < ranks; ++s) {
        out_off[s * ranks + d] = o;  // chunk (s, d) lands at out (d, s)
        out_lens[d * ranks + s] = lens[s * ranks + d];
        o += lens[s * ranks + d];
      }
    if (stats) std::copy(st.begin(), st.end(), stats);
    if (!ranks || !total) return;
    PrivStream ps;
    DBuf dl(n_chunks * 8), di(n_chunks * 8), dso(n_chunks * 8), doo(n_chunks * 8), din(total),
        dstage(total), dout(total);
    MOE_CUDA(cudaMemcpyAsync(dl.p, lens, n_chunks * 8, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(di.p, in_off.data(), n_chunks * 8, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(dso.p, stage_off.data(), n_chunks * 8, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(doo.p, out_off.data(), n_chunks * 8, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(din.p, data, total, cudaMemcpyHostToDevice, ps.s));
    moe::copy_chunks_device(n_chunks, dl.as<uint64_t>(), di.as<uint64_t>(), din.as<uint8_t>(),
                            dso.as<uint64_t>(), dstage.as<uint8_t>(), mx, ps.s);  // phase 1
    moe::copy_chunks_device(n_chunks, dl.as<uint64_t>(), dso.as<uint64_t>(), dstage.as<uint8_t>(),
                            doo.as<uint64_t>(), dout.as<uint8_t>(), mx, ps.s);    // phase 2
    MOE_CUDA(cudaMemcpyAsync(out_data, dout.p, total, cudaMemcpyDeviceToHost, ps.s));
    MOE_CUDA(cudaStreamSynchronize(ps.s));
  });
}

moe_status_t moesim_alltoall_flat(uint64_t ranks, uint64_t n_chunks, const uint64_t* lens,
                                  const uint8_t* data, uint64_t* out_lens, uint8_t* out_data) {
  return guard([&] {
    moe::arg_check(n_chunks == ranks * ranks, "alltoall: payload is not a square rank matrix");
    if (ranks == 0) return;
    std::vector<uint64_t> in_off(n_chunks), out_off(n_chunks);
    uint64_t total = 0, mx = 0;
    for (uint64_t i = 0; i < n_chunks; ++i) {
      in_off[i] = total;
      total += lens[i];
      mx = std::max(mx, lens[i]);
    }
    uint64_t o = 0;
    for (uint64_t d = 0; d < ranks; ++d)
      for (uint64_t s = 0; s < ranks; ++s) {
        out_off[d * ranks + s] = o;
        out_lens[d * ranks + s] = lens[s * ranks + d];
        o += lens[s * ranks + d];
      }
    PrivStream ps;
    DBuf dl(n_chunks * 8), di(n_chunks * 8), dout_off(n_chunks * 8), din(total), dout(total);
    MOE_CUDA(cudaMemcpyAsync(dl.p, lens, n_chunks * 8, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(di.p, in_off.data(), n_chunks * 8, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(dout_off.p, out_off.data(), n_chunks * 8, cudaMemcpyHostToDevice, ps.s));
    if (total) MOE_CUDA(cudaMemcpyAsync(din.p, data, total, cudaMemcpyHostToDevice, ps.s));
    moe::alltoall_flat_device(ranks, dl.as<uint64_t>(), di.as<uint64_t>(), din.as<uint8_t>(),
                              dout_off.as<uint64_t>(), dout.as<uint8_t>(), mx, ps.s);
    if (total) MOE_CUDA(cudaMemcpyAsync(out_data, dout.p, total, cudaMemcpyDeviceToHost, ps.s));
    MOE_CUDA(cudaStreamSynchronize(ps.s));
  });
}

moe_status_t moesim_fuse_slices(uint64_t n, const uint64_t* lens, const uint8_t* data,
                                uint8_t* blob, moe_slice_index_entry_t* index) {
  return guard([&] {
    moe::arg_check(n != 0, "fuse_slices: empty slice list");
    uint64_t total = 0, mx = 0;
    std::vector<uint64_t> off(n);
    for (uint64_t i = 0; i < n; ++i) {
      off[i] = total;
      total += lens[i];
      mx = std::max(mx, lens[i]);
    }
    PrivStream ps;
    DBuf din(total), dblob(total), dlens(n * 8), didx(n * sizeof(moe_slice_index_entry_t)),
        dptr(n * sizeof(void*));
    std::vector<const uint8_t*> ptrs(n);
    for (uint64_t i = 0; i < n; ++i) ptrs[i] = din.as<uint8_t>() + off[i];
    if (total) MOE_CUDA(cudaMemcpyAsync(din.p, data, total, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(dlens.p, lens, n * 8, cudaMemcpyHostToDevice, ps.s));
    MOE_CUDA(cudaMemcpyAsync(dptr.p, ptrs.data(), n * sizeof(void*), cudaMemcpyHostToDevice, ps.s));
    moe::fuse_slices_device(n, dptr.as<const uint8_t*>(), dlens.as<uint64_t>(), dblob.as<uint8_t>(),
                            didx.as<moe_slice_index_entry_t>(), mx, ps.s);
    if (total) MOE_CUDA(cudaMemcpyAsync(blob, dblob.p, total, cudaMemcpyDeviceToHost, ps.s));
    MOE_CUDA(cudaMemcpyAsync(index, didx.p, n * sizeof(moe_slice_index_entry_t),
                             cudaMemcpyDeviceToHost, ps.s));
    MOE_CUDA(cudaStreamSynchronize(ps.s));
  });
}

moe_status_t moesim_split_blob(uint64_t blob_len, const uint8_t* blob, uint64_t n,
                               const moe_slice_index_entry_t* index, uint8_t* out) {
  return guard([&] {
    PrivStream ps;
    // output pointers: slices back to back (only dereferenced for a valid index,
    // whose lengths then sum to blob_len)
    std::vector<uint8_t*> ptrs(n);
    DBuf dout(blob_len), dblob(blob_len), didx(n * sizeof(moe_slice_index_entry_t) + 8),
        dptr(n * sizeof(void*) + 8), dbad(8);
    uint64_t o = 0, mx = 0;
    for (uint64_t i = 0; i < n; ++i) {
      ptrs[i] = dout.as<uint8_t>() + std::min(o, blob_len);
      o += index[i].length;
      mx = std::max(mx, index[i].length);
    }
    if (blob_len) MOE_CUDA(cudaMemcpyAsync(dblob.p, blob, blob_len, cudaMemcpyHostToDevice, ps.s));
    if (n) {
      MOE_CUDA(cudaMemcpyAsync(didx.p, index, n * sizeof(moe_slice_index_entry_t),
                               cudaMemcpyHostToDevice, ps.s));
      MOE_CUDA(cudaMemcpyAsync(dptr.p, ptrs.data(), n * sizeof(void*), cudaMemcpyHostToDevice, ps.s));
    }
    moe::split_blob_device(blob_len, dblob.as<uint8_t>(), n, didx.as<moe_slice_index_entry_t>(),
                           dptr.as<uint8_t*>(), dbad.as<int32_t>(), std::min(mx, blob_len), ps.s);
    int32_t bad = 0;
    MOE_CUDA(cudaMemcpyAsync(&bad, dbad.p, 4, cudaMemcpyDeviceToHost, ps.s));
    MOE_CUDA(cudaStreamSynchronize(ps.s));
    moe::arg_check(bad != 1, "split_blob: slice index is not contiguous");
    moe::arg_check(bad != 2, "split_blob: index does not cover the blob length");
    if (blob_len) MOE_CUDA(cudaMemcpy(out, dout.p, blob_len, cudaMemcpyDeviceToHost));
  });
}

moe_status_t moesim_gen_trace(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                              uint64_t tokens_per_rank, double skew, uint64_t* counts) {
  return guard([&] {
    moe::config_check(experts != 0, "workload.experts: must be >= 1");
    moe::config_check(!(skew < 0.0), "workload.skew: must be >= 0");
    const uint64_t n = (uint64_t)steps * ranks * experts;
    PrivStream ps;
    DBuf dc(n * 8);
    moe::gen_trace_device(seed, steps, ranks, experts, tokens_per_rank, skew, dc.as<uint64_t>(),
                          ps.s);
    if (n) MOE_CUDA(cudaMemcpyAsync(counts, dc.p, n * 8, cudaMemcpyDeviceToHost, ps.s));
    MOE_CUDA(cudaStreamSynchronize(ps.s));
  });
}

moe_status_t moesim_imbalance_ratio(uint32_t steps, uint32_t ranks, uint32_t experts,
                                    const uint64_t* counts, double* out) {
  return guard([&] {
    moe::config_check(experts != 0, "imbalance_ratio: trace carries zero tokens");
    const uint64_t rows = (uint64_t)steps * ranks;
    PrivStream ps;
    DBuf dc(rows * experts * 8), dr(16);
    if (rows) MOE_CUDA(cudaMemcpyAsync(dc.p, counts, rows * experts * 8, cudaMemcpyHostToDevice, ps.s));
    moe::imbalance_device(rows, experts, dc.as<uint64_t>(), dr.as<unsigned long long>(), ps.s);
    unsigned long long r[2];
    MOE_CUDA(cudaMemcpyAsync(r, dr.p, 16, cudaMemcpyDeviceToHost, ps.s));
    MOE_CUDA(cudaStreamSynchronize(ps.s));
    moe::config_check(r[1] != 0, "imbalance_ratio: trace carries zero tokens");
    const double mean = (double)r[1] / (double)experts;
    *out = (double)r[0] / mean;
  });
}

moe_status_t moesim_ring_build_schedule(uint32_t layers, uint32_t ring_slots, int64_t* ops,
                                        uint64_t capacity, uint64_t* n_ops, uint32_t* slots,
                                        int* clamped) {
  return guard([&] {
    bool cl = false;
    const auto sched = moe::ring_schedule(layers, ring_slots, slots, &cl);
    moe::arg_check(capacity >= sched.size(), "ring.ops: capacity too small");
    for (size_t i = 0; i < sched.size(); ++i) {
      ops[4 * i] = sched[i].kind;
      ops[4 * i + 1] = sched[i].layer;
      ops[4 * i + 2] = sched[i].slot;
      ops[4 * i + 3] = sched[i].waits;
    }
    *n_ops = sched.size();
    *clamped = cl ? 1 : 0;
  });
}

// ------------------------------------------------------------ device ops --
moe_status_t moe_fill_uniform(void* out, uint64_t n, moe_dtype_t dtype, uint64_t seed, double lo,
                              double hi, void* stream) {
  return guard([&] { moe::fill_uniform(out, n, dtype, seed, lo, hi, S(stream)); });
}

moe_status_t moe_gen_trace_device(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                                  uint64_t tokens_per_rank, double skew, uint64_t* counts,
                                  void* stream) {
  return guard([&] {
    moe::gen_trace_device(seed, steps, ranks, experts, tokens_per_rank, skew, counts, S(stream));
  });
}

moe_status_t moe_alltoall_flat_device(uint64_t ranks, const uint64_t* lens, const uint64_t* in_off,
                                      const uint8_t* in, const uint64_t* out_off, uint8_t* out,
                                      void* stream) {
  return guard([&] {
    // max chunk length unknown on the host: split each chunk 64 ways
    moe::alltoall_flat_device(ranks, lens, in_off, in, out_off, out, 64ull << 20, S(stream));
  });
}

moe_status_t moe_fuse_slices_device(uint64_t n, const uint8_t* const* slices, const uint64_t* lens,
                                    uint8_t* blob, moe_slice_index_entry_t* index, void* stream) {
  return guard([&] {
    moe::arg_check(n != 0, "fuse_slices: empty slice list");
    moe::fuse_slices_device(n, slices, lens, blob, index, 64ull << 20, S(stream));
  });
}

moe_status_t moe_split_blob_device(uint64_t blob_len, const uint8_t* blob, uint64_t n,
                                   const moe_slice_index_entry_t* index, uint8_t* const* out,
                                   int32_t* bad, void* stream) {
  return guard([&] {
    moe::split_blob_device(blob_len, blob, n, index, out, bad, 64ull << 20, S(stream));
  });
}

moe_status_t moe_route(uint64_t tokens, uint32_t experts, uint32_t top_k, uint64_t capacity,
                       const float* logits, const moe_routing_out_t* out, void* stream) {
  return guard([&] {
    moe::arg_check(out != nullptr && out->expert && out->gate && out->position && out->keep &&
                       out->count1 && out->count2 && out->kept && out->aux_loss,
                   "route.out: every output pointer is required");
    moe::RouteWorkspace ws;
    ws.nchunks = moe::route_chunks(tokens);
    std::vector<void*> tmp;
    auto al = [&](uint64_t bytes) {
      void* p = nullptr;
      MOE_CUDA(cudaMallocAsync(&p, bytes ? bytes : 16, S(stream)));
      tmp.push_back(p);
      return p;
    };
    ws.chunk_cnt = (int32_t*)al(2 * ws.nchunks * experts * 4);
    ws.chunk_off = (int32_t*)al(2 * ws.nchunks * experts * 4);
    ws.psum_part = (float*)al((ws.nchunks + 1) * experts * 4);
    ws.rank_local = (int32_t*)al(tokens * top_k * 4);
    moe::route_forward(tokens, experts, top_k, capacity, logits, *out, ws, S(stream));
    for (void* p : tmp) MOE_CUDA(cudaFreeAsync(p, S(stream)));
  });
}

moe_status_t moe_grouped_gemm(const moe_gemm_problem_t* problem, void* stream) {
  return guard([&] {
    moe::arg_check(problem != nullptr, "gemm.problem: must be non-null");
    moe::grouped_gemm(*problem, S(stream));
  });
}

moe_status_t moe_split_f32_bf16x3(const float* in, uint64_t n, void* out, void* stream) {
  return guard([&] {
    moe::arg_check(n == 0 || (in != nullptr && out != nullptr), "split.in/out: must be non-null");
    moe::split_f32_bf16x3(in, n, out, S(stream));
  });
}

// ------------------------------------------------------------- layer -----
moe_status_t moe_layer_create(const moe_layer_desc_t* desc, moe_layer_t* out) {
  return guard([&] {
    moe::arg_check(desc != nullptr && out != nullptr, "layer.desc: must be non-null");
    *out = reinterpret_cast<moe_layer_t>(new moe::Layer(*desc));
  });
}

moe_status_t moe_layer_destroy(moe_layer_t layer) {
  return guard([&] { delete reinterpret_cast<moe::Layer*>(layer); });
}

uint64_t moe_layer_capacity(moe_layer_t layer) {
  return layer ? reinterpret_cast<moe::Layer*>(layer)->C : 0;
}

moe_status_t moe_layer_forward(moe_layer_t layer, const moe_layer_params_t* params, const void* x,
                               void* y, const float* logits_override, float* logits_out,
                               const moe_routing_out_t* routing, void* stream) {
  return guard([&] {
    moe::arg_check(layer != nullptr && params != nullptr, "forward: layer/params must be non-null");
    reinterpret_cast<moe::Layer*>(layer)->forward(*params, x, y, logits_override, logits_out,
                                                  routing, S(stream));
  });
}

moe_status_t moe_layer_backward(moe_layer_t layer, const moe_layer_params_t* params, const void* dy,
                                float d_aux, void* dx, const moe_layer_grads_t* grads,
                                void* stream) {
  return guard([&] {
    moe::arg_check(layer != nullptr && params != nullptr && grads != nullptr,
                   "backward: layer/params/grads must be non-null");
    reinterpret_cast<moe::Layer*>(layer)->backward(*params, dy, d_aux, dx, *grads, S(stream));
  });
}

moe_status_t moe_layer_train_step_host(moe_layer_t layer, const moe_layer_params_t* params,
                                       const void* x_host, const void* dy_host, float d_aux,
                                       void* y_host, void* dx_host, const moe_layer_grads_t* grads,
                                       void* stream) {
  return guard([&] {
    moe::arg_check(layer != nullptr && params != nullptr && grads != nullptr,
                   "train_step: layer/params/grads must be non-null");
    reinterpret_cast<moe::Layer*>(layer)->train_step_host(*params, x_host, dy_host, d_aux, y_host,
                                                          dx_host, *grads, S(stream));
  });
}

moe_status_t moe_layer_train_step_host_async(moe_layer_t layer, const moe_layer_params_t* params,
                                             const void* x_host, const void* dy_host, float d_aux,
                                             void* y_host, void* dx_host,
                                             const moe_layer_grads_t* grads, void* stream) {
  return guard([&] {
    moe::arg_check(layer != nullptr && params != nullptr && grads != nullptr,
                   "train_step: layer/params/grads must be non-null");
    reinterpret_cast<moe::Layer*>(layer)->train_step_host(*params, x_host, dy_host, d_aux, y_host,
                                                          dx_host, *grads, S(stream), true);
  });
}

moe_status_t moe_layer_host_sync(moe_layer_t layer, void* stream) {
  return guard([&] {
    moe::arg_check(layer != nullptr, "host_sync: layer must be non-null");
    reinterpret_cast<moe::Layer*>(layer)->host_sync(S(stream));
  });
}

moe_status_t moe_layer_set_profiling(moe_layer_t layer, int enabled) {
  return guard([&] {
    moe::arg_check(layer != nullptr, "profiling: layer must be non-null");
    reinterpret_cast<moe::Layer*>(layer)->profiling = enabled != 0;
  });
}

moe_status_t moe_layer_set_peer_timeout(moe_layer_t layer, double seconds) {
  return guard([&] {
    moe::arg_check(layer != nullptr, "peer_timeout: layer must be non-null");
    moe::config_check(seconds >= 0.0, "layer.peer_timeout: must be >= 0 (0 = wait forever)");
    reinterpret_cast<moe::Layer*>(layer)->win.timeout_ns = (uint64_t)(seconds * 1e9);
  });
}

moe_status_t moe_layer_comm_status(moe_layer_t layer, int32_t* code) {
  return guard([&] {
    moe::arg_check(layer != nullptr && code != nullptr, "comm_status: null argument");
    auto* L = reinterpret_cast<moe::Layer*>(layer);
    *code = L->p2p ? moe::p2p_status(L->win) : 0;
    if (*code != 0)
      moe::fail(MOE_ERR_NCCL, "layer.exchange: peer " + std::to_string((*code - 1000) % 16) +
                                  " did not signal slot " + std::to_string((*code - 1000) / 16) +
                                  " within the peer timeout");
  });
}

static void phase_times_of(moe::Layer* L, int which, const char** names, float* ms,
                           uint32_t capacity, uint32_t* count) {
  uint32_t n = 0;
  const auto& lg = L->plog[which];
  if (L->profiling && lg.n > 0) {
    MOE_CUDA(cudaEventSynchronize(lg.ev[lg.n]));
    for (int i = 0; i < lg.n && n < capacity; ++i, ++n) {
      if (names) names[n] = lg.name[i];
      if (ms) MOE_CUDA(cudaEventElapsedTime(&ms[n], lg.ev[i], lg.ev[i + 1]));
    }
  }
  *count = n;
}

moe_status_t moe_layer_phase_times(moe_layer_t layer, const char** names, float* ms,
                                   uint32_t capacity, uint32_t* count) {
  return guard([&] {
    moe::arg_check(layer != nullptr && count != nullptr, "phase_times: null argument");
    auto* L = reinterpret_cast<moe::Layer*>(layer);
    phase_times_of(L, L->last_log, names, ms, capacity, count);
  });
}

moe_status_t moe_layer_phase_times_of(moe_layer_t layer, int backward, const char** names,
                                      float* ms, uint32_t capacity, uint32_t* count) {
  return guard([&] {
    moe::arg_check(layer != nullptr && count != nullptr, "phase_times: null argument");
    phase_times_of(reinterpret_cast<moe::Layer*>(layer), backward ? 1 : 0, names, ms, capacity,
                   count);
  });
}

// -------------------------------------------------------------- comm -----
moe_status_t moe_comm_unique_id(uint8_t id[128]) {
  return guard([&] { moe::comm_unique_id(id); });
}
moe_status_t moe_comm_create(const uint8_t id[128], uint32_t nranks, uint32_t rank, void** comm) {
  return guard([&] {
    moe::arg_check(comm != nullptr && id != nullptr, "comm: null argument");
    moe::config_check(rank < nranks, "comm.rank: must be < nranks");
    *comm = moe::comm_create(id, nranks, rank);
  });
}
moe_status_t moe_comm_destroy(void* comm) {
  return guard([&] { moe::comm_destroy(comm); });
}
moe_status_t moe_alltoall_packed(void* comm, const void* send, void* recv, uint64_t bytes_per_peer,
                                 uint32_t slices_per_peer, int fused, void* stream) {
  return guard([&] {
    moe::arg_check(comm != nullptr, "alltoall.comm: must be non-null");
    moe::alltoall_packed(comm, send, recv, bytes_per_peer, slices_per_peer, fused, S(stream));
  });
}

// ----------------------------------------------------------- buckets -----
moe_status_t moe_grad_buckets_create(void* comm, uint32_t n, const uint64_t* ids_layer_order,
                                     void* const* grads, const uint64_t* numel,
                                     uint32_t capacity, float scale, moe_grad_buckets_t* out) {
  return guard([&] {
    moe::arg_check(out != nullptr, "bucket: out must be non-null");
    *out = reinterpret_cast<moe_grad_buckets_t>(
        new moe::GradBuckets(comm, n, ids_layer_order, grads, numel, capacity, scale));
  });
}

moe_status_t moe_grad_buckets_destroy(moe_grad_buckets_t b) {
  return guard([&] { delete reinterpret_cast<moe::GradBuckets*>(b); });
}

moe_status_t moe_grad_buckets_push(moe_grad_buckets_t b, uint64_t id, void* stream,
                                   int32_t* flushed) {
  return guard([&] {
    moe::arg_check(b != nullptr && flushed != nullptr, "bucket: null argument");
    *flushed = reinterpret_cast<moe::GradBuckets*>(b)->push(id, S(stream));
  });
}

moe_status_t moe_grad_buckets_reset(moe_grad_buckets_t b) {
  return guard([&] {
    moe::arg_check(b != nullptr, "bucket: null argument");
    reinterpret_cast<moe::GradBuckets*>(b)->reset();
  });
}

uint32_t moe_grad_buckets_count(moe_grad_buckets_t b) {
  return b ? reinterpret_cast<moe::GradBuckets*>(b)->count() : 0;
}

moe_status_t moe_grad_buckets_ids(moe_grad_buckets_t b, uint32_t i, uint64_t* ids,
                                  uint32_t capacity, uint32_t* n) {
  return guard([&] {
    auto* g = reinterpret_cast<moe::GradBuckets*>(b);
    moe::arg_check(g != nullptr && n != nullptr, "bucket: null argument");
    if (i >= g->count()) moe::fail(MOE_ERR_OUT_OF_RANGE, "bucket: index out of range");
    const auto& v = g->ids(i);
    *n = (uint32_t)v.size();
    for (uint32_t q = 0; q < v.size() && q < capacity; ++q) ids[q] = v[q];
  });
}

// ------------------------------------------------------- sparse cache -----
moe_status_t moe_sparse_cache_create(const moe_cache_params_t* params, moe_sparse_cache_t* out) {
  return guard([&] {
    moe::arg_check(params != nullptr && out != nullptr, "cache: null argument");
    *out = reinterpret_cast<moe_sparse_cache_t>(new moe::SparseCache(*params));
  });
}

moe_status_t moe_sparse_cache_destroy(moe_sparse_cache_t cache) {
  return guard([&] { delete reinterpret_cast<moe::SparseCache*>(cache); });
}

moe_status_t moe_sparse_cache_access(moe_sparse_cache_t cache, uint64_t block,
                                     moe_cache_access_t* out) {
  return guard([&] {
    moe::arg_check(cache != nullptr && out != nullptr, "cache: null argument");
    *out = reinterpret_cast<moe::SparseCache*>(cache)->access(block);
  });
}

moe_status_t moe_sparse_cache_end_step(moe_sparse_cache_t cache) {
  return guard([&] {
    moe::arg_check(cache != nullptr, "cache: null argument");
    reinterpret_cast<moe::SparseCache*>(cache)->end_step();
  });
}

moe_status_t moe_sparse_cache_state(moe_sparse_cache_t cache, uint64_t* occupancy, uint32_t* steps,
                                    uint64_t* blocks, double* hits, uint64_t capacity,
                                    uint64_t* resident) {
  return guard([&] {
    auto* c = reinterpret_cast<moe::SparseCache*>(cache);
    moe::arg_check(c != nullptr, "cache: null argument");
    if (occupancy) *occupancy = c->occupancy();
    if (steps) *steps = c->steps();
    uint64_t n = 0;
    for (const auto& [b, h] : c->counts()) {
      if (n < capacity) {
        if (blocks) blocks[n] = b;
        if (hits) hits[n] = h;
      }
      ++n;
    }
    if (resident) *resident = n;
  });
}

// ---------------------------------------------------------- prefetch -----
moe_status_t moe_prefetch_create(moe_layer_t layer, const moe_prefetch_desc_t* desc,
                                 moe_prefetch_t* out) {
  return guard([&] {
    moe::arg_check(layer != nullptr && desc != nullptr && out != nullptr, "prefetch: null argument");
    *out = reinterpret_cast<moe_prefetch_t>(
        new moe::Prefetch2D(reinterpret_cast<moe::Layer*>(layer), *desc));
  });
}

moe_status_t moe_prefetch_destroy(moe_prefetch_t p) {
  return guard([&] { delete reinterpret_cast<moe::Prefetch2D*>(p); });
}

moe_status_t moe_prefetch_run(moe_prefetch_t p, uint32_t steps, const void* x, void* y,
                              moe_prefetch_record_t* records, moe_prefetch_summary_t* summary,
                              void* stream) {
  return guard([&] {
    moe::arg_check(p != nullptr && x != nullptr && y != nullptr, "prefetch: null argument");
    reinterpret_cast<moe::Prefetch2D*>(p)->run(steps, x, y, records, summary, S(stream));
  });
}

// -------------------------------------------------------------- ring -----
moe_status_t moe_ring_create(moe_layer_t layer, const moe_ring_desc_t* desc, moe_ring_t* out) {
  return guard([&] {
    moe::arg_check(layer != nullptr && desc != nullptr && out != nullptr, "ring: null argument");
    *out = reinterpret_cast<moe_ring_t>(
        new moe::Ring(reinterpret_cast<moe::Layer*>(layer), *desc));
  });
}
moe_status_t moe_ring_destroy(moe_ring_t ring) {
  return guard([&] { delete reinterpret_cast<moe::Ring*>(ring); });
}
uint64_t moe_ring_section_bytes(moe_layer_t layer) {
  if (!layer) return 0;
  return moe::section_layout(*reinterpret_cast<moe::Layer*>(layer)).bytes;
}
moe_status_t moe_ring_pack_section(moe_layer_t layer, const void* w1, const float* b1,
                                   const void* w2, const float* b2, void* host_section) {
  return guard([&] {
    moe::arg_check(layer && w1 && b1 && w2 && b2 && host_section, "ring.pack: null argument");
    auto* L = reinterpret_cast<moe::Layer*>(layer);
    const moe::SectionLayout s = moe::section_layout(*L);
    uint8_t* h = static_cast<uint8_t*>(host_section);
    MOE_CUDA(cudaMemcpy(h + s.w1, w1, (uint64_t)L->El * L->dff * L->dm * L->esz, cudaMemcpyDeviceToHost));
    MOE_CUDA(cudaMemcpy(h + s.b1, b1, (uint64_t)L->El * L->dff * 4, cudaMemcpyDeviceToHost));
    MOE_CUDA(cudaMemcpy(h + s.w2, w2, (uint64_t)L->El * L->dm * L->dff * L->esz, cudaMemcpyDeviceToHost));
    MOE_CUDA(cudaMemcpy(h + s.b2, b2, (uint64_t)L->El * L->dm * 4, cudaMemcpyDeviceToHost));
  });
}
moe_status_t moe_ring_run(moe_ring_t ring, const void* x, void* y, moe_ring_timeline_t* timeline,
                          void* stream) {
  return guard([&] {
    moe::arg_check(ring != nullptr && x != nullptr && y != nullptr, "ring.run: null argument");
    reinterpret_cast<moe::Ring*>(ring)->run(x, y, timeline, S(stream));
  });
}

}  // extern "C"
