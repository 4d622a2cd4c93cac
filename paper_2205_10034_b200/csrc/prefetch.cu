// 2D prefetch with the Algorithm-1 CPU cache, executed (
// PAPER.md:215-320; the reference simulates it in run_2d_schedule,
// prefetch_cache.cpp:97-204).
//
// Three tiers for the sparse (expert) parameters of a stack of MoE layers:
//   backing store  a file holding every layer's section ("SSD"),
//   CPU cache      pinned host blocks managed by SparseCache (Algorithm 1),
//   GPU slots      lookahead + 1 HBM sections the layers compute from.
// For every (step, layer) in order the host consults the cache and does the
// backing-store I/O its outcome implies (hit: none; fresh: read into a new
// block; evict: write the victim back, read into its block; stream-through:
// read into a pinned staging buffer, cache untouched), then the H2D of the
// section is queued on a copy stream behind compute(t - lookahead)'s start —
// "prefetch for layer t + lookahead issued when compute(t) starts"
// (prefetch_cache.cpp:121-125) — and compute(t) (layer forward + residual)
// waits for it.  Every decay cycle the cache decays; every flush_period steps
// the resident blocks are written back (prefetch_cache.cpp:176-183).  The
// host runs ahead of the GPU, so backing-store I/O overlaps earlier layers'
// compute; pinned blocks are only rewritten after the H2D that read them
// completes.  CUDA events give the timeline and the reference's metrics
// (makespan, per-layer stall = gap between consecutive computes).
#include <fcntl.h>
#include <unistd.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "layer.h"
#include "prefetch.h"
#include "ring.h"

namespace moe {

namespace {
double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}
}  // namespace

Prefetch2D::Prefetch2D(Layer* layer, const moe_prefetch_desc_t& d)
    : L(layer), cache(d.cache) {
  config_check(d.num_layers >= 1, "prefetch.num_layers: must be >= 1");
  config_check(d.lookahead >= 1, "cache.lookahead: must be >= 1");
  arg_check(d.host_sections != nullptr && d.gate_weights != nullptr && d.backing_path != nullptr,
            "prefetch.host_sections/gate_weights/backing_path: must be non-null");
  N = d.num_layers;
  lookahead = d.lookahead;
  flush_period = d.flush_period ? d.flush_period : d.cache.decay_steps;
  lay = section_layout(*L);
  wg.assign(d.gate_weights, d.gate_weights + N);
  path = d.backing_path;
  fd = ::open(path.c_str(), O_RDWR | O_CREAT | O_TRUNC, 0600);
  require(fd >= 0, MOE_ERR_INVALID_ARGUMENT, "prefetch.backing_path: cannot open " + path);
  for (uint32_t i = 0; i < N; ++i) write_block(i, d.host_sections[i]);
  ::fsync(fd);
  K = lookahead + 1;
  gslots.resize(K);
  for (uint32_t s = 0; s < K; ++s) MOE_CUDA(cudaMalloc(&gslots[s], lay.bytes));
  for (int s = 0; s < 2; ++s) MOE_CUDA(cudaMallocHost(&stage[s], lay.bytes));
  const uint64_t act = L->T * L->dm * L->esz;
  MOE_CUDA(cudaMalloc(&hbuf[0], act));
  MOE_CUDA(cudaMalloc(&hbuf[1], act));
  MOE_CUDA(cudaMalloc(&tmp, act));
  MOE_CUDA(cudaStreamCreateWithFlags(&copy, cudaStreamNonBlocking));
  MOE_CUDA(cudaEventCreate(&ev_start));
}

Prefetch2D::~Prefetch2D() {
  if (copy) cudaStreamSynchronize(copy);
  for (void* p : gslots) cudaFree(p);
  for (auto& [b, blk] : blocks) cudaFreeHost(blk.ptr);
  for (void* p : stage) cudaFreeHost(p);
  cudaFree(hbuf[0]);
  cudaFree(hbuf[1]);
  cudaFree(tmp);
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  cudaEventDestroy(ev_start);
  if (copy) cudaStreamDestroy(copy);
  if (fd >= 0) {
    ::close(fd);
    ::unlink(path.c_str());
  }
}

void Prefetch2D::read_block(uint32_t b, void* dst) {
  uint64_t done = 0;
  while (done < lay.bytes) {
    const ssize_t r = ::pread(fd, static_cast<uint8_t*>(dst) + done, lay.bytes - done,
                              (off_t)((uint64_t)b * lay.bytes + done));
    require(r > 0, MOE_ERR_CUDA, "prefetch: backing-store read failed");
    done += (uint64_t)r;
  }
  bytes_read += lay.bytes;
}

void Prefetch2D::write_block(uint32_t b, const void* src) {
  uint64_t done = 0;
  while (done < lay.bytes) {
    const ssize_t r = ::pwrite(fd, static_cast<const uint8_t*>(src) + done, lay.bytes - done,
                               (off_t)((uint64_t)b * lay.bytes + done));
    require(r > 0, MOE_ERR_CUDA, "prefetch: backing-store write failed");
    done += (uint64_t)r;
  }
}

cudaEvent_t Prefetch2D::event() {
  cudaEvent_t e;
  MOE_CUDA(cudaEventCreate(&e));
  evs.push_back(e);
  return e;
}

void Prefetch2D::run(uint32_t steps, const void* x, void* y, moe_prefetch_record_t* recs,
                     moe_prefetch_summary_t* sum, cudaStream_t st) {
  const uint64_t n = L->T * L->dm;
  const uint64_t act = n * L->esz;
  const uint64_t total = (uint64_t)steps * N;
  // the previous run ended synchronised: forget its events before destroying them
  for (auto& [b, blk] : blocks) blk.last = nullptr;
  stage_last[0] = stage_last[1] = nullptr;
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  evs.clear();
  std::vector<cudaEvent_t> h0(total), h1(total), c0(total), c1(total);
  std::vector<double> io(total, 0.0);
  std::vector<moe_cache_access_t> outcome(total);
  for (uint64_t t = 0; t < total; ++t) {
    h0[t] = event();
    h1[t] = event();
    c0[t] = event();
    c1[t] = event();
  }
  bytes_read = bytes_written = 0;
  MOE_CUDA(cudaEventRecord(ev_start, st));
  MOE_CUDA(cudaStreamWaitEvent(copy, ev_start, 0));
  MOE_CUDA(cudaMemcpyAsync(hbuf[0], x, act, cudaMemcpyDeviceToDevice, st));
  int cur = 0;
  // a pinned buffer may be rewritten only after the H2D that last read it
  auto drain = [&](cudaEvent_t& last) {
    if (last) MOE_CUDA(cudaEventSynchronize(last));
    last = nullptr;
  };
  for (uint64_t t = 0; t < total; ++t) {
    const uint32_t step = (uint32_t)(t / N), layer = (uint32_t)(t % N);
    // ---- sparse dimension: CPU cache, backing-store I/O (host) ----
    const double t0 = now_ms();
    const moe_cache_access_t o = cache.access(layer);
    outcome[t] = o;
    const void* src = nullptr;
    cudaEvent_t* src_last = nullptr;
    if (o.kind == MOE_CACHE_HIT) {
      Block& blk = blocks.at(layer);
      src = blk.ptr;
      src_last = &blk.last;
    } else if (o.kind == MOE_CACHE_FETCHED_FRESH) {
      Block blk;
      MOE_CUDA(cudaMallocHost(&blk.ptr, lay.bytes));
      read_block(layer, blk.ptr);
      auto it = blocks.emplace(layer, blk).first;
      src = it->second.ptr;
      src_last = &it->second.last;
    } else if (o.kind == MOE_CACHE_EVICTED_AND_FETCHED) {
      auto vit = blocks.find((uint32_t)o.victim);
      require(vit != blocks.end(), MOE_ERR_LOGIC, "prefetch: evicted block not resident");
      Block blk = vit->second;
      blocks.erase(vit);
      drain(blk.last);
      write_block((uint32_t)o.victim, blk.ptr);  // write back, then refetch into the block
      bytes_written += lay.bytes;
      read_block(layer, blk.ptr);
      auto it = blocks.emplace(layer, blk).first;
      src = it->second.ptr;
      src_last = &it->second.last;
    } else {  // stream-through: staging buffer, cache untouched
      const int sidx = (int)(stream_count++ & 1);
      drain(stage_last[sidx]);
      read_block(layer, stage[sidx]);
      src = stage[sidx];
      src_last = &stage_last[sidx];
    }
    io[t] = now_ms() - t0;
    // ---- H2D into GPU slot t % K, issued when compute(t - lookahead) starts ----
    if (t >= lookahead) MOE_CUDA(cudaStreamWaitEvent(copy, c0[t - lookahead], 0));
    MOE_CUDA(cudaEventRecord(h0[t], copy));
    MOE_CUDA(cudaMemcpyAsync(gslots[t % K], src, lay.bytes, cudaMemcpyHostToDevice, copy));
    MOE_CUDA(cudaEventRecord(h1[t], copy));
    *src_last = h1[t];
    // ---- compute(t): layer forward on the slot + residual ----
    MOE_CUDA(cudaStreamWaitEvent(st, h1[t], 0));
    MOE_CUDA(cudaEventRecord(c0[t], st));
    const uint8_t* s = static_cast<const uint8_t*>(gslots[t % K]);
    moe_layer_params_t w;
    w.wg = wg[layer];
    w.bg = nullptr;
    w.w1 = s + lay.w1;
    w.b1 = reinterpret_cast<const float*>(s + lay.b1);
    w.w2 = s + lay.w2;
    w.b2 = reinterpret_cast<const float*>(s + lay.b2);
    L->forward(w, hbuf[cur], tmp, nullptr, nullptr, nullptr, st);
    residual_add(L->dt, hbuf[cur], tmp, hbuf[cur ^ 1], n, st);
    cur ^= 1;
    MOE_CUDA(cudaEventRecord(c1[t], st));
    if (layer + 1 == N) {
      cache.end_step();
      if ((step + 1) % flush_period == 0) {  // CPU -> backing-store flush of resident blocks
        const double f0 = now_ms();
        for (auto& [b, blk] : blocks) {
          write_block(b, blk.ptr);
          bytes_written += lay.bytes;
        }
        io[t] += now_ms() - f0;
      }
    }
  }
  MOE_CUDA(cudaMemcpyAsync(y, hbuf[cur], act, cudaMemcpyDeviceToDevice, st));
  MOE_CUDA(cudaStreamSynchronize(st));
  MOE_CUDA(cudaStreamSynchronize(copy));
  float mk = 0.f, comp = 0.f, stall = 0.f, prev_end = 0.f;
  double io_total = 0.0;
  for (uint64_t t = 0; t < total; ++t) {
    float a, b, c, e;
    MOE_CUDA(cudaEventElapsedTime(&a, ev_start, h0[t]));
    MOE_CUDA(cudaEventElapsedTime(&b, ev_start, h1[t]));
    MOE_CUDA(cudaEventElapsedTime(&c, ev_start, c0[t]));
    MOE_CUDA(cudaEventElapsedTime(&e, ev_start, c1[t]));
    if (recs) {
      moe_prefetch_record_t& r = recs[t];
      r.step = (uint32_t)(t / N);
      r.layer = (uint32_t)(t % N);
      r.kind = outcome[t].kind;
      r.victim = outcome[t].victim;
      r.io_ms = (float)io[t];
      r.h2d_start = a;
      r.h2d_end = b;
      r.compute_start = c;
      r.compute_end = e;
    }
    stall += std::max(0.f, c - prev_end);
    prev_end = e;
    comp += e - c;
    mk = std::max(mk, e);
    io_total += io[t];
  }
  if (sum) {
    sum->makespan_ms = mk;
    sum->compute_total_ms = comp;
    sum->stall_total_ms = stall;
    sum->io_total_ms = (float)io_total;
    sum->bytes_read = bytes_read;
    sum->bytes_written = bytes_written;
    sum->h2d_bytes = total * lay.bytes;
    sum->gpu_slots = K;
    sum->section_bytes = lay.bytes;
  }
}

}  // namespace moe
