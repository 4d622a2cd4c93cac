// The MoE layer: gate GEMM (K1) -> routing (K2) -> dispatch into the
// Fusion-packed send buffer (K3) -> EP all-to-all over NCCL (K4) -> grouped
// expert FFN on tcgen05 (K5) -> all-to-all back (K4) -> weighted combine (K6),
// and the backward of all of it (4 all-to-alls per layer).
//
// Layout in HBM:
//   send/home buffers  [E][Cs][d]       expert-major; experts of rank r are the
//                                       contiguous block r*El..r*El+El-1, so the
//                                       message to rank r is ONE contiguous
//                                       region (Fusion packing, collectives.cpp:
//                                       88-98: SliceIndex = (j, j*Cs*d, kept*d))
//   recv buffers       [P][El][Cs][d]   per (source rank, local expert) slice,
//                                       receive order = source rank order
//                                       (alltoall_flat, collectives.cpp:10-21)
//   expert activations [P*El*Cs][d_ff]  same row space as recv
// Cs = C rounded up to 64 rows; rows [kept, round_up(kept,64)) are zero so the
// weight-gradient GEMM can run whole 64-row K blocks.  No host synchronisation:
// every count lives on the device and the GEMM tile schedulers read it there.
#include <nccl.h>

#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.h"
#include "ep_p2p.h"
#include "layer.h"
#include "nccl_check.h"

namespace moe {


namespace {

template <typename T>
T* dalloc(std::vector<void*>& owned, uint64_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  MOE_CUDA(cudaMalloc(&p, n * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}
void* dalloc_bytes(std::vector<void*>& owned, uint64_t n) {
  void* p = nullptr;
  MOE_CUDA(cudaMalloc(&p, n ? n : 16));
  owned.push_back(p);
  return p;
}

}  // namespace

Layer::Layer(const moe_layer_desc_t& d) : desc(d) {
  E = d.num_experts;
  k = d.top_k;
  dm = d.d_model;
  dff = d.d_ff;
  T = d.tokens;
  P = d.ep_size ? d.ep_size : 1;
  rank = d.ep_rank;
  dt = d.dtype;
  config_check(E >= 1, "layer.num_experts: must be >= 1");
  config_check(E <= 256, "layer.num_experts: must be <= 256");
  config_check(k == 1 || k == 2, "layer.top_k: must be 1 or 2");
  config_check(k == 1 || E >= 2, "layer.top_k: top-2 needs >= 2 experts");
  config_check(d.capacity_factor > 0.0, "layer.capacity_factor: must be > 0");
  config_check(dt == MOE_DTYPE_BF16 || dt == MOE_DTYPE_F32, "layer.dtype: must be bf16 or fp32");
  config_check(E % P == 0, "layer.ep_size: must divide num_experts");
  config_check(rank < P, "layer.ep_rank: must be < ep_size");
  config_check(P == 1 || d.nccl_comm != nullptr, "layer.nccl_comm: required when ep_size > 1");
  config_check(d.gate_grad_reduce <= 1, "layer.gate_grad_reduce: must be 0 (layer) or 1 (caller)");
  config_check(d.placement == MOE_PLACEMENT_CONTIGUOUS || d.placement == MOE_PLACEMENT_ROUND_ROBIN,
               "layer.placement: must be MOE_PLACEMENT_CONTIGUOUS or MOE_PLACEMENT_ROUND_ROBIN");
  if (dt == MOE_DTYPE_BF16) {
    config_check(dm % 128 == 0, "layer.d_model: bf16 path needs a multiple of 128");
    config_check(dff % 128 == 0, "layer.d_ff: bf16 path needs a multiple of 128");
  } else {
    config_check(dm % 8 == 0, "layer.d_model: must be a multiple of 8");
    config_check(dff % 8 == 0, "layer.d_ff: must be a multiple of 8");
  }
  El = E / P;
  esz = dt == MOE_DTYPE_BF16 ? 2 : 4;
  comm = d.nccl_comm;
  const double c = (double)k * d.capacity_factor * (double)T / (double)E;
  C = (uint64_t)std::ceil(c);
  // fp32 layers run their expert GEMMs as split-bf16 tcgen05 GEMMs (widths the
  // tcgen05 tiles take); MOE_F32_GEMM=simt keeps the FFMA path
  {
    const char* env = std::getenv("MOE_F32_GEMM");
    split32 = dt == MOE_DTYPE_F32 && dm % 128 == 0 && dff % 128 == 0 &&
              !(env && std::string(env) == "simt");
  }
  pad = (dt == MOE_DTYPE_BF16 || split32) ? 64 : 1;
  if (split32) {  // one launch holds every K chunk: groups x chunks <= 1024 tile groups
    auto nchunks = [](uint64_t K) {
      uint64_t n = 1;
      while (K / n > 512 || (K / 64) % n) ++n;
      return n;
    };
    const uint64_t cs = (P > 1 && d.exchange == MOE_EXCHANGE_P2P ? P : 1) *
                        round_up((uint64_t)std::ceil((double)k * d.capacity_factor * (double)T /
                                                     (double)E), 64);
    const uint64_t nmax =
        std::max({nchunks(dm), nchunks(dff), ceil_div(std::max<uint64_t>(cs, 1), (uint64_t)512)});
    split32 = nmax <= 64 && (uint64_t)E * nmax <= 1024;
  }
  Cs = round_up(C ? C : 1, pad);
  rows = (uint64_t)P * El * Cs;
  Epad = (uint32_t)round_up(E, 64);
  config_check(rows < (1ull << 31), "layer.tokens: slot rows exceed int32 indexing");

  MOE_CUDA(cudaGetDevice(&device));
  // routing state
  logits = dalloc<float>(owned, T * E);
  expert = dalloc<int32_t>(owned, T * k);
  position = dalloc<int32_t>(owned, T * k);
  slot = dalloc<int32_t>(owned, T * k);
  gate = dalloc<float>(owned, T * k);
  keep = dalloc<uint8_t>(owned, T * k);
  count1 = dalloc<int32_t>(owned, E);
  count2 = dalloc<int32_t>(owned, E);
  kept = dalloc<int32_t>(owned, E);
  aux = dalloc<float>(owned, 1);
  rr = d.placement == MOE_PLACEMENT_ROUND_ROBIN && P > 1;
  if (rr) {
    pexpert = dalloc<int32_t>(owned, T * k);
    pkept = dalloc<int32_t>(owned, E);
  }
  rws.nchunks = route_chunks(T);
  rws.chunk_cnt = dalloc<int32_t>(owned, 2 * rws.nchunks * E);
  rws.chunk_off = dalloc<int32_t>(owned, 2 * rws.nchunks * E);
  rws.psum_part = dalloc<float>(owned, (rws.nchunks + 1) * E);
  rws.rank_local = dalloc<int32_t>(owned, T * k);
  // token buffers
  const uint64_t slot_bytes = (uint64_t)E * Cs * dm * esz;
  p2p = P > 1 && d.exchange == MOE_EXCHANGE_P2P;
  config_check(d.exchange == MOE_EXCHANGE_P2P || d.exchange == MOE_EXCHANGE_NCCL,
               "layer.exchange: must be MOE_EXCHANGE_P2P or MOE_EXCHANGE_NCCL");
  if (p2p) {
    // receive / home buffers live in one IPC window that every peer maps
    p2p_setup(win, comm, P, rank, E, Cs, (uint64_t)dm * esz, (uint64_t)E * dm + E, 0);
    xr = win.base + win.off_xr;
    dYr = win.base + win.off_dyr;
    Yh = win.base + win.off_yh;
    dXh = win.base + win.off_dxh;
  }
  // P2P receive regions hold one contiguous group per local expert
  ngroups = p2p ? El : P * El;
  if (!p2p) {
    xs = dalloc_bytes(owned, slot_bytes);
    xr = P > 1 ? dalloc_bytes(owned, slot_bytes) : xs;
    cnt_recv = P > 1 ? dalloc<int32_t>(owned, E) : kept;
  }
  {
    const uint64_t mr = p2p ? (uint64_t)P * Cs : Cs;
    cs_part = dalloc<float>(owned, colsum_ws_floats(ngroups, dm, mr));
    const uint64_t nt = colsum_ticket_ints(ngroups, dm);
    cs_ticket = dalloc<int32_t>(owned, nt);
    MOE_CUDA(cudaMemset(cs_ticket, 0, nt * sizeof(int32_t)));
    // fixed-order reduction workspaces (deterministic gradients, reduce.cu)
    db1_ws = dalloc<float>(owned, gemm_colsum_ws_floats(ngroups, dff, mr));
    if (d.has_gate_bias) dbg_ws = dalloc<float>(owned, std::max<uint64_t>(1, route_dbg_ws_floats(T, E)));
  }
  gm = dalloc<int32_t>(owned, E);
  ga = dalloc<int32_t>(owned, E);
  gb = dalloc<int32_t>(owned, E);
  gmk = dalloc<int32_t>(owned, E);
  gak = dalloc<int32_t>(owned, E);
  gbk = dalloc<int32_t>(owned, E);
  // rows per expert group: the P2P receive region holds every source's rows
  gstride = p2p ? (uint64_t)P * Cs : Cs;
  if (split32) {
    const uint64_t kc = 512;  // K chunk: bounds the truncating tensor-core accumulation
    xr3 = dalloc_bytes(owned, 3 * rows * dm * 2);
    dy3 = dalloc_bytes(owned, 3 * rows * dm * 2);
    a3 = dalloc_bytes(owned, 3 * rows * dff * 2);
    dh3 = dalloc_bytes(owned, 3 * rows * dff * 2);
    w1_3 = dalloc_bytes(owned, 3 * (uint64_t)El * dff * dm * 2);
    w2_3 = dalloc_bytes(owned, 3 * (uint64_t)El * dff * dm * 2);
    const uint64_t np_m = std::max(ceil_div((uint64_t)dm, kc) * dff, ceil_div((uint64_t)dff, kc) * dm);
    s_part = dalloc<float>(owned, std::max(np_m * rows, ceil_div(gstride, kc) * El * dff * dm));
    s_cs = dalloc<float>(owned, colsum_ws_floats(ngroups, dff, gstride));
    const uint64_t nt = (uint64_t)E * 64;  // groups x K chunks (chunks <= 64)
    for (auto& t : s_tab) {
      t.m = dalloc<int32_t>(owned, nt);
      t.a = dalloc<int32_t>(owned, nt);
      t.c = dalloc<int32_t>(owned, nt);
      t.b = dalloc<int32_t>(owned, nt);
      t.k = dalloc<int32_t>(owned, nt);
    }
  }
  Gp = dalloc_bytes(owned, rows * dff * esz);
  Aact = dalloc_bytes(owned, rows * dff * esz);
  Yl = dalloc_bytes(owned, slot_bytes);
  if (!p2p) Yh = P > 1 ? dalloc_bytes(owned, slot_bytes) : Yl;
  // backward
  dgate = dalloc<float>(owned, T * k);
  if (!p2p) {
    dYs = dalloc_bytes(owned, slot_bytes);
    dYr = P > 1 ? dalloc_bytes(owned, slot_bytes) : dYs;
  }
  dH = dalloc_bytes(owned, rows * dff * esz);
  dXl = dalloc_bytes(owned, slot_bytes);
  if (!p2p) dXh = P > 1 ? dalloc_bytes(owned, slot_bytes) : dXl;
  if (dt == MOE_DTYPE_BF16) dl_lp = dalloc_bytes(owned, T * Epad * 2);
  else dl_f32 = dalloc<float>(owned, T * E);
  // Every row of the activation buffers holds finite values from here on, so
  // zero pad rows of the partner operand annihilate them in the RAGGED_K GEMMs
  // (the P2P window is zeroed by p2p_setup).
  if (xs) MOE_CUDA(cudaMemset(xs, 0, slot_bytes));
  if (!p2p && xr != xs) MOE_CUDA(cudaMemset(xr, 0, slot_bytes));
  MOE_CUDA(cudaMemset(Gp, 0, rows * dff * esz));
  MOE_CUDA(cudaMemset(Aact, 0, rows * dff * esz));
  MOE_CUDA(cudaMemset(dH, 0, rows * dff * esz));
  if (dYs) MOE_CUDA(cudaMemset(dYs, 0, slot_bytes));
  if (!p2p && dYr != dYs) MOE_CUDA(cudaMemset(dYr, 0, slot_bytes));
  // gate GEMM tables: one group of T rows; split-K groups for dwg
  {
    std::vector<int32_t> one = {(int32_t)T, 0, 0, 0};
    gate_tab = dalloc<int32_t>(owned, 4);
    MOE_CUDA(cudaMemcpy(gate_tab, one.data(), 16, cudaMemcpyHostToDevice));
    const uint64_t split_rows = 1024;
    nsplit = (uint32_t)std::max<uint64_t>(1, ceil_div(T, split_rows));
    config_check(nsplit <= 1024, "layer.tokens: too many tokens for the split-K gate GEMM");
    std::vector<int32_t> sm(nsplit), sa(nsplit), sb(nsplit, 0);
    for (uint32_t s = 0; s < nsplit; ++s) {
      sa[s] = (int32_t)(s * split_rows);
      sm[s] = (int32_t)std::min<uint64_t>(split_rows, T - std::min<uint64_t>(T, s * split_rows));
    }
    for (uint32_t q = 0; q < nsplit; ++q) sb[q] = (int32_t)q;  // split q -> its own partial
    dwg_ws = dalloc<float>(owned, dt == MOE_DTYPE_BF16 ? (uint64_t)nsplit * dm * Epad
                                                        : std::max<uint64_t>(1, gate_wgrad_f32_ws_floats(T, dm, E)));
    split_m = dalloc<int32_t>(owned, nsplit);
    split_a = dalloc<int32_t>(owned, nsplit);
    split_b = dalloc<int32_t>(owned, nsplit);
    MOE_CUDA(cudaMemcpy(split_m, sm.data(), nsplit * 4, cudaMemcpyHostToDevice));
    MOE_CUDA(cudaMemcpy(split_a, sa.data(), nsplit * 4, cudaMemcpyHostToDevice));
    MOE_CUDA(cudaMemcpy(split_b, sb.data(), nsplit * 4, cudaMemcpyHostToDevice));
  }
  for (auto& lg : plog)
    for (int i = 0; i < kMaxPhases + 1; ++i) MOE_CUDA(cudaEventCreate(&lg.ev[i]));
}

Layer::~Layer() {
  if (p2p) p2p_teardown(win);  // device sync + BYE handshake, then unmap / free
  if (bw_side) {
    cudaStreamSynchronize(bw_side);
    cudaStreamDestroy(bw_side);
    cudaEventDestroy(bw_fork);
    cudaEventDestroy(bw_join);
  }
  for (auto& lg : plog)
    for (int i = 0; i < kMaxPhases + 1; ++i) cudaEventDestroy(lg.ev[i]);
  for (void* p : owned) cudaFree(p);
  if (x_stage) {
    for (int i = 0; i < 3; ++i) cudaStreamSynchronize(hp_stream[i]);
    cudaFree(x_stage);
    for (int i = 0; i < 3; ++i) cudaStreamDestroy(hp_stream[i]);
    for (int bb = 0; bb < 2; ++bb)
      for (int i = 0; i < 5; ++i) cudaEventDestroy(hp_ev[bb][i]);
    cudaEventDestroy(hp_entry);
  }
}

void Layer::mark(const char* name, cudaStream_t st) {
  PhaseLog& lg = plog[cur_log];
  if (!profiling || lg.n >= kMaxPhases) return;
  lg.name[lg.n] = name;
  MOE_CUDA(cudaEventRecord(lg.ev[lg.n + 1], st));
  ++lg.n;
}

void Layer::a2a(const void* send, void* recv, uint64_t bytes_per_peer, cudaStream_t st) {
  MOE_NCCL(ncclAlltoAll(send, recv, bytes_per_peer, ncclUint8, (ncclComm_t)comm, st));
}

RemoteRows Layer::remote_rows(uint64_t home_off) const {
  RemoteRows r;
  r.peers_host = win.peer_host;
  r.peers_dev = win.peer_dev;
  r.home_off = home_off;
  r.cnt = reinterpret_cast<const int32_t*>(win.base + win.off_cnt);
  r.P = P;
  r.me = rank;
  r.E = E;
  r.El = El;
  r.Cs = Cs;
  return r;
}

// One fp32 GEMM as split-bf16 tcgen05 GEMMs over K chunks of <= 512, all
// chunks in ONE launch (group (c, g) writes partial c): p is the problem on
// three-plane operands; partial c lands at out_parts + c * part_stride.
// RAGGED_M: K cut into n equal 64-multiples (per-group k_begin_g, c_row =
// c * rows + a_row); RAGGED_K: every group's rows cut at 512 (output c*El+b).
void Layer::split_gemm(moe_gemm_problem_t p, float* out_parts, uint64_t part_stride, int* nparts,
                       cudaStream_t st) {
  p.dtype_ab = MOE_DTYPE_BF16;
  p.dtype_c = MOE_DTYPE_F32;
  p.split_terms = 6;
  p.epilogue = MOE_EPI_STORE;
  p.bias = nullptr;
  p.C = out_parts;
  const uint32_t G = p.groups;
  // this forward's tables for (kind, chunks), built on first use
  auto tables = [&](int kind, uint32_t n, uint32_t chunk) -> ChunkTables& {
    const int key = kind * 4096 + (int)n * 64 + (int)(chunk / 64);
    ChunkTables* slot = &s_tab[0];
    for (auto& t : s_tab) {
      if (t.key == key && t.step == fwd_step) return t;
      if (t.step != fwd_step || t.key < 0) slot = &t;
    }
    chunk_tables(kind, G, (int)n, (int)chunk, (int)rows, (int)p.num_b, p.m, p.a_row, p.b, slot->m,
                 slot->a, kind == 0 ? slot->c : nullptr, slot->b, kind == 0 ? slot->k : nullptr,
                 st);
    slot->key = key;
    slot->step = fwd_step;
    return *slot;
  };
  if (p.kind == MOE_GEMM_RAGGED_M) {
    const uint32_t kb = p.K / 64;
    uint32_t n = 1;
    while (p.K / n > 512 || kb % n) ++n;
    const uint32_t chunk = p.K / n;
    const ChunkTables& t = tables(0, n, chunk);
    arg_check(part_stride == rows * (uint64_t)p.N, "split_gemm: RAGGED_M partial stride");
    p.groups = G * n;
    p.m = t.m;
    p.a_row = t.a;
    p.c_row = t.c;
    p.b = t.b;
    p.k_begin_g = t.k;
    p.k_len = chunk;
    p.c_rows = n * rows;
    *nparts = (int)n;
  } else {
    const uint32_t n = (uint32_t)ceil_div(gstride, (uint64_t)512);
    const ChunkTables& t = tables(1, n, 512);
    arg_check(part_stride == (uint64_t)p.num_b * p.M * p.N, "split_gemm: RAGGED_K partial stride");
    p.groups = G * n;
    p.m = t.m;
    p.a_row = t.a;
    p.b = t.b;
    p.num_b *= n;
    *nparts = (int)n;
  }
  grouped_gemm(p, st);
}

moe_gemm_problem_t Layer::expert_problem() const {
  moe_gemm_problem_t p;
  std::memset(&p, 0, sizeof(p));
  p.kind = MOE_GEMM_RAGGED_M;
  p.dtype_ab = dt;
  p.dtype_c = dt;
  p.groups = ngroups;
  p.a_rows = rows;
  p.num_b = El;
  p.m = gm;
  p.a_row = ga;
  p.c_row = ga;
  p.b = gb;
  return p;
}

void Layer::forward(const moe_layer_params_t& w, const void* x, void* y, const float* override_logits,
                    float* logits_out, const moe_routing_out_t* rout, cudaStream_t st) {
  arg_check((x != nullptr && y != nullptr) || T == 0, "forward.x/y: must be non-null");
  arg_check(w.w1 && w.w2 && w.b1 && w.b2, "forward.params: expert weights must be non-null");
  arg_check(override_logits || w.wg, "forward.params.wg: gate weight required");
  cur_log = last_log = 0;
  plog[0].n = 0;
  x_saved_ptr = x;
  if (profiling) MOE_CUDA(cudaEventRecord(plog[0].ev[0], st));
  const uint64_t ph = ++phase;
  ++fwd_step;  // new group tables this step: the split-fp32 chunk tables go stale
  if (p2p) p2p_wait(win, SLOT_PHASE, ph - 1, st);  // peers done reading our previous writes
  // K1: logits = x wg^T (+ bg), fp32 out
  if (override_logits) {
    MOE_CUDA(cudaMemcpyAsync(logits, override_logits, T * E * 4, cudaMemcpyDeviceToDevice, st));
  } else if (T && dt == MOE_DTYPE_F32) {
    gate_logits_f32(T, dm, E, static_cast<const float*>(x), static_cast<const float*>(w.wg),
                    desc.has_gate_bias ? static_cast<const float*>(w.bg) : nullptr, logits, st);
  } else if (T) {
    moe_gemm_problem_t p;
    std::memset(&p, 0, sizeof(p));
    p.kind = MOE_GEMM_RAGGED_M;
    p.epilogue = MOE_EPI_STORE;
    p.dtype_ab = dt;
    p.dtype_c = MOE_DTYPE_F32;
    p.groups = 1;
    p.N = E;
    p.K = dm;
    p.a_rows = T;
    p.num_b = 1;
    p.m = gate_tab;
    p.a_row = gate_tab + 1;
    p.c_row = gate_tab + 2;
    p.b = gate_tab + 3;
    p.A = x;
    p.B = w.wg;
    p.C = logits;
    p.bias = desc.has_gate_bias ? w.bg : nullptr;
    p.ldc = E;
    grouped_gemm(p, st);
  }
  mark("gate_gemm", st);
  // K2: routing
  moe_routing_out_t ro{expert, gate, position, keep, count1, count2, kept, aux};
  route_forward(T, E, k, C, logits, ro, rws, st);
  if (rr) relabel_experts(T, k, E, P, expert, kept, pexpert, pkept, st);
  mark("route", st);
  // K3 (+K4 in P2P mode): dispatch into the Fusion-packed send buffer, or
  // straight into the owning ranks' receive buffers over NVLink
  if (p2p) {
    p2p_counts(win, dkept(), ph, st);
    p2p_wait(win, SLOT_CNT, ph, st);
    mark("a2a_counts", st);  // count all-gather + waiting for the slowest peer's routing
    p2p_dispatch(win, T, dm, k, C, dt, x, dexp(), position, slot, ph, st);
    mark("dispatch_p2p", st);
    p2p_wait(win, SLOT_DISPATCH, ph, st);
    p2p_local_groups(win, gm, ga, gb, xr, st);
  } else {
    dispatch_tokens(T, dm, E, k, C, pad, dt, x, dexp(), position, dkept(), xs, slot, st);
    mark("dispatch", st);
  }
  // K4: counts + payload exchange (one message per peer)
  if (P > 1 && !p2p) {
    MOE_NCCL(ncclGroupStart());
    a2a(dkept(), cnt_recv, El * sizeof(int32_t), st);
    a2a(xs, xr, El * Cs * dm * esz, st);
    MOE_NCCL(ncclGroupEnd());
  }
  mark("a2a_dispatch", st);
  if (!p2p) build_groups(P, El, Cs, cnt_recv, gm, ga, gb, gmk, gak, gbk, st);
  // K5: H = X W1^T + b1 (stored), A = gelu(H); Y = A W2^T + b2
  const bool fused_return = p2p && dt == MOE_DTYPE_BF16;
  if (split32) {
    const uint64_t wn = (uint64_t)El * dff * dm;
    split_f32_bf16x3(static_cast<const float*>(xr), rows * dm, xr3, st);
    split_f32_bf16x3(static_cast<const float*>(w.w1), wn, w1_3, st);
    split_f32_bf16x3(static_cast<const float*>(w.w2), wn, w2_3, st);
    int np = 0;
    moe_gemm_problem_t p = expert_problem();
    p.N = dff;
    p.K = dm;
    p.A = xr3;
    p.B = w1_3;
    p.ldc = dff;
    split_gemm(p, s_part, rows * dff, &np, st);
    // A = gelu(h) goes straight to its bf16 planes (ffn2's and wgrad-w2's operand)
    split_finish(1, s_part, np, rows * dff, ngroups, gm, ga, gb, (uint32_t)gstride, dff, w.b1, nullptr,
                 nullptr, static_cast<float*>(Gp), a3, rows * dff, st);
    mark("ffn1", st);
    p = expert_problem();
    p.N = dm;
    p.K = dff;
    p.A = a3;
    p.B = w2_3;
    p.ldc = dm;
    split_gemm(p, s_part, rows * dm, &np, st);
    split_finish(0, s_part, np, rows * dm, ngroups, gm, ga, gb, (uint32_t)gstride, dm, w.b2, nullptr,
                 static_cast<float*>(Yl), nullptr, nullptr, 0, st);
  } else {
  {
    moe_gemm_problem_t p = expert_problem();
    p.epilogue = MOE_EPI_GELU;
    p.N = dff;
    p.K = dm;
    p.A = xr;
    p.B = w.w1;
    p.C = Aact;
    p.C2 = Gp;
    p.bias = w.b1;
    p.ldc = dff;
    grouped_gemm(p, st);
  }
  mark("ffn1", st);
  {
    moe_gemm_problem_t p = expert_problem();
    p.epilogue = MOE_EPI_STORE;
    p.N = dm;
    p.K = dff;
    p.A = Aact;
    p.B = w.w2;
    p.C = Yl;
    p.bias = w.b2;
    p.ldc = dm;
    if (fused_return) {
      // the epilogue stores Y rows straight into the source ranks' home buffers
      const RemoteRows rr = remote_rows(win.off_yh);
      grouped_gemm(p, st, &rr);
    } else {
      grouped_gemm(p, st);
    }
  }
  }  // !split32
  mark("ffn2", st);
  if (p2p) {
    if (fused_return) p2p_signal(win, SLOT_Y, ph, st);
    else p2p_push_home(win, win.off_yh, Yl, SLOT_Y, ph, st);
    p2p_wait(win, SLOT_Y, ph, st);
  } else if (P > 1) {
    a2a(Yl, Yh, El * Cs * dm * esz, st);
  }
  mark("a2a_combine", st);
  // K6: weighted combine
  combine_tokens(T, dm, k, dt, Yh, slot, gate, y, st);
  mark("combine", st);
  if (p2p) p2p_signal(win, SLOT_PHASE, ph, st);
  if (logits_out)
    MOE_CUDA(cudaMemcpyAsync(logits_out, logits, T * E * 4, cudaMemcpyDeviceToDevice, st));
  if (rout) {
    auto cp = [&](void* dst, const void* src, uint64_t n) {
      if (dst) MOE_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToDevice, st));
    };
    cp(rout->expert, expert, T * k * 4);
    cp(rout->gate, gate, T * k * 4);
    cp(rout->position, position, T * k * 4);
    cp(rout->keep, keep, T * k);
    cp(rout->count1, count1, E * 4);
    cp(rout->count2, count2, E * 4);
    cp(rout->kept, kept, E * 4);
    cp(rout->aux_loss, aux, 4);
  }
  has_forward = true;
}

// MOE_BWD_FORK=0 keeps the backward on one stream (A/B switch)
static bool bwd_fork_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MOE_BWD_FORK");
    return !(e && e[0] == '0');
  }();
  return on;
}

void Layer::backward(const moe_layer_params_t& w, const void* dy, float d_aux, void* dx,
                     const moe_layer_grads_t& g, cudaStream_t st) {
  require(has_forward, MOE_ERR_LOGIC, "backward: no forward pass recorded on this layer");
  arg_check((dy != nullptr && dx != nullptr) || T == 0, "backward.dy/dx: must be non-null");
  arg_check(g.dw1 && g.db1 && g.dw2 && g.db2 && g.dwg, "backward.grads: must be non-null");
  arg_check(w.wg != nullptr, "backward.params.wg: gate weight required");
  cur_log = last_log = 1;
  plog[1].n = 0;
  if (profiling) MOE_CUDA(cudaEventRecord(plog[1].ev[0], st));
  const uint64_t ph = ++phase;
  // K6^T: dgate and the gate-scaled dY into the send layout (+ zero pad rows),
  // or straight into the owning ranks' receive buffers (P2P)
  if (p2p) {
    p2p_wait(win, SLOT_PHASE, ph - 1, st);
    p2p_combine_bwd(win, T, dm, k, dt, dy, slot, gate, dexp(), position, dgate, ph, st);
  } else {
    combine_backward(T, dm, E, k, C, pad, dt, dy, Yh, slot, gate, dkept(), dYs, dgate, st);
  }
  mark("combine_bwd", st);
  // The received dY and its column sums (db2) do not depend on the routing
  // backward / gate weight gradient: with the fork on they run on a side
  // stream beside them (two short memory-bound chains overlap instead of
  // queueing), joined before dgrad-ffn2.  Not for the NCCL exchange (its
  // collectives stay on one stream) and not in profiled steps (phases stay
  // attributable).
  const bool fork = bwd_fork_enabled() && (p2p || P == 1) && !profiling;
  cudaStream_t sd = st;
  auto dy_and_db2 = [&](cudaStream_t s) {
    if (p2p) {
      p2p_wait(win, SLOT_DY, ph, s);
      p2p_local_groups(win, gm, ga, gb, dYr, s);  // zero the K-block pad rows of recv_dy
    }
    else if (P > 1) a2a(dYs, dYr, El * Cs * dm * esz, s);
    mark("a2a_dy", s);
    // db2 = column sums of dY, while dY is still warm in L2 (after the weight
    // gradients the L2 is full of dirty fp32 dW lines and every read pays a
    // write-back)
    if (split32)  // + dY's bf16 planes (dgrad-ffn2's / wgrad-w2's operand) in the same pass
      split_colsum_f32(static_cast<const float*>(dYr), ngroups, gm, ga, gb, El, (uint32_t)gstride,
                       dm, dy3, rows * dm, cs_part, g.db2, s);
    else
      group_colsum(ngroups, gm, ga, gb, El, dm, dt, dYr, g.db2, s, p2p ? (uint64_t)P * Cs : Cs,
                   cs_part, cs_ticket);
    mark("bias_grads", s);
  };
  if (fork) {
    if (!bw_side) {
      MOE_CUDA(cudaStreamCreateWithFlags(&bw_side, cudaStreamNonBlocking));
      MOE_CUDA(cudaEventCreateWithFlags(&bw_fork, cudaEventDisableTiming));
      MOE_CUDA(cudaEventCreateWithFlags(&bw_join, cudaEventDisableTiming));
    }
    sd = bw_side;
    MOE_CUDA(cudaEventRecord(bw_fork, st));
    MOE_CUDA(cudaStreamWaitEvent(sd, bw_fork, 0));
    dy_and_db2(sd);
    MOE_CUDA(cudaEventRecord(bw_join, sd));
  }
  // K2^T: dlogits (and dbg, summed over token blocks in a fixed order)
  route_backward(T, E, k, logits, expert, gate, keep, count1, dgate, d_aux, dl_f32, dl_lp,
                 dt == MOE_DTYPE_BF16 ? MOE_DTYPE_BF16 : MOE_DTYPE_F32,
                 dt == MOE_DTYPE_BF16 ? Epad : E, desc.has_gate_bias ? g.dbg : nullptr, dbg_ws,
                 st);
  mark("route_bwd", st);
  // gate weight gradient dwg = dlogits^T x (split-K): needs only local data,
  // so it runs while the dY rows of the peers are still arriving
  if (dt == MOE_DTYPE_F32) {
    gate_wgrad_f32(T, dm, E, dl_f32, static_cast<const float*>(x_saved_ptr), g.dwg, dwg_ws, st);
  } else if (!T) {
    MOE_CUDA(cudaMemsetAsync(g.dwg, 0, (uint64_t)E * dm * 4, st));
  } else {
    // split-K over token blocks: split q stores its [dm][Epad] partial, then
    // the partials are summed in split order and transposed to [E][dm]
    moe_gemm_problem_t p;
    std::memset(&p, 0, sizeof(p));
    p.kind = MOE_GEMM_RAGGED_K;
    p.epilogue = MOE_EPI_STORE;
    p.dtype_ab = dt;
    p.dtype_c = MOE_DTYPE_F32;
    p.groups = nsplit;
    p.M = dm;
    p.N = Epad;
    p.a_rows = T;
    p.b_rows = T;
    p.num_b = nsplit;
    p.m = split_m;
    p.a_row = split_a;
    p.b = split_b;
    p.A = x_saved_ptr;
    p.B = dl_lp;
    p.ldb = Epad;
    p.C = dwg_ws;
    p.ldc = Epad;
    grouped_gemm(p, st);
    sum_parts(dwg_ws, nsplit, (uint64_t)dm * Epad, dm, E, Epad, true, g.dwg, st);
  }
  // the replicated gate gradients are final here: push them to the peers now
  // so the closing all-reduce only sums (no wait on a late peer's push)
  const bool reduce_gate = desc.gate_grad_reduce == 0;
  if (p2p && reduce_gate)
    p2p_allreduce_push(win, g.dwg, (uint64_t)E * dm, desc.has_gate_bias ? g.dbg : nullptr,
                       desc.has_gate_bias && g.dbg ? E : 0, ph, st);
  mark("gate_wgrad", st);
  if (fork) MOE_CUDA(cudaStreamWaitEvent(st, bw_join, 0));
  else dy_and_db2(st);
  // Weight-gradient GEMMs (RAGGED_K over the slices of each expert):
  // dW1[j] = sum dH^T X, dW2[j] = sum dY^T A.
  auto wgrad = [&](bool w1, cudaStream_t s) {
    if (split32) {  // dW = sum over row chunks of split-bf16 RAGGED_K GEMMs
      moe_gemm_problem_t p;
      std::memset(&p, 0, sizeof(p));
      p.kind = MOE_GEMM_RAGGED_K;
      p.groups = ngroups;
      p.a_rows = rows;
      p.num_b = El;
      p.m = p2p ? gm : gmk;
      p.a_row = p2p ? ga : gak;
      p.b = p2p ? gb : gbk;
      p.M = w1 ? dff : dm;
      p.N = w1 ? dm : dff;
      p.A = w1 ? dh3 : dy3;
      p.B = w1 ? xr3 : a3;
      p.ldc = p.N;
      const uint64_t wn = (uint64_t)El * dff * dm;
      int np = 0;
      split_gemm(p, s_part, wn, &np, s);
      sum_parts(s_part, np, wn, 1, wn, wn, false, static_cast<float*>(w1 ? g.dw1 : g.dw2), s);
      return;
    }
    moe_gemm_problem_t p;
    std::memset(&p, 0, sizeof(p));
    p.kind = MOE_GEMM_RAGGED_K;
    p.epilogue = MOE_EPI_STORE;
    p.dtype_ab = dt;
    p.dtype_c = MOE_DTYPE_F32;
    p.groups = ngroups;
    p.a_rows = rows;
    p.num_b = El;
    p.m = p2p ? gm : gmk;
    p.a_row = p2p ? ga : gak;
    p.b = p2p ? gb : gbk;
    if (w1) {
      p.M = dff;
      p.N = dm;
      p.A = dH;
      p.B = xr;
      p.C = g.dw1;
      p.ldc = dm;
    } else {
      p.M = dm;
      p.N = dff;
      p.A = dYr;
      p.B = Aact;
      p.C = g.dw2;
      p.ldc = dff;
    }
    grouped_gemm(p, s);
  };
  // K5^T dgrad: dH = (dY W2) * gelu'(h) (stored by ffn1), db1 = column sums
  // of dH fused into the same epilogue (per-block partials, fixed-order sum);
  // dXe = dH W1
  const bool fused_return = p2p && dt == MOE_DTYPE_BF16;
  if (split32) {
    int np = 0;  // dy3: dY's planes, written with db2 (bias_grads)
    moe_gemm_problem_t p = expert_problem();
    p.b_mn_major = 1;
    p.N = dff;
    p.K = dm;
    p.A = dy3;
    p.B = w2_3;
    p.ldc = dff;
    split_gemm(p, s_part, rows * dff, &np, st);
    // dH = h * gelu'(h) to its bf16 planes (dgrad-ffn1's / wgrad-w1's operand)
    // and db1 = its column sums (chunk partials in s_cs, fixed-order sum)
    split_finish_dgelu_colsum(s_part, np, rows * dff, ngroups, gm, ga, gb, El, (uint32_t)gstride,
                              dff, static_cast<const float*>(Gp), nullptr, dh3, rows * dff, s_cs,
                              g.db1, st);
    mark("dgrad_ffn2", st);
    p = expert_problem();
    p.b_mn_major = 1;
    p.N = dm;
    p.K = dff;
    p.A = dh3;
    p.B = w1_3;
    p.ldc = dm;
    split_gemm(p, s_part, rows * dm, &np, st);
    split_finish(0, s_part, np, rows * dm, ngroups, gm, ga, gb, (uint32_t)gstride, dm, nullptr, nullptr,
                 static_cast<float*>(dXl), nullptr, nullptr, 0, st);
  } else {
  {
    moe_gemm_problem_t p = expert_problem();
    p.epilogue = MOE_EPI_DGELU;
    p.b_mn_major = 1;
    p.N = dff;
    p.K = dm;
    p.A = dYr;
    p.B = w.w2;
    p.C = dH;
    p.aux = Gp;
    p.colsum = g.db1;
    p.colsum_ws = db1_ws;
    p.colsum_max_m = p2p ? (uint64_t)P * Cs : Cs;
    p.ldc = dff;
    grouped_gemm(p, st);
  }
  mark("dgrad_ffn2", st);
  {
    moe_gemm_problem_t p = expert_problem();
    p.epilogue = MOE_EPI_STORE;
    p.b_mn_major = 1;
    p.N = dm;
    p.K = dff;
    p.A = dH;
    p.B = w.w1;
    p.C = dXl;
    p.ldc = dm;
    if (fused_return) {
      const RemoteRows rr = remote_rows(win.off_dxh);  // dX rows straight to their sources
      grouped_gemm(p, st, &rr);
    } else {
      grouped_gemm(p, st);
    }
  }
  }  // !split32
  mark("dgrad_ffn1", st);
  if (p2p) {
    if (fused_return) p2p_signal(win, SLOT_DX, ph, st);
    else p2p_push_home(win, win.off_dxh, dXl, SLOT_DX, ph, st);
  }
  else if (P > 1) a2a(dXl, dXh, El * Cs * dm * esz, st);
  mark("a2a_dx", st);
  wgrad(true, st);
  mark("wgrad_w1", st);
  wgrad(false, st);
  mark("wgrad_w2", st);
  if (p2p) p2p_wait(win, SLOT_DX, ph, st);
  // gate dgrad with the combine backward folded into its epilogue:
  // dx[t] = dlogits[t] wg + sum_i dXe[slot_i]
  if (T && dt == MOE_DTYPE_F32) {
    gate_dx_f32(T, dm, E, k, dl_f32, static_cast<const float*>(w.wg),
                static_cast<const float*>(dXh), slot, static_cast<float*>(dx), st);
  } else if (T) {
    moe_gemm_problem_t p;
    std::memset(&p, 0, sizeof(p));
    p.kind = MOE_GEMM_RAGGED_M;
    p.epilogue = MOE_EPI_GATHER_ADD;
    p.dtype_ab = dt;
    p.dtype_c = dt;
    p.b_mn_major = 1;
    p.groups = 1;
    p.N = dm;
    p.K = dt == MOE_DTYPE_BF16 ? Epad : E;
    p.a_rows = T;
    p.num_b = 1;
    p.b_rows = E;
    p.m = gate_tab;
    p.a_row = gate_tab + 1;
    p.c_row = gate_tab + 2;
    p.b = gate_tab + 3;
    p.A = dt == MOE_DTYPE_BF16 ? dl_lp : (const void*)dl_f32;
    p.B = w.wg;
    p.C = dx;
    p.ldc = dm;
    p.gather_src = dXh;
    p.gather_idx = slot;
    p.gather_k = k;
    grouped_gemm(p, st);
  }
  mark("gate_dgrad_gather_dx", st);
  if (p2p && reduce_gate) {
    // replicated gate gradients: sum the pushed partials in rank order
    p2p_allreduce_finish(win, g.dwg, (uint64_t)E * dm, desc.has_gate_bias ? g.dbg : nullptr,
                         desc.has_gate_bias && g.dbg ? E : 0, ph, st);
  } else if (P > 1 && reduce_gate) {
    MOE_NCCL(ncclGroupStart());
    MOE_NCCL(ncclAllReduce(g.dwg, g.dwg, (uint64_t)E * dm, ncclFloat32, ncclSum, (ncclComm_t)comm, st));
    if (desc.has_gate_bias && g.dbg)
      MOE_NCCL(ncclAllReduce(g.dbg, g.dbg, E, ncclFloat32, ncclSum, (ncclComm_t)comm, st));
    MOE_NCCL(ncclGroupEnd());
  }
  mark("allreduce_gate", st);
  if (p2p) p2p_signal(win, SLOT_PHASE, ph, st);
}

void Layer::train_step_host(const moe_layer_params_t& w, const void* x_host, const void* dy_host,
                            float d_aux, void* y_host, void* dx_host, const moe_layer_grads_t& g,
                            cudaStream_t st, bool deferred) {
  // Three-stream pipeline over double-buffered staging: H2D of step i+1 and
  // D2H of step i-1 overlap the compute of step i (PCIe is full duplex and the
  // copy engines need no SMs).  Finer-grained than whole steps: the forward
  // starts once x has landed (dy still in flight), y goes back to the host
  // while the backward runs, and input / output stages are released
  // separately (the H2D of step i+2 only waits for the compute of step i, the
  // forward of step i+2 for the D2H of step i), so in steady state each copy
  // engine streams back to back and the step time is max(H2D, compute, D2H).
  // The caller's stream waits for this step's D2H, so y_host / dx_host / the
  // gradients are valid once `st` reaches this call.
  const uint64_t bytes = T * dm * esz;
  if (!x_stage) {
    MOE_CUDA(cudaMalloc(&x_stage, 8 * bytes + 64));
    for (int i = 0; i < 3; ++i) MOE_CUDA(cudaStreamCreateWithFlags(&hp_stream[i], cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b)
      for (int i = 0; i < 5; ++i)
        MOE_CUDA(cudaEventCreateWithFlags(&hp_ev[b][i], cudaEventDisableTiming));
    MOE_CUDA(cudaEventCreateWithFlags(&hp_entry, cudaEventDisableTiming));
    // the first step's copies must not start before work already queued on st
    MOE_CUDA(cudaEventRecord(hp_entry, st));
    MOE_CUDA(cudaStreamWaitEvent(hp_stream[0], hp_entry, 0));
  }
  cudaStream_t h2d = hp_stream[0], comp = hp_stream[1], d2h = hp_stream[2];
  // Every call: the compute stream waits for whatever the caller queued on st
  // since the last call (an optimizer step writing params, a consumer reading
  // the gradients this step's backward overwrites).  The copy-in stream does
  // not: it only reads the caller's host buffers and writes private staging.
  MOE_CUDA(cudaEventRecord(hp_entry, st));
  MOE_CUDA(cudaStreamWaitEvent(comp, hp_entry, 0));
  const int b = (int)(hp_iter & 1);
  cudaEvent_t* ev_b = hp_ev[b];
  uint8_t* base = static_cast<uint8_t*>(x_stage) + (uint64_t)b * 4 * bytes;
  void* xd = base;
  void* dyd = base + bytes;
  void* yd = base + 2 * bytes;
  void* dxd = base + 3 * bytes;
  if (hp_iter >= 2) MOE_CUDA(cudaStreamWaitEvent(h2d, ev_b[3], 0));  // inputs b consumed
  MOE_CUDA(cudaMemcpyAsync(xd, x_host, bytes, cudaMemcpyHostToDevice, h2d));
  MOE_CUDA(cudaEventRecord(ev_b[0], h2d));
  MOE_CUDA(cudaMemcpyAsync(dyd, dy_host, bytes, cudaMemcpyHostToDevice, h2d));
  MOE_CUDA(cudaEventRecord(ev_b[1], h2d));
  MOE_CUDA(cudaStreamWaitEvent(comp, ev_b[0], 0));
  if (hp_iter >= 2) MOE_CUDA(cudaStreamWaitEvent(comp, ev_b[4], 0));  // outputs b drained
  forward(w, xd, yd, nullptr, nullptr, nullptr, comp);
  MOE_CUDA(cudaEventRecord(ev_b[2], comp));
  MOE_CUDA(cudaStreamWaitEvent(comp, ev_b[1], 0));
  backward(w, dyd, d_aux, dxd, g, comp);
  MOE_CUDA(cudaEventRecord(ev_b[3], comp));
  MOE_CUDA(cudaStreamWaitEvent(d2h, ev_b[2], 0));
  MOE_CUDA(cudaMemcpyAsync(y_host, yd, bytes, cudaMemcpyDeviceToHost, d2h));
  MOE_CUDA(cudaStreamWaitEvent(d2h, ev_b[3], 0));
  MOE_CUDA(cudaMemcpyAsync(dx_host, dxd, bytes, cudaMemcpyDeviceToHost, d2h));
  MOE_CUDA(cudaEventRecord(ev_b[4], d2h));
  if (!deferred) {
    MOE_CUDA(cudaStreamWaitEvent(st, ev_b[4], 0));
  } else {
    // Deferred outputs: st waits for this step's compute (gradients final,
    // params free to update) and for the PREVIOUS step's copy-out, so the
    // D2H of step i overlaps the compute of step i+1 even when the caller
    // queues an optimizer step on st between calls.
    MOE_CUDA(cudaStreamWaitEvent(st, ev_b[3], 0));
    if (hp_iter >= 1) MOE_CUDA(cudaStreamWaitEvent(st, hp_ev[b ^ 1][4], 0));
  }
  ++hp_iter;
}

void Layer::host_sync(cudaStream_t st) {
  if (!x_stage || hp_iter == 0) return;
  // the copy-out stream is in order: the last step's event covers all
  MOE_CUDA(cudaStreamWaitEvent(st, hp_ev[(hp_iter - 1) & 1][4], 0));
}

// --------------------------------------------------------------- comm -----
void comm_unique_id(uint8_t id[128]) {
  ncclUniqueId u;
  MOE_NCCL(ncclGetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
}

void* comm_create(const uint8_t id[128], uint32_t nranks, uint32_t rank) {
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t c = nullptr;
  MOE_NCCL(ncclCommInitRank(&c, (int)nranks, u, (int)rank));
  return c;
}

void comm_destroy(void* c) {
  if (c) MOE_NCCL(ncclCommDestroy((ncclComm_t)c));
}

void alltoall_packed(void* comm, const void* send, void* recv, uint64_t bytes_per_peer,
                     uint32_t slices_per_peer, int fused, cudaStream_t st) {
  ncclComm_t c = (ncclComm_t)comm;
  int n = 0, me = 0;
  MOE_NCCL(ncclCommCount(c, &n));
  MOE_NCCL(ncclCommUserRank(c, &me));
  if (fused || slices_per_peer <= 1) {
    MOE_NCCL(ncclAlltoAll(send, recv, bytes_per_peer, ncclUint8, c, st));
    return;
  }
  arg_check(bytes_per_peer % slices_per_peer == 0,
            "alltoall.slices_per_peer: must divide bytes_per_peer");
  const uint64_t sl = bytes_per_peer / slices_per_peer;
  MOE_NCCL(ncclGroupStart());
  for (int p = 0; p < n; ++p) {
    for (uint32_t s = 0; s < slices_per_peer; ++s) {
      const uint64_t off = (uint64_t)p * bytes_per_peer + s * sl;
      MOE_NCCL(ncclSend(static_cast<const uint8_t*>(send) + off, sl, ncclUint8, p, c, st));
      MOE_NCCL(ncclRecv(static_cast<uint8_t*>(recv) + off, sl, ncclUint8, p, c, st));
    }
  }
  MOE_NCCL(ncclGroupEnd());
}

}  // namespace moe
