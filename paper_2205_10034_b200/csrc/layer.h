// Internal MoE-layer object behind the opaque moe_layer_t handle.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "ep_p2p.h"
#include "kernels.h"
#include "moe_b200.h"

namespace moe {

struct Layer {
  static constexpr int kMaxPhases = 32;

  explicit Layer(const moe_layer_desc_t& d);
  ~Layer();
  Layer(const Layer&) = delete;
  Layer& operator=(const Layer&) = delete;

  void forward(const moe_layer_params_t& w, const void* x, void* y, const float* override_logits,
               float* logits_out, const moe_routing_out_t* rout, cudaStream_t st);
  void backward(const moe_layer_params_t& w, const void* dy, float d_aux, void* dx,
                const moe_layer_grads_t& g, cudaStream_t st);
  void train_step_host(const moe_layer_params_t& w, const void* x_host, const void* dy_host,
                       float d_aux, void* y_host, void* dx_host, const moe_layer_grads_t& g,
                       cudaStream_t st, bool deferred = false);
  // deferred-output mode: make st wait for every outstanding copy-out
  void host_sync(cudaStream_t st);

  moe_gemm_problem_t expert_problem() const;
  RemoteRows remote_rows(uint64_t home_off) const;
  void a2a(const void* send, void* recv, uint64_t bytes_per_peer, cudaStream_t st);
  void mark(const char* name, cudaStream_t st);

  moe_layer_desc_t desc;
  uint32_t E = 0, k = 0, dm = 0, dff = 0, P = 1, rank = 0, El = 0, Epad = 0;
  uint64_t T = 0, C = 0, Cs = 0, rows = 0;
  uint32_t pad = 1;
  moe_dtype_t dt = MOE_DTYPE_BF16;
  uint64_t esz = 2;
  void* comm = nullptr;
  int device = 0;
  bool p2p = false;       // EP exchange over NVLink peer memory
  P2PWindow win;
  uint64_t phase = 0;     // forward/backward phase counter (P2P epochs)
  uint32_t ngroups = 1;   // expert GEMM groups: P*El slices, or El experts (P2P)

  std::vector<void*> owned;
  // routing state
  float* logits = nullptr;
  int32_t *expert = nullptr, *position = nullptr, *slot = nullptr;
  float* gate = nullptr;
  uint8_t* keep = nullptr;
  int32_t *count1 = nullptr, *count2 = nullptr, *kept = nullptr;
  float* aux = nullptr;
  RouteWorkspace rws;
  // token/expert buffers
  void *xs = nullptr, *xr = nullptr;
  int32_t* cnt_recv = nullptr;
  int32_t *gm = nullptr, *ga = nullptr, *gb = nullptr, *gmk = nullptr, *gak = nullptr,
          *gbk = nullptr;
  // round-robin placement: physical expert ids / kept counts for the exchange
  bool rr = false;
  int32_t *pexpert = nullptr, *pkept = nullptr;
  const int32_t* dexp() const { return rr ? pexpert : expert; }
  const int32_t* dkept() const { return rr ? pkept : kept; }
  float* cs_part = nullptr;      // db2 chunk partials (group_colsum)
  int32_t* cs_ticket = nullptr;  // db2 chunk tickets, self re-arming
  float* db1_ws = nullptr;       // db1 partials of the DGELU epilogue [groups][rows/32][dff]
  float* dbg_ws = nullptr;       // dbg partials [token blocks][E]
  float* dwg_ws = nullptr;       // dwg split-K partials [nsplit][dm][Epad] (fp32: [T/128][E][dm])
  void *Gp = nullptr, *Aact = nullptr, *Yl = nullptr, *Yh = nullptr;
  // backward buffers
  float* dgate = nullptr;
  void *dYs = nullptr, *dYr = nullptr, *dH = nullptr, *dXl = nullptr, *dXh = nullptr;
  float* dl_f32 = nullptr;
  void* dl_lp = nullptr;
  // gate GEMM tables
  int32_t* gate_tab = nullptr;
  int32_t *split_m = nullptr, *split_a = nullptr, *split_b = nullptr;
  uint32_t nsplit = 1;
  // fp32 expert GEMMs on the bf16 tensor cores (f32split.cu): three bf16
  // planes per operand, K-chunk partials summed in fp32 by split_finish
  bool split32 = false;
  uint64_t gstride = 0;  // rows per expert group (P2P: P * Cs, else Cs)
  void *xr3 = nullptr, *a3 = nullptr, *dy3 = nullptr, *dh3 = nullptr, *w1_3 = nullptr,
       *w2_3 = nullptr;
  float* s_part = nullptr;        // K-chunk partials
  float* s_cs = nullptr;          // db1 column-sum chunk partials (N = d_ff)
  // K-chunk group tables (m, a_row, c_row, b, k) of the split-fp32 GEMM
  // launches, built once per forward (the group tables are fixed by then) for
  // each (kind, chunks) shape: 4 slots
  struct ChunkTables {
    int32_t *m = nullptr, *a = nullptr, *c = nullptr, *b = nullptr, *k = nullptr;
    int key = -1;
    uint64_t step = 0;
  } s_tab[4];
  uint64_t fwd_step = 0;
  void split_gemm(moe_gemm_problem_t p, float* out_parts, uint64_t part_stride, int* nparts,
                  cudaStream_t st);
  const void* x_saved_ptr = nullptr;
  void* x_stage = nullptr;          // host-buffer pipeline: 2 x (x, dy, y, dx)
  cudaStream_t hp_stream[3] = {};   // h2d, compute, d2h
  cudaStream_t bw_side = nullptr;    // backward: dY receipt + db2 beside the routing backward
  cudaEvent_t bw_fork = nullptr, bw_join = nullptr;
  // per stage: x landed, dy landed, forward done, backward done, d2h done
  cudaEvent_t hp_ev[2][5] = {};
  cudaEvent_t hp_entry = nullptr;   // caller-stream state at each train_step_host entry
  uint64_t hp_iter = 0;
  bool has_forward = false;
  // profiling
  bool profiling = false;
  // per-phase events of the last forward (0) and the last backward (1): kept
  // apart so a caller can read both after one synchronisation
  struct PhaseLog {
    int n = 0;
    const char* name[kMaxPhases] = {};
    cudaEvent_t ev[kMaxPhases + 1] = {};
  } plog[2];
  int cur_log = 0;   // the call being recorded
  int last_log = 0;  // the most recent call
};

void comm_unique_id(uint8_t id[128]);
void* comm_create(const uint8_t id[128], uint32_t nranks, uint32_t rank);
void comm_destroy(void* c);
void alltoall_packed(void* comm, const void* send, void* recv, uint64_t bytes_per_peer,
                     uint32_t slices_per_peer, int fused, cudaStream_t st);

// moesim_ops.cu
void copy_chunks_device(uint64_t n, const uint64_t* lens, const uint64_t* in_off,
                        const uint8_t* in, const uint64_t* out_off, uint8_t* out, uint64_t max_len,
                        cudaStream_t st);
void gen_trace_device(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                      uint64_t tokens, double skew, uint64_t* counts, cudaStream_t st);
void imbalance_device(uint64_t rows, uint32_t experts, const uint64_t* counts,
                      unsigned long long* out2, cudaStream_t st);
void alltoall_flat_device(uint64_t R, const uint64_t* lens, const uint64_t* in_off,
                          const uint8_t* in, const uint64_t* out_off, uint8_t* out,
                          uint64_t max_len, cudaStream_t st);
void fuse_slices_device(uint64_t n, const uint8_t* const* slices, const uint64_t* lens,
                        uint8_t* blob, moe_slice_index_entry_t* index, uint64_t max_len,
                        cudaStream_t st);
void split_blob_device(uint64_t blob_len, const uint8_t* blob, uint64_t n,
                       const moe_slice_index_entry_t* index, uint8_t* const* out, int32_t* bad,
                       uint64_t max_len, cudaStream_t st);

}  // namespace moe
