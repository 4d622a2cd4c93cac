// Internal kernel entry points (host launchers) shared by the library's
// translation units.  Not part of the public ABI (include/moe_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "moe_b200.h"

namespace moe {

// Kernel launch accounting (moe_kernel_launch_count).
void count_launch(uint64_t n = 1);

// Remote row destinations for expert parallelism over peer memory: output row
// r of local expert group j came from source s (rows [off_s, off_s + cnt[s][e])
// of the group, e = me*El + j) and is stored straight into rank s's buffer at
// window offset `home_off`, row e*Cs + (r - off_s) — the GEMM epilogue performs
// the return all-to-all tile by tile.
struct RemoteRows {
  uint8_t* const* peers_host;  // [P] window bases (host copies, for tensor maps)
  uint8_t** peers_dev;         // [P] window bases (device array)
  uint64_t home_off;
  const int32_t* cnt;          // device [P][E] kept counts
  uint32_t P, me, E, El;
  uint64_t Cs;
};

// Upper bound on the CTAs (SMs) a persistent tcgen05 GEMM launched from this
// thread may occupy (0: all SMs).  Used to run two GEMMs side by side on
// disjoint SM sets; set with the scoped GemmCtaBudget.
int& gemm_cta_budget();
// MOE_GEMM_MC=0 disables the 2-pair multicast clusters of the expert GEMMs (A/B switch)
bool gemm_multicast_enabled();
struct GemmCtaBudget {
  int saved;
  explicit GemmCtaBudget(int n) : saved(gemm_cta_budget()) { gemm_cta_budget() = n; }
  ~GemmCtaBudget() { gemm_cta_budget() = saved; }
};

// K5: grouped GEMM. bf16 -> tcgen05 (gemm_tc.cu), fp32 -> SIMT FFMA (gemm_simt.cu).
void tc_grouped_gemm(const moe_gemm_problem_t& p, cudaStream_t st,
                     const RemoteRows* remote = nullptr);
void simt_grouped_gemm(const moe_gemm_problem_t& p, cudaStream_t st);
inline void grouped_gemm(const moe_gemm_problem_t& p, cudaStream_t st,
                         const RemoteRows* remote = nullptr) {
  if (p.dtype_ab == MOE_DTYPE_BF16) tc_grouped_gemm(p, st, remote);
  else simt_grouped_gemm(p, st);
}

// K2: routing over fp32 logits (routing.cu).
struct RouteWorkspace {
  int32_t* chunk_cnt = nullptr;  // [2][nchunks][E]
  int32_t* chunk_off = nullptr;  // [2][nchunks][E]
  float* psum_part = nullptr;    // [E][nchunks] partial softmax mass, then [E] totals
  int32_t* rank_local = nullptr; // [T][k]
  uint64_t nchunks = 0;
};
uint64_t route_chunks(uint64_t T);
void route_forward(uint64_t T, uint32_t E, uint32_t k, uint64_t C, const float* logits,
                   const moe_routing_out_t& out, const RouteWorkspace& ws, cudaStream_t st);

// Routing backward: dlogits [T, ld] (fp32 and/or bf16 copy) from dgate [T,k]
// and d_aux.  Columns E..ld-1 of the bf16 copy are zeroed.
void route_backward(uint64_t T, uint32_t E, uint32_t k, const float* logits, const int32_t* expert,
                    const float* gate, const uint8_t* keep, const int32_t* count1,
                    const float* dgate, float d_aux, float* dlogits_f32, void* dlogits_lp,
                    moe_dtype_t lp_dtype, uint32_t ld, float* dbg, float* dbg_ws,
                    cudaStream_t st);
inline uint64_t route_dbg_ws_floats(uint64_t T, uint32_t E) { return ((T + 63) / 64) * E; }

// K3: dispatch tokens into the slot buffer [E][C][d] (send layout: rank-major,
// then local expert, then position).  slot[t*k+i] = e*C+pos or -1.
// Rows [kept_e, round_up(kept_e, pad)) of every expert are zero-filled.
void dispatch_tokens(uint64_t T, uint32_t d, uint32_t E, uint32_t k, uint64_t C, uint32_t pad,
                     moe_dtype_t dt, const void* x, const int32_t* expert, const int32_t* position,
                     const int32_t* kept, void* buf, int32_t* slot, cudaStream_t st);

// K6: combine y[t] = sum_i keep_i g_i Y[slot_i] (fp32 accumulate).
void combine_tokens(uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt, const void* Y,
                    const int32_t* slot, const float* gate, void* y, cudaStream_t st);

// K6 backward: dgate[t,i] = <dy_t, Y[slot_i]>, dY[slot_i] = g_i * dy_t; pad rows
// of dY zero-filled like dispatch.
void combine_backward(uint64_t T, uint32_t d, uint32_t E, uint32_t k, uint64_t C, uint32_t pad,
                      moe_dtype_t dt, const void* dy, const void* Y, const int32_t* slot,
                      const float* gate, const int32_t* kept, void* dY, float* dgate,
                      cudaStream_t st);

// fp32 gate GEMMs (gate_f32.cu): logits = x wg^T (+ bg); dwg = dl^T x
// (zeroes dwg first); dx = dl wg + sum_i dXe[slot_i].  E <= 256.
void gate_logits_f32(uint64_t T, uint32_t d, uint32_t E, const float* x, const float* wg,
                     const float* bg, float* logits, cudaStream_t st);
void gate_wgrad_f32(uint64_t T, uint32_t d, uint32_t E, const float* dl, const float* x,
                    float* dwg, float* ws, cudaStream_t st);
constexpr int kGateWgradTok = 32;  // tokens per gate_wgrad_f32 block (one partial each)
inline uint64_t gate_wgrad_f32_ws_floats(uint64_t T, uint32_t d, uint32_t E) {
  return ((T + kGateWgradTok - 1) / kGateWgradTok) * (uint64_t)E * d;
}
void gate_dx_f32(uint64_t T, uint32_t d, uint32_t E, uint32_t k, const float* dl, const float* wg,
                 const float* dXe, const int32_t* slot, float* dx, cudaStream_t st);

// dx[t] = dx_gate[t] (fp32, may be null) + sum_i dXe[slot_i].
void gather_dx(uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt, const void* dXe,
               const int32_t* slot, const float* dx_gate, void* dx, cudaStream_t st);

// Column sums over the valid rows of each (source, expert) slot group:
// out[b][n] = sum over groups g with gb[g]==b of sum_{r<m[g]} X[a_row[g]+r][n].
// With one group per b (bf16), deterministic: row chunks of 256 rows reduce
// through part_ws (colsum_ws_floats) in chunk order; ticket
// (colsum_ticket_ints, zeroed once) re-arms itself.
uint64_t colsum_ws_floats(uint32_t groups, uint32_t N, uint64_t max_rows);
uint64_t colsum_ticket_ints(uint32_t groups, uint32_t N);
void group_colsum(uint32_t groups, const int32_t* gm, const int32_t* ga, const int32_t* gb,
                  uint32_t num_b, uint32_t N, moe_dtype_t dt, const void* X, float* out,
                  cudaStream_t st, uint64_t max_rows, float* part_ws = nullptr,
                  int32_t* ticket = nullptr);

// Fixed-order reductions (reduce.cu) replacing float atomics on the gradient
// paths, so gradients are bitwise reproducible:
//   sum_parts : out[r][c] (or out[c][r] when transpose) =
//               sum_{p < nparts} part[p*part_stride + r*ldp + c], p ascending
//   seg_colsum: out[b][n] = sum over groups g (ascending) with gb[g] == b of
//               sum_{ch < ceil(gm[g]/chunk)} ws[(g*maxch + ch)*N + n]
void sum_parts(const float* part, uint32_t nparts, uint64_t part_stride, uint64_t rows,
               uint64_t cols, uint64_t ldp, bool transpose, float* out, cudaStream_t st);
void seg_colsum(uint32_t groups, const int32_t* gm, const int32_t* gb, uint32_t num_b, uint32_t N,
                uint32_t chunk, uint32_t maxch, const float* ws, float* out, cudaStream_t st);
// Workspace of the DGELU column-sum epilogue (moe_gemm_problem_t.colsum_ws):
// [groups][ceil(max_m / 32)][N] floats.
inline uint64_t gemm_colsum_ws_floats(uint32_t groups, uint32_t N, uint64_t max_m) {
  return (uint64_t)groups * ((max_m + 31) / 32) * N;
}

// fp32 GEMMs on the bf16 tensor cores (f32split.cu): x = p0 + p1 + p2 bf16
// planes (out = 3 stacked planes of n), and the fused K-chunk sum + epilogue
// (mode 0: + bias; 1: GeLU / GeLU' of (sum + bias) into out / out2; 2: sum x
// aux) over the rows of each group, pad rows [m, stride) zeroed.
void split_f32_bf16x3(const float* in, uint64_t n, void* out, cudaStream_t st);
// MODE 2 with the bias gradient fused: db[gb[g]] = column sums of the stored
// rows (32-row chunk partials in cs_part [groups][ceil(stride/32)][N], then
// seg_colsum in chunk order)
void split_finish_dgelu_colsum(const float* part, int nparts, uint64_t part_stride,
                               uint32_t groups, const int32_t* gm, const int32_t* ga,
                               const int32_t* gb, uint32_t num_b, uint32_t stride, uint32_t N,
                               const float* aux, float* out, void* out3, uint64_t n3,
                               float* cs_part, float* db, cudaStream_t st);
// fp32 rows -> their three bf16 planes, and db = column sums of each group's
// rows (same chunk partials + seg_colsum); rows past round_up(m, 64) untouched
void split_colsum_f32(const float* in, uint32_t groups, const int32_t* gm, const int32_t* ga,
                      const int32_t* gb, uint32_t num_b, uint32_t stride, uint32_t N, void* out3,
                      uint64_t n3, float* cs_part, float* db, cudaStream_t st);
void split_finish(int mode, const float* part, int nparts, uint64_t part_stride, uint32_t groups,
                  const int32_t* gm, const int32_t* ga, const int32_t* gb, uint32_t stride,
                  uint32_t N, const float* bias, const float* aux, float* out, float* out2,
                  void* out3 = nullptr, uint64_t n3 = 0, cudaStream_t st = nullptr);
// K-chunk group tables (group (c, g) = c*groups + g): RAGGED_M (kind 0) keeps
// the rows and sets c_row = c*rows + a_row, k = c*chunk; RAGGED_K (kind 1) cuts
// every group's rows into chunks: m = clamp(m - c*chunk, 0, chunk), a_row +=
// c*chunk, output b = c*nb + b.  oc / ok unused (nullable) for kind 1.
void chunk_tables(int kind, uint32_t groups, int nchunks, int chunk, int rows, int nb,
                  const int32_t* gm, const int32_t* ga, const int32_t* gb, int32_t* om,
                  int32_t* oa, int32_t* oc, int32_t* ob, int32_t* ok, cudaStream_t st);

// Round-robin placement relabel (include/moe_b200.h): pexpert = pi(expert),
// pkept[pi(e)] = kept[e], pi(e) = (e % P) * (E / P) + e / P.
void relabel_experts(uint64_t T, uint32_t k, uint32_t E, uint32_t P, const int32_t* expert,
                     const int32_t* kept, int32_t* pexpert, int32_t* pkept, cudaStream_t st);

// Build the expert GEMM group tables for P source ranks x El local experts from
// the received kept counts cnt[s][j]: group g = s*El + j, m = cnt, a_row =
// (s*El+j)*Cs (Cs = slot stride), b = j.  Also the RAGGED_K order (grouped by
// expert): gk = j*P + s with the same rows.
void build_groups(uint32_t P, uint32_t El, uint64_t Cs, const int32_t* cnt, int32_t* gm,
                  int32_t* ga, int32_t* gb, int32_t* gm_k, int32_t* ga_k, int32_t* gb_k,
                  cudaStream_t st);

// Data-plane helpers (moesim_ops.cu).
void fill_uniform(void* out, uint64_t n, moe_dtype_t dt, uint64_t seed, double lo, double hi,
                  cudaStream_t st);
void convert_f32_to(const float* in, void* out, uint64_t n, moe_dtype_t dt, cudaStream_t st);

}  // namespace moe
