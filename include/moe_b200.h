/*
 * moe_b200.h — C-ABI of the B200-native SE-MoE MoE-layer hot path.
 *
 * The reference (`/root/reference/proj`, "moesim") exposes its path only as the
 * C++ library target moesim::core (core/CMakeLists.txt:3-25) with value-type
 * signatures and C++ exceptions.  This header is the drop-in boundary:
 *
 *   1. moesim_* — byte/bit-exact equivalents of the reference functions that
 *      exist on the path, executed on the GPU, with host buffers in and out
 *      (the reference's calling convention).  The C++ wrappers in
 *      include/moesim_b200.hpp restore the reference's exact signatures and
 *      exception types.
 *   2. moe_*    — the performance path on device pointers (the MoE-layer operator
 *      the reference does not have).
 *
 * Conventions:
 *   - every call returns moe_status_t; moe_last_error() returns the thread-local
 *     message of the last failing call in the reference's "<field>: <reason>"
 *     form;
 *   - MOE_ERR_INVALID_ARGUMENT <-> std::invalid_argument,
 *     MOE_ERR_OUT_OF_RANGE <-> std::out_of_range, MOE_ERR_CONFIG <->
 *     moesim::ConfigError, MOE_ERR_LOGIC <-> std::logic_error;
 *   - device calls enqueue on the caller's stream (cudaStream_t passed as void*)
 *     and never synchronise the host unless documented;
 *   - the caller owns activations and parameters; a handle owns its workspaces.
 *   - no torch types, plain pointers and sizes only.
 */
#ifndef MOE_B200_H_
#define MOE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOE_ABI_VERSION 1

typedef enum moe_status {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument  (collectives.cpp:11-13)      */
  MOE_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range      (topology.cpp:48,62-63)       */
  MOE_ERR_CONFIG = 3,           /* moesim::ConfigError    (types.hpp:24-26)             */
  MOE_ERR_LOGIC = 4,            /* std::logic_error       (sim_engine.cpp:31)           */
  MOE_ERR_CUDA = 5,
  MOE_ERR_NCCL = 6
} moe_status_t;

typedef enum moe_dtype { MOE_DTYPE_F32 = 0, MOE_DTYPE_BF16 = 1 } moe_dtype_t;

const char* moe_last_error(void);
int moe_abi_version(void);
/* Number of kernels this library launched since load (all entry points). */
uint64_t moe_kernel_launch_count(void);
/* sizeof() of an ABI struct by type name ("moe_gemm_problem_t", ...), 0 if
 * unknown — lets FFI bindings verify their struct layouts at load time. */
uint64_t moe_abi_sizeof(const char* type_name);

/* ======================================================================
 * 1. moesim compatibility layer (host buffers, device execution)
 * ====================================================================== */

/* moesim::SliceIndexEntry (collectives.hpp:60-66). */
typedef struct moe_slice_index_entry {
  uint64_t slice_id;
  uint64_t offset;
  uint64_t length;
} moe_slice_index_entry_t;

/* moesim::alltoall_flat (collectives.hpp:36, collectives.cpp:10-21):
 * out[i][j] = in[j][i].  The R x R chunk matrix is flattened row-major
 * [src][dst]: lens[n_chunks], data = concatenation in that order; the output
 * uses the same convention.  n_chunks != ranks*ranks -> INVALID_ARGUMENT
 * ("alltoall: payload is not a square rank matrix"). */
moe_status_t moesim_alltoall_flat(uint64_t ranks, uint64_t n_chunks, const uint64_t* lens,
                                  const uint8_t* data, uint64_t* out_lens, uint8_t* out_data);

/* collectives.cpp:31-79 alltoall_hierarchical on a (clusters, nodes_per_cluster,
 * gpus_per_node) topology: phase 1 stages every chunk inside its source node
 * on the GPU whose local rank matches the destination's (NVLink), phase 2
 * moves it along the rail; delivered chunks equal moesim_alltoall_flat.  Both
 * phases run on the GPU.  stats (NULL or 14 entries): phase-1 hops per link
 * class [nvlink, pcie, ssd_io, tor, leaf, spin], phase-2 hops, phase-1 and
 * phase-2 transfer counts (AlltoAllStats, collectives.hpp:38-47).  Errors as
 * the reference: CONFIG for a zero topology dimension, INVALID_ARGUMENT for a
 * non-square payload or a rank count that differs from the topology's. */
moe_status_t moesim_alltoall_hierarchical(uint32_t clusters, uint32_t nodes_per_cluster,
                                          uint32_t gpus_per_node, uint64_t ranks,
                                          uint64_t n_chunks, const uint64_t* lens,
                                          const uint8_t* data, uint64_t* out_lens,
                                          uint8_t* out_data, uint64_t* stats);

/* moesim::fuse_slices (collectives.hpp:78, collectives.cpp:88-98). n == 0 ->
 * INVALID_ARGUMENT ("fuse_slices: empty slice list"). blob gets sum(lens). */
moe_status_t moesim_fuse_slices(uint64_t n, const uint64_t* lens, const uint8_t* data,
                                uint8_t* blob, moe_slice_index_entry_t* index);

/* moesim::split_blob (collectives.hpp:79, collectives.cpp:100-118): validates
 * contiguity + coverage (INVALID_ARGUMENT otherwise), writes the slices back to
 * back into out (sum of lengths == blob_len bytes). */
moe_status_t moesim_split_blob(uint64_t blob_len, const uint8_t* blob, uint64_t n,
                               const moe_slice_index_entry_t* index, uint8_t* out);

/* moesim::gen_trace (workload.hpp:41-42, workload.cpp:19-53): counts is
 * uint64 [steps][ranks][experts]. experts == 0 or skew < 0 -> CONFIG. */
moe_status_t moesim_gen_trace(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                              uint64_t tokens_per_rank, double skew, uint64_t* counts);

/* moesim::imbalance_ratio (workload.hpp:46, workload.cpp:55-66); zero tokens
 * -> CONFIG ("imbalance_ratio: trace carries zero tokens"). */
moe_status_t moesim_imbalance_ratio(uint32_t steps, uint32_t ranks, uint32_t experts,
                                    const uint64_t* counts, double* out);

/* moesim::build_schedule (ring_offload.hpp:45, ring_offload.cpp:31-50).
 * ops: int64 [n][4] = (kind 0=load 1=compute 2=release, layer, slot,
 * waits_release_of or -1); capacity must be >= 3*layers + min(slots, layers).
 * ring_slots == 0 or layers == 0 -> CONFIG. */
moe_status_t moesim_ring_build_schedule(uint32_t layers, uint32_t ring_slots, int64_t* ops,
                                        uint64_t capacity, uint64_t* n_ops, uint32_t* slots,
                                        int* clamped);

/* ======================================================================
 * 2. device data-plane ops (device pointers, caller's stream)
 * ====================================================================== */

/* Fill out[i] = lo + (hi-lo) * u_i with u_i the i-th SplitMix64(seed) draw
 * (rng.hpp:23-32), rounded to dtype.  Bit-identical to the sequential stream. */
moe_status_t moe_fill_uniform(void* out, uint64_t n, moe_dtype_t dtype, uint64_t seed, double lo,
                              double hi, void* stream);

/* Device gen_trace: counts (uint64, zeroed by the call) [steps][ranks][experts]. */
moe_status_t moe_gen_trace_device(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                                  uint64_t tokens_per_rank, double skew, uint64_t* counts,
                                  void* stream);

/* Single-device R x R ragged transpose (alltoall_flat with the ranks emulated
 * on one GPU): chunk (s,d) of length lens[s*R+d] at in + in_off[s*R+d] goes to
 * out + out_off[d*R+s].  Offsets/lengths are device arrays. */
moe_status_t moe_alltoall_flat_device(uint64_t ranks, const uint64_t* lens, const uint64_t* in_off,
                                      const uint8_t* in, const uint64_t* out_off, uint8_t* out,
                                      void* stream);

/* Fusion packing on the device: n slices (device pointer table) -> one blob;
 * index (device, n entries) = (i, exclusive prefix of lens, lens). */
moe_status_t moe_fuse_slices_device(uint64_t n, const uint8_t* const* slices, const uint64_t* lens,
                                    uint8_t* blob, moe_slice_index_entry_t* index, void* stream);
/* Inverse: validates the index on the device (status word *bad = 1 on a
 * non-contiguous or non-covering index) and scatters the slices out. */
moe_status_t moe_split_blob_device(uint64_t blob_len, const uint8_t* blob, uint64_t n,
                                   const moe_slice_index_entry_t* index, uint8_t* const* out,
                                   int32_t* bad, void* stream);

/* Routing (DESIGN.md Appendix A; K2): fp32 logits [T,E] ->
 * expert/gate/position/keep [T,k], count1/count2/kept [E], aux (1 float).
 * Bit-exact integers vs the oracle given identical logits. */
typedef struct moe_routing_out {
  int32_t* expert;   /* [T,k] */
  float* gate;       /* [T,k] */
  int32_t* position; /* [T,k] */
  uint8_t* keep;     /* [T,k] */
  int32_t* count1;   /* [E] pre-drop top-1 counts */
  int32_t* count2;   /* [E] pre-drop top-2 counts */
  int32_t* kept;     /* [E] min(count1+count2, C) */
  float* aux_loss;   /* [1] */
} moe_routing_out_t;

moe_status_t moe_route(uint64_t tokens, uint32_t experts, uint32_t top_k, uint64_t capacity,
                       const float* logits, const moe_routing_out_t* out, void* stream);

/* Grouped GEMM (K5) exposed for tests and callers with their own layouts.
 * bf16 inputs on tcgen05 (sm_100a), fp32 inputs on the SIMT FP32 path.
 *   kind RAGGED_M : for group g, rows m < m[g]:
 *       C[c_row[g]+m, n] = epi( sum_k A[a_row[g]+m, k] * B_{b[g]}(n, k) )
 *     A row-major [*, K]; B_b = w + b*N*K, K-major ([N][K]) or MN-major ([K][N]).
 *   kind RAGGED_K : for output o (= b[g]), C_o[m, n] += sum over groups g with
 *     b[g] == o of sum_{r < m[g]} A[a_row[g]+r, m] * B[a_row[g]+r, n]
 *     (A row-major [*, M], B row-major [*, N]; rows past m[g] up to the next
 *     multiple of 64 must be zero).  Groups of one output must be contiguous.
 * Group tables are device int32 arrays of length `groups`. */
typedef enum moe_gemm_kind { MOE_GEMM_RAGGED_M = 0, MOE_GEMM_RAGGED_K = 1 } moe_gemm_kind_t;
typedef enum moe_gemm_epilogue {
  MOE_EPI_STORE = 0,      /* C = acc (+bias) in dtype_c                                */
  MOE_EPI_GELU = 1,       /* h = acc+bias: C = gelu(h), C2 = gelu'(h) (erf GeLU)        */
  MOE_EPI_DGELU = 2,      /* C = acc * AUX[row, n] (AUX = the gelu'(h) C2 stored);
                             colsum (optional) += column sums of the stored C           */
  MOE_EPI_ATOMIC_ADD = 3, /* fp32 C += acc (split-K); transpose_c allowed               */
  MOE_EPI_GATHER_ADD = 4  /* C[t] = acc + sum_i gather_src[gather_idx[t*k+i]] (idx -1
                             skipped): combine-backward folded into the gate dgrad GEMM  */
} moe_gemm_epilogue_t;

typedef struct moe_gemm_problem {
  moe_gemm_kind_t kind;
  moe_gemm_epilogue_t epilogue;
  moe_dtype_t dtype_ab;   /* BF16 (tcgen05) or F32 (SIMT) */
  moe_dtype_t dtype_c;    /* output dtype (F32 required for ATOMIC_ADD) */
  int b_mn_major;         /* RAGGED_M: B stored [K][N] instead of [N][K] */
  int transpose_c;        /* store C^T (C[n*ldc + m]) */
  uint32_t groups;
  uint32_t M, N, K;       /* RAGGED_M: N, K (M ragged). RAGGED_K: M, N (K ragged) */
  uint64_t a_rows;        /* rows allocated in A (and B for RAGGED_K) */
  uint32_t num_b;         /* number of B matrices (RAGGED_M) / outputs (RAGGED_K) */
  const int32_t* m;       /* [groups] */
  const int32_t* a_row;   /* [groups] */
  const int32_t* c_row;   /* [groups] RAGGED_M only */
  const int32_t* b;       /* [groups] */
  const void* A;
  const void* B;
  void* C;
  void* C2;               /* GELU pre-activation output (same layout as C) */
  const void* aux;        /* DGELU: pre-activation, same layout/dtype as C */
  const float* bias;      /* [num_b][N] or NULL */
  uint64_t ldc;           /* elements; RAGGED_K outputs are [num_b][M][ldc] */
  uint64_t lda;           /* A row stride in elements (0: K for RAGGED_M, M for RAGGED_K) */
  uint64_t ldb;           /* B row stride in elements (0: natural) */
  uint64_t b_rows;        /* rows allocated in B (0: num_b * (N or K), RAGGED_K: a_rows) */
  uint64_t c_rows;        /* rows allocated in C (0: a_rows for RAGGED_M)                */
  float* colsum;          /* DGELU: [num_b][N] fp32 column sums of the stored C (written,
                             not accumulated; fixed summation order: bitwise reproducible),
                             or NULL                                                    */
  const void* gather_src; /* GATHER_ADD: [*, N] rows in dtype_c                          */
  const int32_t* gather_idx; /* GATHER_ADD: [rows][gather_k] row indices or -1          */
  uint32_t gather_k;
  float* colsum_ws;       /* DGELU with colsum: partials [groups][ceil(colsum_max_m/32)][N] */
  uint64_t colsum_max_m;  /* DGELU with colsum: upper bound of m[g] over the groups      */
  /* split-fp32 products on the bf16 tensor cores (fp32 STORE only): with
   * split_terms = 6, A and B each hold three stacked bf16 planes of an fp32
   * tensor (x = p0 + p1 + p2, moe_split_f32_bf16x3), plane j at row offset j x
   * (a_rows | b_rows, the single-plane row counts), and C = the sum of the six
   * leading plane products (error ~2^-22 relative per product). */
  uint32_t split_terms;   /* 0 or 1: plain; 6: split-fp32                                */
  uint32_t k_begin;       /* RAGGED_M: K sub-range [k_begin, k_begin + k_len) (multiples */
  uint32_t k_len;         /*   of 64; k_len 0 = to K) -- bounds accumulation chains      */
  const int32_t* k_begin_g; /* RAGGED_M, nullable: per-group K start (overrides k_begin;
                               with c_row, one launch computes every K chunk's partial) */
} moe_gemm_problem_t;

moe_status_t moe_grouped_gemm(const moe_gemm_problem_t* problem, void* stream);

/* fp32 -> three stacked bf16 planes (n elements each) with in = p0 + p1 + p2
 * exactly (the split_terms = 6 operand format); n % 4 == 0, in 16-byte aligned. */
moe_status_t moe_split_f32_bf16x3(const float* in, uint64_t n, void* out, void* stream);

/* ======================================================================
 * 3. the MoE layer (K1..K6 + EP exchange), forward and backward
 * ====================================================================== */

typedef struct moe_layer_desc {
  uint32_t num_experts;    /* E, global */
  uint32_t top_k;          /* 1 (Switch) or 2 (GShard) */
  uint32_t d_model;        /* d */
  uint32_t d_ff;           /* d_ff */
  double capacity_factor;  /* cf; C = ceil(k * cf * T / E) */
  uint64_t tokens;         /* T, tokens per rank per call */
  moe_dtype_t dtype;       /* BF16 (tcgen05 path) or F32 (SIMT FP32 path) */
  int has_gate_bias;
  uint32_t ep_size;        /* P ranks; E % P == 0 */
  uint32_t ep_rank;
  void* nccl_comm;         /* ncclComm_t when ep_size > 1 (see moe_comm_*) */
  uint32_t exchange;       /* ep_size > 1: MOE_EXCHANGE_P2P (default) or MOE_EXCHANGE_NCCL */
  uint32_t placement;      /* ep_size > 1: MOE_PLACEMENT_CONTIGUOUS (default) or _ROUND_ROBIN */
  uint32_t gate_grad_reduce; /* ep_size > 1: 0 = backward sums the replicated gate gradients
                                dwg/dbg over the EP group (default); 1 = left to the caller,
                                e.g. one fused moe_grad_buckets all-reduce for a layer stack */
} moe_layer_desc_t;

/* Expert placement over the ep_size ranks.  CONTIGUOUS: expert e lives on rank
 * e / (E/P) as local expert e % (E/P).  ROUND_ROBIN: on rank e % P as local
 * expert e / P, so a skewed (Zipf-like) routing distribution whose hot experts
 * have neighbouring ids is spread over all ranks instead of landing on rank 0.
 * Routing semantics (positions, capacity, outputs) do not depend on it; the
 * caller passes the weights of this rank's local experts in local order. */
#define MOE_PLACEMENT_CONTIGUOUS 0
#define MOE_PLACEMENT_ROUND_ROBIN 1

/* EP token exchange.  P2P: the dispatch / combine-backward kernels store rows
 * straight into the peers' receive buffers over NVLink (CUDA IPC mappings,
 * exact row counts, no capacity padding on the wire) and expert outputs are
 * pushed back the same way; device-side epoch flags order producers and
 * consumers (no host synchronisation).  NCCL: capacity-padded ncclAlltoAll of
 * the packed buffers (the baseline lowering). */
#define MOE_EXCHANGE_P2P 0
#define MOE_EXCHANGE_NCCL 1

typedef struct moe_layer* moe_layer_t;

/* Parameters (device, caller-owned).  wg [E][d], bg [E] (fp32, optional);
 * this rank's local experts (E/P of them): w1 [E/P][d_ff][d], b1 [E/P][d_ff]
 * (fp32), w2 [E/P][d][d_ff], b2 [E/P][d] (fp32).  wg/w1/w2 in the layer dtype. */
typedef struct moe_layer_params {
  const void* wg;
  const float* bg;
  const void* w1;
  const float* b1;
  const void* w2;
  const float* b2;
} moe_layer_params_t;

/* Gradients (device, fp32, overwritten): shapes as the parameters. */
typedef struct moe_layer_grads {
  float* dwg;
  float* dbg;
  float* dw1;
  float* db1;
  float* dw2;
  float* db2;
} moe_layer_grads_t;

moe_status_t moe_layer_create(const moe_layer_desc_t* desc, moe_layer_t* out);
moe_status_t moe_layer_destroy(moe_layer_t layer);
/* C = ceil(k * cf * T / E) for this layer. */
uint64_t moe_layer_capacity(moe_layer_t layer);

/* y [T,d] = MoE(x [T,d]).  When logits_override != NULL routing uses those
 * fp32 logits [T,E] instead of x wg^T + bg (parity tests). `routing` (optional)
 * receives device copies of the routing outputs.  Saves what backward needs. */
moe_status_t moe_layer_forward(moe_layer_t layer, const moe_layer_params_t* params, const void* x,
                               void* y, const float* logits_override, float* logits_out,
                               const moe_routing_out_t* routing, void* stream);

/* Backward of the last forward: dy [T,d] and d_aux (upstream gradient of the
 * aux loss) -> dx [T,d] and parameter gradients.  With ep_size > 1 dwg/dbg are
 * summed over the EP group (the gate is replicated). */
moe_status_t moe_layer_backward(moe_layer_t layer, const moe_layer_params_t* params, const void* dy,
                                float d_aux, void* dx, const moe_layer_grads_t* grads,
                                void* stream);

/* One training step of the layer from HOST buffers (the end-to-end API):
 * H2D x_host, dy_host (pinned) -> forward + backward -> D2H y_host, dx_host.
 * Parameter gradients stay on the device in `grads`.  Runs on the layer's own
 * copy-in / compute / copy-out streams over double-buffered staging so that
 * consecutive calls overlap H2D, compute and D2H; `stream` is made to wait for
 * this step's D2H, i.e. outputs, gradients and the reuse of the host buffers
 * are safe once `stream` reaches this call; the step's compute waits for all
 * work queued on `stream` before the call (e.g. an optimizer step that updates
 * params from the previous step's grads).  Do not interleave with
 * moe_layer_forward/backward on the same layer without synchronising. */
moe_status_t moe_layer_train_step_host(moe_layer_t layer, const moe_layer_params_t* params,
                                       const void* x_host, const void* dy_host, float d_aux,
                                       void* y_host, void* dx_host, const moe_layer_grads_t* grads,
                                       void* stream);

/* The same step with deferred outputs (the pipelined training loop): when
 * `stream` reaches this call the gradients are final and params may be
 * updated on `stream`, the host input buffers may be reused, and y_host /
 * dx_host of the PREVIOUS call are complete; this call's y_host / dx_host are
 * complete once `stream` reaches the next call or moe_layer_host_sync.  Lets
 * the copy-out of step i overlap the compute of step i+1 although the caller
 * queues work (an optimizer step) on `stream` between calls. */
moe_status_t moe_layer_train_step_host_async(moe_layer_t layer, const moe_layer_params_t* params,
                                             const void* x_host, const void* dy_host, float d_aux,
                                             void* y_host, void* dx_host,
                                             const moe_layer_grads_t* grads, void* stream);
/* Make `stream` wait for every outstanding copy-out of train_step_host_async. */
moe_status_t moe_layer_host_sync(moe_layer_t layer, void* stream);

/* Per-phase device timings (ms) of the last forward/backward when profiling is
 * enabled with moe_layer_set_profiling(layer, 1): names/values as parallel
 * arrays; returns the count (<= capacity).  Synchronises the layer's events. */
moe_status_t moe_layer_set_profiling(moe_layer_t layer, int enabled);
moe_status_t moe_layer_phase_times(moe_layer_t layer, const char** names, float* ms,
                                   uint32_t capacity, uint32_t* count);
/* The same for the last forward (backward = 0) or the last backward (1): the
 * two are recorded into separate events, so both can be read after one
 * forward + backward without a synchronisation in between. */
moe_status_t moe_layer_phase_times_of(moe_layer_t layer, int backward, const char** names,
                                      float* ms, uint32_t capacity, uint32_t* count);

/* Peer-wait limit of the NVLink exchange (default MOE_P2P_TIMEOUT_S or 600 s;
 * 0 = wait forever, like NCCL).  A peer that misses it does not kill the
 * context: the waits record an error code, later waits return at once, and
 * moe_layer_comm_status reports it (MOE_ERR_NCCL, "layer.exchange: peer p did
 * not signal slot s ...").  comm_status synchronises with the device. */
moe_status_t moe_layer_set_peer_timeout(moe_layer_t layer, double seconds);
moe_status_t moe_layer_comm_status(moe_layer_t layer, int32_t* code);

/* ----------------------------------------------------------------------
 * EP communicator (NCCL over NVLink): the unique id is exchanged by the host
 * (e.g. torch.distributed) as 128 opaque bytes.
 * ---------------------------------------------------------------------- */
moe_status_t moe_comm_unique_id(uint8_t id[128]);
moe_status_t moe_comm_create(const uint8_t id[128], uint32_t nranks, uint32_t rank, void** comm);
moe_status_t moe_comm_destroy(void* comm);

/* Packed EP all-to-all (Fusion communication, §4.2): send holds one
 * contiguous message of `bytes_per_peer` per destination rank in rank order;
 * recv receives one per source rank in rank order (SPEC.md:336 receive order).
 * fused = 0 issues `slices_per_peer` messages per peer instead (the unfused
 * lowering of lower_slice_transfer, collectives.cpp:250-267) for comparison. */
moe_status_t moe_alltoall_packed(void* comm, const void* send, void* recv, uint64_t bytes_per_peer,
                                 uint32_t slices_per_peer, int fused, void* stream);

/* Gradient-bucket fusion for replicated parameters (the gates of a stack of
 * MoE layers).  Replaces GradBucket / make_gradient_buckets
 * (collectives.hpp:80-109, collectives.cpp:120-162): the n parameter ids are
 * registered in REVERSE layer order into buckets of at most `capacity`; a
 * bucket flushes exactly once, when its last gradient is pushed, with its
 * payload in registration order.  On the device a flush packs the bucket's
 * fp32 gradients into one flat buffer, issues ONE ncclAllReduce(sum) over
 * `comm` and unpacks them multiplied by `scale` (e.g. 1/world for a mean) — on
 * the stream passed to push, no host synchronisation.  grads/numel may both be
 * NULL (bookkeeping only); comm may be NULL (one rank).  Errors:
 * INVALID_ARGUMENT for capacity 0, a duplicate push or an unknown id. */
typedef struct moe_grad_buckets* moe_grad_buckets_t;
moe_status_t moe_grad_buckets_create(void* comm, uint32_t n, const uint64_t* ids_layer_order,
                                     void* const* grads, const uint64_t* numel,
                                     uint32_t capacity, float scale, moe_grad_buckets_t* out);
moe_status_t moe_grad_buckets_destroy(moe_grad_buckets_t b);
/* *flushed = index of the bucket this push completed (its all-reduce is
 * enqueued on stream), or -1 while the bucket is still held. */
moe_status_t moe_grad_buckets_push(moe_grad_buckets_t b, uint64_t id, void* stream,
                                   int32_t* flushed);
moe_status_t moe_grad_buckets_reset(moe_grad_buckets_t b);
uint32_t moe_grad_buckets_count(moe_grad_buckets_t b);
/* ids of bucket i in registration order (capacity entries max); *n = count */
moe_status_t moe_grad_buckets_ids(moe_grad_buckets_t b, uint32_t i, uint64_t* ids,
                                  uint32_t capacity, uint32_t* n);

/* Algorithm-1 CPU cache policy for sparse (expert) parameter blocks, the
 * cache of SE-MoE's 2D prefetch.  Replaces SparseCache /
 * CachePolicyParams (prefetch_cache.hpp:18-83) with identical decisions:
 * resident -> CACHE_HIT (count += 1); occupancy + 1 < cpu_size -> FETCHED_FRESH
 * (count 1); coldest count >= threshold (ties: lowest id) -> EVICTED_AND_FETCHED
 * (victim reported); else STREAM_THROUGH.  Every decay_steps end_step() calls
 * multiply all counts by beta.  Errors: CONFIG for beta outside (0, 1],
 * decay_steps < 1, threshold < 0 ("cache.<field>: <reason>"). */
typedef struct moe_cache_params {
  uint64_t cpu_size;     /* cacheable blocks */
  double threshold;      /* minimum hit count an eviction victim must reach */
  double beta;           /* decay factor in (0, 1] */
  uint32_t decay_steps;  /* steps per decay cycle, >= 1 */
} moe_cache_params_t;
typedef enum moe_cache_kind {
  MOE_CACHE_HIT = 0,
  MOE_CACHE_FETCHED_FRESH = 1,
  MOE_CACHE_EVICTED_AND_FETCHED = 2,
  MOE_CACHE_STREAM_THROUGH = 3
} moe_cache_kind_t;
typedef struct moe_cache_access {
  int32_t kind;     /* moe_cache_kind_t */
  uint64_t victim;  /* EVICTED_AND_FETCHED only */
} moe_cache_access_t;
typedef struct moe_sparse_cache* moe_sparse_cache_t;
moe_status_t moe_sparse_cache_create(const moe_cache_params_t* params, moe_sparse_cache_t* out);
moe_status_t moe_sparse_cache_destroy(moe_sparse_cache_t cache);
moe_status_t moe_sparse_cache_access(moe_sparse_cache_t cache, uint64_t block,
                                     moe_cache_access_t* out);
moe_status_t moe_sparse_cache_end_step(moe_sparse_cache_t cache);
/* occupancy (fresh admissions), steps into the current decay cycle, and the
 * resident blocks with their counts sorted by id (capacity entries max) */
moe_status_t moe_sparse_cache_state(moe_sparse_cache_t cache, uint64_t* occupancy, uint32_t* steps,
                                    uint64_t* blocks, double* hits, uint64_t capacity,
                                    uint64_t* resident);

/* 2D prefetch executed on the GPU box (the reference
 * simulates it in run_2d_schedule, prefetch_cache.hpp:85-130): a stack of
 * num_layers MoE layers whose expert sections live in three tiers — a
 * backing-store file (the SSD tier, written from host_sections at create),
 * pinned CPU blocks managed by the Algorithm-1 cache, and lookahead + 1 HBM
 * slots.  For every (step, layer) the cache decides the backing-store I/O, the
 * section's H2D is issued when compute(t - lookahead) starts, and compute(t)
 * (layer forward + residual, gate weights resident) waits for it. */
typedef struct moe_prefetch_desc {
  uint32_t num_layers;
  uint32_t lookahead;                 /* layers of prefetch depth, >= 1 */
  moe_cache_params_t cache;           /* cpu_size in sections */
  uint32_t flush_period;              /* steps between CPU->store flushes; 0 = decay_steps */
  const void* const* host_sections;   /* [num_layers] section images (moe_ring_pack_section) */
  const void* const* gate_weights;    /* [num_layers] device pointers (wg) */
  const char* backing_path;           /* file for the backing store (created, removed at destroy) */
} moe_prefetch_desc_t;
typedef struct moe_prefetch_record {  /* one (step, layer) */
  uint32_t step, layer;
  int32_t kind;                       /* moe_cache_kind_t of the access */
  uint64_t victim;
  float io_ms;                        /* host time in backing-store reads / writes */
  float h2d_start, h2d_end;           /* ms from the run start (CUDA events) */
  float compute_start, compute_end;
} moe_prefetch_record_t;
typedef struct moe_prefetch_summary {
  float makespan_ms, compute_total_ms, stall_total_ms, io_total_ms;
  uint64_t bytes_read, bytes_written, h2d_bytes, section_bytes;
  uint32_t gpu_slots;
} moe_prefetch_summary_t;
typedef struct moe_prefetch* moe_prefetch_t;
moe_status_t moe_prefetch_create(moe_layer_t layer, const moe_prefetch_desc_t* desc,
                                 moe_prefetch_t* out);
moe_status_t moe_prefetch_destroy(moe_prefetch_t p);
/* `steps` passes over the stack from x (device) to y; records: steps*num_layers
 * entries or NULL.  Synchronises the stream (the timeline is read back). */
moe_status_t moe_prefetch_run(moe_prefetch_t p, uint32_t steps, const void* x, void* y,
                              moe_prefetch_record_t* records, moe_prefetch_summary_t* summary,
                              void* stream);

/* ======================================================================
 * 4. ring-of-sections inference (K7)
 * ====================================================================== */

/* N MoE layers whose expert weights live in pinned host memory rotate
 * through K HBM slots (ring_offload.hpp:16-64).  Layer i's experts (w1,b1,w2,b2
 * for all E experts of one rank, packed) are host_sections[i] of
 * section_bytes; dense parameters (the gates) stay resident. */
typedef struct moe_ring_desc {
  uint32_t num_layers;
  uint32_t ring_slots;
  const void* const* host_sections; /* [num_layers] pinned host pointers */
  const void* const* gate_weights;  /* [num_layers] device pointers (wg) */
  const float* const* gate_bias;    /* [num_layers] device pointers or NULL */
} moe_ring_desc_t;

typedef struct moe_ring* moe_ring_t;

typedef struct moe_ring_timeline {
  /* per layer, ms since the start event */
  float* load_start;
  float* load_end;
  float* compute_start;
  float* compute_end;
  float makespan_ms;
  float compute_total_ms;
  uint64_t peak_gpu_bytes;     /* dense + K * section */
  uint64_t baseline_gpu_bytes; /* dense + N * section */
  uint32_t slots;
  int clamped;
} moe_ring_timeline_t;

moe_status_t moe_ring_create(moe_layer_t layer, const moe_ring_desc_t* desc, moe_ring_t* out);
moe_status_t moe_ring_destroy(moe_ring_t ring);
uint64_t moe_ring_section_bytes(moe_layer_t layer);
/* Pack one layer's experts (device tensors) into a host section layout. */
moe_status_t moe_ring_pack_section(moe_layer_t layer, const void* w1, const float* b1,
                                   const void* w2, const float* b2, void* host_section);
/* Residual stack h_{i+1} = h_i + MoE_i(h_i) over the N layers, expert weights
 * streamed host -> HBM on a copy stream in the calculation-release-load order
 * of build_schedule.  Fills `timeline` (synchronises on completion). */
moe_status_t moe_ring_run(moe_ring_t ring, const void* x, void* y, moe_ring_timeline_t* timeline,
                          void* stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* MOE_B200_H_ */
