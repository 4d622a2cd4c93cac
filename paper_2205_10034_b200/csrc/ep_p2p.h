// Expert-parallel token exchange over NVLink peer memory (K4, P2P mode).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "moe_b200.h"

namespace moe {

// Flag slots in each rank's window: flags[slot][src] is written by rank src.
enum P2PSlot : int {
  SLOT_PHASE = 0,     // src finished phase n (its reads of our writes are done)
  SLOT_CNT = 1,       // src's kept counts for phase n are in our count matrix
  SLOT_DISPATCH = 2,  // src's token rows for phase n are in our recv_x
  SLOT_Y = 3,         // src pushed our expert outputs into our home Y
  SLOT_DY = 4,        // src's g*dy rows are in our recv_dy
  SLOT_DX = 5,        // src pushed our dX rows into our home dX
  SLOT_GRAD = 6,      // src's replicated-gradient partials are in our red[src]
  SLOT_BYE = 7,       // src has finished all work and will not write here again
  NSLOT = 8
};

// One cudaMalloc per rank holding everything peers write into; mapped into
// every peer with CUDA IPC.  Offsets are identical on all ranks.
//   recv_x / recv_dy : [El][Rmax][d], Rmax = P*Cs; the region of local expert
//                      j holds the rows of every source back to back in source
//                      order (source s at offset sum_{s'<s} cnt[s'][e]) so the
//                      expert GEMM sees ONE group per expert for any P
//   home_y / home_dx : [E][Cs][d], rows returned to their source positions
//   cnt              : [P][E] kept counts of every source (all-gathered)
//   red              : [P][n_red] fp32 partials of the replicated (gate)
//                      gradients, one row per source
struct P2PWindow {
  uint32_t P = 1, me = 0, E = 0, El = 0;
  uint64_t Cs = 0, Rmax = 0, row_bytes = 0, n_red = 0;
  uint8_t* base = nullptr;
  uint64_t bytes = 0;
  uint64_t off_xr = 0, off_dyr = 0, off_yh = 0, off_dxh = 0, off_cnt = 0, off_flags = 0,
           off_ctr = 0, off_red = 0;
  uint8_t* peer_host[8] = {};
  uint8_t** peer_dev = nullptr;
  int32_t* err = nullptr;
  uint64_t timeout_ns = 0;  // peer-wait limit, 0 = wait forever
};

void p2p_setup(P2PWindow& w, void* nccl_comm, uint32_t P, uint32_t me, uint32_t E, uint64_t Cs,
               uint64_t row_bytes, uint64_t n_red, cudaStream_t st);
void p2p_teardown(P2PWindow& w);
// Device error code of the peer waits (0 = ok, 1000 + 16*slot + peer = that
// peer timed out); synchronous read.
int32_t p2p_status(const P2PWindow& w);

// Wait until flags[slot][src] >= target for every src != me (device spin;
// after w.timeout_ns it records an error code and gives up instead of hanging).
void p2p_wait(const P2PWindow& w, int slot, uint64_t target, cudaStream_t st);
// Write `value` into every peer's flags[slot][me] (after all prior work on st).
void p2p_signal(const P2PWindow& w, int slot, uint64_t value, cudaStream_t st);

// All-gather of the kept counts: kept[E] -> every rank's cnt[me][:]; SLOT_CNT.
void p2p_counts(const P2PWindow& w, const int32_t* kept, uint64_t epoch, cudaStream_t st);

// K3 fused with K4: rows x[t] go straight into the owning rank's recv_x at
// [j][off(me, e) + pos]; then SLOT_DISPATCH := epoch at every peer.
void p2p_dispatch(const P2PWindow& w, uint64_t T, uint32_t d, uint32_t k, uint64_t C,
                  moe_dtype_t dt, const void* x, const int32_t* expert, const int32_t* position,
                  int32_t* slot, uint64_t epoch, cudaStream_t st);

// Receiver side: group tables for the El local experts (one group each, m =
// sum over sources) and zeroing of rows [m, round_up(m, 64)) of `buf`
// (recv_x or recv_dy) so the weight-gradient GEMM can run whole K blocks.
void p2p_local_groups(const P2PWindow& w, int32_t* gm, int32_t* ga, int32_t* gb, void* buf,
                      cudaStream_t st);

// K6^T fused with K4: dgate from the local home Y; g*dy rows straight into the
// owning rank's recv_dy at the dispatch positions; SLOT_DY := epoch.
void p2p_combine_bwd(const P2PWindow& w, uint64_t T, uint32_t d, uint32_t k, moe_dtype_t dt,
                     const void* dy, const int32_t* slot, const float* gate,
                     const int32_t* expert, const int32_t* position, float* dgate, uint64_t epoch,
                     cudaStream_t st);

// Return expert outputs: rows of source s in local expert region j of `src`
// ([El][Rmax] row space) go to rank s's home buffer (window offset home_off) at
// [(me*El + j)*Cs + r]; then `slot` := epoch at every peer.
void p2p_push_home(const P2PWindow& w, uint64_t home_off, const void* src, int slot,
                   uint64_t epoch, cudaStream_t st);

// Sum-all-reduce of replicated fp32 gradients (a[0:na] ++ b[0:nb], na % 4 ==
// 0, na + nb <= n_red) over peer memory: every rank stores its partial into
// red[me] of every window (SLOT_GRAD := epoch), then sums red[0..P-1] in rank
// order, so all replicas end bitwise identical.  Replaces ncclAllReduce for
// the small gate gradients (latency, not bandwidth, bound).
// The same in two halves: push this rank's partials (as soon as they are
// final), finish = wait for every peer's push and sum in source order.
void p2p_allreduce_push(const P2PWindow& w, const float* a, uint64_t na, const float* b,
                        uint64_t nb, uint64_t epoch, cudaStream_t st);
void p2p_allreduce_finish(const P2PWindow& w, float* a, uint64_t na, float* b, uint64_t nb,
                          uint64_t epoch, cudaStream_t st);
void p2p_allreduce_f32(const P2PWindow& w, float* a, uint64_t na, float* b, uint64_t nb,
                       uint64_t epoch, cudaStream_t st);

}  // namespace moe
