// Expert-parallel token exchange over NVLink peer memory (K4, P2P mode).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "moe_b200.h"

namespace moe {

// Flag slots in each rank's window: flags[slot][src] is written by rank src.
enum P2PSlot : int { SLOT_PHASE = 0, SLOT_DISPATCH = 1, SLOT_Y = 2, SLOT_DY = 3, SLOT_DX = 4,
                     NSLOT = 5 };

// One cudaMalloc per rank holding everything peers write into; mapped into
// every peer with CUDA IPC.  Offsets are identical on all ranks.
struct P2PWindow {
  uint32_t P = 1, me = 0;
  uint8_t* base = nullptr;          // local window
  uint64_t bytes = 0;
  uint64_t off_xr = 0, off_dyr = 0, off_yh = 0, off_dxh = 0, off_cnt = 0, off_flags = 0,
           off_ctr = 0;
  uint8_t* peer_host[8] = {};       // host copy of the peer base pointers
  uint8_t** peer_dev = nullptr;     // device array [P] of peer base pointers
  int32_t* err = nullptr;           // device error word (timeouts)
};

void p2p_setup(P2PWindow& w, void* nccl_comm, uint32_t P, uint32_t me, uint64_t slice_bytes,
               uint64_t home_bytes, uint32_t E, cudaStream_t st);
void p2p_teardown(P2PWindow& w);

// Wait until flags[slot][src] >= target for every src != me (device spin with
// a timeout that traps instead of hanging the GPU).
void p2p_wait(const P2PWindow& w, int slot, uint64_t target, cudaStream_t st);
// Write `value` into every peer's flags[slot][me] (after all prior work on st).
void p2p_signal(const P2PWindow& w, int slot, uint64_t value, cudaStream_t st);

// K3 fused with K4: rows x[t] go straight to recv_x of the owning rank at
// [me][j][pos]; kept counts to cnt_recv[me][j]; pad rows [kept, round64)
// zeroed remotely; then SLOT_DISPATCH := epoch at every peer.
void p2p_dispatch(const P2PWindow& w, uint64_t T, uint32_t d, uint32_t E, uint32_t El,
                  uint32_t k, uint64_t C, uint64_t Cs, moe_dtype_t dt, const void* x,
                  const int32_t* expert, const int32_t* position, const int32_t* kept,
                  int32_t* slot, uint64_t epoch, cudaStream_t st);

// K6^T fused with K4: dgate from the local home Y; g*dy rows straight to the
// owning rank's recv_dy; pads zeroed remotely; SLOT_DY := epoch.
void p2p_combine_bwd(const P2PWindow& w, uint64_t T, uint32_t d, uint32_t E, uint32_t El,
                     uint32_t k, uint64_t C, uint64_t Cs, moe_dtype_t dt, const void* dy,
                     const int32_t* slot, const float* gate, const int32_t* expert,
                     const int32_t* position, const int32_t* kept, float* dgate, uint64_t epoch,
                     cudaStream_t st);

// Return expert outputs: rows [0, cnt[s][j]) of local slice (s, j) of `src`
// (recv row space) go to rank s's home buffer (window offset home_off) at
// [(me*El + j)*Cs]; then `slot` := epoch at every peer.
void p2p_push_home(const P2PWindow& w, uint64_t home_off, const void* src, uint32_t El,
                   uint64_t Cs, uint32_t d, uint64_t esz, int slot, uint64_t epoch,
                   cudaStream_t st);

}  // namespace moe
