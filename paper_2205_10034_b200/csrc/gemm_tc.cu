// K5 — grouped expert GEMM on 5th-generation tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel per shape class (384 threads; CTA
// pairs, cta_group::2, for the expert GEMMs -- 2-pair multicast clusters for
// the bf16 STORE ones):
//   warps 0..7   epilogue: warp w owns TMEM lanes 32*(w%4).. and half the columns;
//                tcgen05.ld -> bias / GeLU / GeLU' / gather-add -> bf16|fp32 ->
//                64B-swizzled smem staging -> TMA bulk tensor store (partial
//                row blocks fall back to masked stores); GeLU' operands arrive
//                by TMA one chunk ahead; optional fused column sums (bias grad).
//   warp 8       TMA producer (one lane): A/B tiles -> 128B-swizzled smem ring
//   warp 9       MMA issuer (pair leader): tcgen05.mma 256xBNx16, fp32 accum in TMEM
//   warp 10      TMEM allocator (2 x BN columns: double-buffered accumulator)
//   warp 11      group-table scan (tiles per group -> prefix sums in smem)
// Work items come from device-side group tables (no host sync on routing
// counts — the paper's CPU-side scheduling overhead):
//   RAGGED_M : group g = one (source, expert) slice of m[g] rows; tiles =
//              ceil(m/128) x ceil(N/BN); B = the expert's weight (K- or MN-major)
//   RAGGED_K : weight gradients; a segment = consecutive groups of one output,
//              K runs over the groups' rows (zero-padded to 64), A/B MN-major.
// The reference has no expert compute at all (cost model only:
// prefetch_cache.cpp:86-95, ring_offload.hpp:21); DESIGN.md §K5.
#include <cuda.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace moe {

namespace tc {

#ifndef MOE_COOP_GATHER
#define MOE_COOP_GATHER 1
#endif
constexpr int BM = 128;
constexpr int BK = 64;
constexpr int THREADS = 384;
constexpr int EPI_WARPS = 8;
constexpr int MAX_GROUPS = 1024;
constexpr int STG = 2048;  // one 32-row x 64B staging tile

// CG = CTAs per MMA (cta_group): CG == 2 pairs two SMs on a 256 x BN tile,
// each CTA holding its 128 A rows and BN/2 B columns (halves the per-SM smem
// operand traffic of the 128 x 256 single-CTA MMA).
template <int BN, int EPI, bool CF32, int CG, int KIND = 0>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN;
  static constexpr int CW = CF32 ? 16 : 32;  // epilogue chunk width (columns): 64B per row
  static constexpr int NOUT = (EPI == MOE_EPI_GELU) ? 2 : 1;
  // DGELU: aux tile (TMA, double-buffered); GATHER_ADD: 2 gathered sources x 2 buffers
  // DGELU: aux tile (TMA, double-buffered); GATHER_ADD: 2 gathered sources x
  // the 4 chunks of a warp's tile (all prefetched when the tile starts)
  static constexpr int NAUX = (EPI == MOE_EPI_DGELU) ? 2 : (EPI == MOE_EPI_GATHER_ADD ? 8 : 0);
  // output staging buffers per warp: single-buffered (the TMA store of chunk
  // c must have read the buffer before chunk c+1 is staged) for the expert
  // GEMMs -- the freed shared memory buys operand stages, and these kernels
  // wait on operands (per-expert weights from DRAM), not on the epilogue:
  // weight gradients 5 -> 6 stages (A/B on c2: 0.50 -> 0.45 ms), GeLU /
  // GeLU' epilogues 4 -> 5 stages (round 2: c2 step -1.1%, c3 -0.9%, 3+3
  // interleaved runs); double-buffered only for the fp32-output ones
#ifndef MOE_WGRAD_NBUF
#define MOE_WGRAD_NBUF 1
#endif
#ifndef MOE_GELU_NBUF
#define MOE_GELU_NBUF 1
#endif
#ifndef MOE_DGELU_NBUF
#define MOE_DGELU_NBUF 1
#endif
  static constexpr int NBUF = KIND == 1 && EPI == MOE_EPI_STORE ? MOE_WGRAD_NBUF
                              : EPI == MOE_EPI_GELU ? MOE_GELU_NBUF
                              : EPI == MOE_EPI_DGELU ? MOE_DGELU_NBUF
                              : CF32 ? 2 : 1;
  // + the warp's bias slice of the current tile (STORE/GELU): BN/2 floats
  static constexpr int BIAS_BYTES =
      KIND == 0 && (EPI == MOE_EPI_STORE || EPI == MOE_EPI_GELU) ? BN * 2 : 0;
  // staging tiles stay 2 KB aligned (the TMA swizzle follows address bits)
  static constexpr int WARP_EPI_BYTES = (NBUF * NOUT + NAUX) * STG;
  // as many operand stages as fit next to the epilogue buffers (<= 8)
  static constexpr int FIT =
      (232448 - 6 * 1024 - EPI_WARPS * (WARP_EPI_BYTES + BIAS_BYTES) - (MAX_GROUPS + 1) * 4) /
      STAGE_BYTES;
  static constexpr int STAGES = FIT > 8 ? 8 : FIT;
  static_assert(STAGES >= (EPI == MOE_EPI_GATHER_ADD ? 2 : 3), "pipeline depth");
  static constexpr int EPI_OFF = STAGES * STAGE_BYTES;
  static constexpr int BIAS_OFF = EPI_OFF + EPI_WARPS * WARP_EPI_BYTES;
  static constexpr int BAR_OFF = BIAS_OFF + EPI_WARPS * BIAS_BYTES;
  static constexpr int BAR_BYTES = (2 * STAGES + 4 + 2 * EPI_WARPS) * 8;
  static constexpr int HOLD_OFF = BAR_OFF + BAR_BYTES;
  static constexpr int TAB_OFF = ((HOLD_OFF + 16 + 15) / 16) * 16;
  static constexpr int SMEM = TAB_OFF + (MAX_GROUPS + 1) * 4 + 1024;  // + alignment slack
  static_assert(SMEM <= 232448, "smem budget");
};

struct Args {
  int groups;
  int M, N, K;
  const int* gm;
  const int* ga;
  const int* gc;
  const int* gb;
  void* C;
  void* C2;
  const float* bias;
  float* colsum;  // DGELU: per-warp partials [groups][cs_maxch][N] (reduced by seg_colsum)
  int cs_maxch;
  const void* gsrc;
  const int* gidx;
  int gk;
  long long ldc;
  int transpose_c;
  int num_b;
  int c_direct;  // C rows not 16-byte aligned (e.g. N = E = 2): no TMA stores, scalar stores
  // split-fp32 mode (terms == 6): A and B are three stacked bf16 planes each
  // (x = p0 + p1 + p2), a_plane / b_plane rows apart; the K loop runs the six
  // leading plane products, the main one (p0 q0) last; K range [k_begin,
  // k_begin + k_len) (RAGGED_M) so the caller can bound the accumulation chains
  int terms;
  long long a_plane, b_plane;
  int k_begin, k_len;
  const int* gkb;  // RAGGED_M: per-group K start (nullable: k_begin for all)
};

// plane pairs of the split-fp32 products, smallest first: the tensor core's
// fp32 accumulation truncates (tc_accum_probe.py: -168 ulp mean at K = 4096),
// so the large p0 q0 chain goes last onto an accumulator still small
__constant__ int kSplitA[6] = {2, 1, 0, 1, 0, 0};
__constant__ int kSplitB[6] = {0, 1, 2, 0, 1, 0};

// Per-peer destinations of the remote-store epilogue (RemoteRows on device).
struct RemoteOut {
  CUtensorMap maps[8];  // [P] bf16 [E*Cs][N] views of each peer's destination buffer
  uint8_t** peers;
  unsigned long long home_off;
  const int* cnt;
  int P, me, E, El;
  long long Cs;
};

// Exclusive scan of vals[0..n) (smem) into out[0..n] by one warp.
__device__ void warp_scan_smem(const int* vals, int n, int* out) {
  const int lane = threadIdx.x & 31;
  const int chunk = (n + 31) / 32;
  const int lo = min(n, lane * chunk), hi = min(n, lo + chunk);
  int s = 0;
  for (int i = lo; i < hi; ++i) s += vals[i];
  int incl = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int run = incl - s;
  for (int i = lo; i < hi; ++i) {
    const int v = vals[i];
    out[i] = run;
    run += v;
  }
  if (lane == 31) out[n] = incl;
}

// write 32 values (bf16: 32 cols = 4 x 16B) or 16 (fp32: 16 cols = 4 x 16B)
// of row r into a 64B-row SWIZZLE_64B staging tile
template <bool CF32>
__device__ __forceinline__ void stage_row(uint8_t* stg, uint32_t r, const float* f) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 o;
    if (CF32) {
      o = make_uint4(__float_as_uint(f[j * 4 + 0]), __float_as_uint(f[j * 4 + 1]),
                     __float_as_uint(f[j * 4 + 2]), __float_as_uint(f[j * 4 + 3]));
    } else {
      o.x = pack_bf16x2(f[j * 8 + 0], f[j * 8 + 1]);
      o.y = pack_bf16x2(f[j * 8 + 2], f[j * 8 + 3]);
      o.z = pack_bf16x2(f[j * 8 + 4], f[j * 8 + 5]);
      o.w = pack_bf16x2(f[j * 8 + 6], f[j * 8 + 7]);
    }
    *reinterpret_cast<uint4*>(stg + sw64(r, j)) = o;
  }
}

// masked direct store of one row's chunk (partial tiles)
template <bool CF32>
__device__ __forceinline__ void store_row_direct(void* base, long long off, int ncols,
                                                 const float* f, bool vec_ok = true) {
  constexpr int CW = CF32 ? 16 : 32;
  if (CF32) {
    float* p = reinterpret_cast<float*>(base) + off;
    if (vec_ok && ncols >= CW) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(p + q * 4) =
            make_float4(f[q * 4], f[q * 4 + 1], f[q * 4 + 2], f[q * 4 + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < CW; ++i)
        if (i < ncols) p[i] = f[i];
    }
  } else {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(base) + off;
    if (vec_ok && ncols >= CW) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 o;
        o.x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
        o.y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
        o.z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
        o.w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
        *reinterpret_cast<uint4*>(p + q * 8) = o;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CW; ++i)
        if (i < ncols) p[i] = f2bf(f[i]);
    }
  }
}

template <int BN, bool A_MN, bool B_MN, int KIND, int EPI, bool CF32, int CG, bool REMOTE>
__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                   const __grid_constant__ CUtensorMap tmAux,
                   const __grid_constant__ CUtensorMap tmAh, const Args args,
                   const __grid_constant__ RemoteOut ro) {
  using C_ = Cfg<BN, EPI, CF32, CG, KIND>;
  constexpr int TM = BM * CG;  // tile rows per work item (the CTA pair)
  // Pair mode (cluster of 2): one CTA pair per cluster.  Multicast mode
  // (cluster of 4, launched with a preferred cluster size of 4 where the
  // tile grid allows): two pairs per cluster work on the two column blocks
  // of one row block (consecutive work items), and each CTA loads half of
  // the A rows it shares with its counterpart in the other pair and
  // multicasts them to both -- a quarter less operand traffic through the
  // L2, which bounds these GEMMs.  Clusters the GPU could only place as
  // pairs run pair mode.
  const uint32_t crank_c = CG == 2 ? cluster_ctarank() : 0;
  const bool mc = CG == 2 && cluster_nctarank() == 4;
  const uint32_t crank = crank_c & 1;      // rank inside the pair (0 = leader)
  const uint32_t lead = crank_c & ~1u;     // the pair leader's cluster rank
  const uint32_t ahalf = crank_c >> 1;     // multicast mode: the A half this CTA loads
  const uint16_t pmask = (uint16_t)(3u << lead);
  const uint16_t amask = (uint16_t)((1u << crank_c) | (1u << (crank_c ^ 2u)));
  const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nunits = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  constexpr int CW = C_::CW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C_::BAR_OFF);
  uint64_t* empty = full + C_::STAGES;
  uint64_t* tfull = empty + C_::STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* abar = tempty + 2;  // [EPI_WARPS][2] aux-tile arrival barriers
  uint32_t* tmem_hold = reinterpret_cast<uint32_t*>(smem + C_::HOLD_OFF);
  int* tab = reinterpret_cast<int*>(smem + C_::TAB_OFF);  // [MAX_GROUPS+1]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = args.groups;
  const int nblk_n = (args.N + BN - 1) / BN;

  // ---- setup ---------------------------------------------------------
  // Warp roles: 0-7 epilogue, 8 TMA producer, 9 MMA issuer, 10 TMEM
  // allocator, 11 group-table scan.  The issue arbiter favours the highest
  // warp id on an SM sub-partition, so the producer and the MMA issuer (which
  // share sub-partitions 0/1 with epilogue warps) win issue slots over the
  // epilogue math instead of starving the tensor pipe.
  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 9 && lane == 0) {
    for (int s = 0; s < C_::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], mc ? 2 : 1);  // multicast: both pairs' MMAs read the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS * CG);  // leader's counts both CTAs' epilogues
    }
    for (int a = 0; a < 2 * EPI_WARPS; ++a) mbar_init(&abar[a], 1);
    fence_mbar_init();
  }
  if (warp == 10) {
    if (CG == 2) tmem_alloc_2sm(tmem_hold, C_::TMEM_COLS);
    else tmem_alloc(tmem_hold, C_::TMEM_COLS);
    tc_fence_before();
  }
  // everything above touched only this CTA's shared memory / TMEM: wait for
  // the previous kernel here (PDL), then let the next one start launching
  pdl_wait();
  pdl_trigger();
  int* scratch = reinterpret_cast<int*>(smem);  // stage 0 is free during setup
  if (KIND == 0) {
    for (int g = threadIdx.x; g < G; g += THREADS) {
      const int m = args.gm[g];
      scratch[g] = ((m + TM - 1) / TM) * nblk_n;
    }
  } else {
    for (int g = threadIdx.x; g < G; g += THREADS) {
      const bool start = (EPI == MOE_EPI_ATOMIC_ADD) || g == 0 || args.gb[g] != args.gb[g - 1];
      scratch[g] = start ? 1 : 0;
    }
  }
  __syncthreads();
  if (warp == 11) {
    if (KIND == 0) {
      warp_scan_smem(scratch, G, tab);
    } else {
      int* pos = scratch + MAX_GROUPS + 1;
      warp_scan_smem(scratch, G, pos);
      __syncwarp();
      for (int g = lane; g < G; g += 32)
        if (scratch[g]) tab[pos[g]] = g;
      if (lane == 0) tab[pos[G]] = G;
      if (lane == 0) tab[MAX_GROUPS] = pos[G];
    }
  }
  __syncthreads();
  if (CG == 2) cluster_sync_all();  // peer barriers initialised before any TMA signals them
  if (mc && (unit & 1) != (int)ahalf) __trap();  // clusters are aligned blockIdx quads
  tc_fence_after();
  const uint32_t tmem_base = *tmem_hold;

  int total_work;
  const int mt = args.M / TM;  // RAGGED_K only
  if (KIND == 0) total_work = tab[G];
  else total_work = tab[MAX_GROUPS] * mt * nblk_n;

  auto decode = [&](int w, int& g, int& mb, int& nb) {
    if (KIND == 0) {
      int lo = 0, hi = G;  // last g with tab[g] <= w (skips empty groups)
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (tab[mid] <= w) lo = mid; else hi = mid;
      }
      g = lo;
      const int local = w - tab[g];
      mb = local / nblk_n;
      nb = local % nblk_n;
    } else {
      const int per = mt * nblk_n;
      g = w / per;  // segment index
      const int local = w % per;
      mb = local / nblk_n;
      nb = local % nblk_n;
    }
  };
  auto num_kblocks = [&](int g) -> int {
    if (KIND == 0) return (args.k_len / BK) * args.terms;
    int n = 0;
    for (int q = tab[g]; q < tab[g + 1]; ++q) n += (args.gm[q] + BK - 1) / BK;
    return n * args.terms;
  };

  // Last block of a ragged group with <= 128 rows left: run it as an M = 128
  // pair tile (each CTA 64 rows; TMEM lanes 0-63 hold output columns [0, BN/2),
  // lanes 64-127 columns [BN/2, BN) — the 2-SM M=128 accumulator layout), which
  // halves the padding waste of 256-row tiles.
  auto is_tail = [&](int g, int mb) -> bool {
    if (CG != 2 || KIND != 0) return false;
    const int rem = args.gm[g] - mb * TM;
    return rem > 0 && rem <= BM;
  };
  constexpr uint32_t IDESC = umma_idesc_bf16(TM, BN, A_MN, B_MN);
  constexpr uint32_t IDESC_T = umma_idesc_bf16(CG == 2 ? 128 : TM, BN, A_MN, B_MN);
  constexpr int BH = BN / CG;  // B columns held by this CTA

  if (warp == 8) {
    // ================= TMA producer =================
    // CG == 2: this CTA loads its 128 A rows and BN/2 B columns; all bytes
    // complete on the LEADER's full barrier, which only the leader arms.
    if (lane == 0) {
      const uint32_t full0 = smem_u32(&full[0]);
      uint32_t it = 0;
      for (int w = unit; w < total_work; w += nunits) {
        int g, mb, nb;
        decode(w, g, mb, nb);
        auto load = [&](void* dst, const CUtensorMap* m, int s, int c0, int c1) {
          if (CG == 2)
            tma_load_2d_2sm(dst, m, mapa_shared(full0 + s * 8, lead), c0, c1);
          else
            tma_load_2d(dst, m, &full[s], c0, c1);
        };
        // multicast half of the shared A rows (both pairs' CTAs of this rank)
        auto load_mc = [&](void* dst, const CUtensorMap* m, int s, int c0, int c1) {
          tma_load_2d_2sm_mc(dst, m, mapa_shared(full0 + s * 8, lead), amask, c0, c1);
        };
        auto arm = [&](int s) {
          if (crank == 0) mbar_arrive_expect_tx(&full[s], C_::STAGE_BYTES * CG);
        };
        if (KIND == 0) {
          const bool tail = is_tail(g, mb);
          const int arow = args.ga[g] + mb * TM + (int)crank * (tail ? 64 : BM);
          const int brow = args.gb[g] * (B_MN ? args.K : args.N);
          const int bcol = nb * BN + (int)crank * BH;
          const int nk = args.k_len / BK, kb0 = (args.gkb ? args.gkb[g] : args.k_begin) / BK;
          const int nkb = nk * args.terms;
          for (int i = 0; i < nkb; ++i, ++it) {
            const int t = args.terms == 1 ? 0 : i / nk;
            const int kb = kb0 + (args.terms == 1 ? i : i % nk);
            const int pa = args.terms == 1 ? 0 : (int)(kSplitA[t] * args.a_plane);
            const int pb = args.terms == 1 ? 0 : (int)(kSplitB[t] * args.b_plane);
            const int s = it % C_::STAGES;
            mbar_wait(&empty[s], ((it / C_::STAGES) & 1) ^ 1);
            uint8_t* sA = smem + s * C_::STAGE_BYTES;
            uint8_t* sB = sA + C_::A_BYTES;
            arm(s);
            if (mc && !tail)  // this CTA's half: box {64, 64}, to both pairs
              load_mc(sA + ahalf * 8192, &tmAh, s, kb * BK, arow + pa + (int)ahalf * 64);
            else
              load(sA, &tmA, s, kb * BK, arow + pa);  // A K-major box {64,128}
            if (!B_MN) {
              load(sB, &tmB, s, kb * BK, brow + bcol + pb);
            } else {
#pragma unroll
              for (int j = 0; j < BH / 64; ++j)
                load(sB + j * 8192, &tmB, s, bcol + j * 64, brow + pb + kb * BK);
            }
          }
        } else {
          const int acol = mb * TM + (int)crank * BM;
          const int bcol = nb * BN + (int)crank * BH;
          for (int t = 0; t < args.terms; ++t) {
            const int pa = args.terms == 1 ? 0 : (int)(kSplitA[t] * args.a_plane);
            const int pb = args.terms == 1 ? 0 : (int)(kSplitB[t] * args.b_plane);
            for (int q = tab[g]; q < tab[g + 1]; ++q) {
              const int rows = args.gm[q];
              const int r0 = args.ga[q];
              for (int kb = 0; kb * BK < rows; ++kb, ++it) {
                const int s = it % C_::STAGES;
                mbar_wait(&empty[s], ((it / C_::STAGES) & 1) ^ 1);
                uint8_t* sA = smem + s * C_::STAGE_BYTES;
                uint8_t* sB = sA + C_::A_BYTES;
                arm(s);
                const int row = r0 + kb * BK;
                if (mc) {
                  load_mc(sA + ahalf * 8192, &tmA, s, acol + (int)ahalf * 64, row + pa);
                } else {
#pragma unroll
                  for (int j = 0; j < BM / 64; ++j)
                    load(sA + j * 8192, &tmA, s, acol + j * 64, row + pa);
                }
#pragma unroll
                for (int j = 0; j < BH / 64; ++j)
                  load(sB + j * 8192, &tmB, s, bcol + j * 64, row + pb);
              }
            }
          }
        }
      }
    }
  } else if (warp == 9) {
    // ================= MMA issuer (leader CTA only when paired) =================
    // Two issue loops, chosen per instantiation by measurement (A/B on one
    // B200): with a heavy epilogue (GeLU, GeLU', fp32 outputs) the whole warp
    // walks the loop in uniform control flow and one elected lane issues (the
    // descriptors stay in uniform registers, ~4x fewer instructions per K
    // block, which matters when the epilogue warps compete for issue slots);
    // with a light epilogue a single lane runs the loop (measured ~5% faster
    // for the K = 4096 GEMMs).  Per 64-wide K block: 4 MMAs whose descriptors
    // differ by a constant (+32 B K-major, +2 KiB MN-major start address).
    constexpr bool kWarpIssue = EPI == MOE_EPI_GELU || EPI == MOE_EPI_DGELU || CF32;
    constexpr uint64_t ADV_A = A_MN ? (2048 >> 4) : (32 >> 4);
    constexpr uint64_t ADV_B = B_MN ? (2048 >> 4) : (32 >> 4);
    if (crank == 0 && (kWarpIssue || lane == 0)) {
      uint32_t it = 0, tcount = 0;
      for (int w = unit; w < total_work; w += nunits, ++tcount) {
        int g, mb, nb;
        decode(w, g, mb, nb);
        const int nkb = num_kblocks(g);
        const uint32_t idesc = is_tail(g, mb) ? IDESC_T : IDESC;
        const uint32_t acc = tcount & 1;
        mbar_wait(&tempty[acc], ((tcount >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C_::STAGES;
          mbar_wait(&full[s], (it / C_::STAGES) & 1);
          tc_fence_after();
          const uint32_t aBase = smem_u32(smem + s * C_::STAGE_BYTES);
          const uint32_t bBase = aBase + C_::A_BYTES;
          const uint64_t da0 = A_MN ? umma_desc_sw128(aBase, 8192, 1024) : umma_desc_sw128(aBase, 16, 1024);
          const uint64_t db0 = B_MN ? umma_desc_sw128(bBase, 8192, 1024) : umma_desc_sw128(bBase, 16, 1024);
          if (!kWarpIssue || elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint32_t accum = (kb | kk) != 0 ? 1u : 0u;
              if (CG == 2) tc_mma_bf16_2sm(d_tmem, da0 + kk * ADV_A, db0 + kk * ADV_B, idesc, accum);
              else tc_mma_bf16(d_tmem, da0 + kk * ADV_A, db0 + kk * ADV_B, idesc, accum);
            }
            if (CG == 2) tc_commit_2sm_mc(&empty[s], mc ? (uint16_t)0xF : pmask);
            else tc_commit(&empty[s]);
          }
          if (kWarpIssue) __syncwarp();
        }
        if (!kWarpIssue || elect_one()) {
          if (CG == 2) tc_commit_2sm_mc(&tfull[acc], pmask);
          else tc_commit(&tfull[acc]);
        }
        if (kWarpIssue) __syncwarp();
      }
    }
  } else if (warp < EPI_WARPS) {
    // ================= epilogue (8 warps) =================
    const int ew = warp;
    const int q = warp & 3;           // TMEM lane quarter (hardware: warp % 4)
    const int half = ew >> 2;         // column half of the tile
    constexpr int HALF = BN / 2;
    // out[NBUF] [, out2[NBUF]] [, aux[2]]
    uint8_t* const stg_base = smem + C_::EPI_OFF + ew * C_::WARP_EPI_BYTES;
    uint8_t* const auxb = stg_base + C_::NBUF * C_::NOUT * STG;
    uint32_t nst = 0;  // bulk store groups committed by this warp (selects the buffer)
    uint64_t* ab = abar + 2 * ew;
    uint32_t aph[2] = {0, 0};
    uint32_t tcount = 0;
    const uint32_t tempty0 = smem_u32(&tempty[0]);
    // this warp's slice of tile w: first row, output row, valid rows, columns
    struct Geo {
      int g, mb, nb, row0, tcol, nch, nvalid, bidx, col_base;
      bool tail;
      long long orow0;
    };
    auto geo_of = [&](int w) {
      Geo t;
      decode(w, t.g, t.mb, t.nb);
      t.tail = is_tail(t.g, t.mb);
      t.row0 = t.tail ? t.mb * TM + (int)crank * 64 + (q & 1) * 32
                      : t.mb * TM + (int)crank * BM + q * 32;
      t.tcol = t.tail ? half * (BN / 4) : half * HALF;
      t.nch = (t.tail ? BN / 4 : HALF) / CW;
      if (KIND == 0) {
        t.nvalid = min(32, max(0, args.gm[t.g] - t.row0));
        t.orow0 = (long long)args.gc[t.g] + t.row0;
        t.bidx = args.gb[t.g];
      } else {
        t.nvalid = 32;
        t.bidx = args.gb[tab[t.g]];
        t.orow0 = (long long)t.bidx * args.M + t.row0;
      }
      t.col_base = t.nb * BN + (t.tail ? (q >> 1) * (BN / 2) : 0) + t.tcol;
      return t;
    };
    for (int w = unit; w < total_work; w += nunits, ++tcount) {
      const Geo geo = geo_of(w);
      const int g = geo.g;
      const int row0 = geo.row0, nch = geo.nch, nvalid = geo.nvalid, bidx = geo.bidx, tcol = geo.tcol;
      const long long orow0 = geo.orow0;
      // REMOTE: lane i holds the exclusive row offset, inside this expert's
      // contiguous receive region, of source (me + i) % P -- the receiver
      // keeps its own rows first (rotated source order, ep_p2p.cu)
      int rexcl = 0, rexp = 0;
      if (REMOTE) {
        rexp = ro.me * ro.El + bidx;
        const int cv = lane < ro.P ? ro.cnt[((ro.me + lane) % ro.P) * ro.E + rexp] : 0;
        int incl = cv;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += u;
        }
        rexcl = incl - cv;
      }
      // rotated position of the source of group row r (warp-collective)
      auto src_of = [&](int r) {
        int sidx = 0;
#pragma unroll
        for (int qq = 1; qq < 8; ++qq) {
          const int oq = __shfl_sync(0xffffffffu, rexcl, qq);
          if (qq < ro.P && r >= oq) sidx = qq;
        }
        return sidx;
      };
      const int col_base = geo.col_base;
      if (EPI == MOE_EPI_DGELU && lane == 0 && col_base < args.N) {
        mbar_arrive_expect_tx(&ab[0], STG);
        tma_load_2d(auxb, &tmAux, &ab[0], col_base, (int)orow0);
      }
      // bias slice of this warp's columns -> shared memory (coalesced, once per
      // tile, overlapping the wait for the accumulator)
      float* const bsm = reinterpret_cast<float*>(smem + C_::BIAS_OFF + ew * C_::BIAS_BYTES);
      const bool use_bias = C_::BIAS_BYTES > 0 && args.bias != nullptr;
      constexpr int NBV = (C_::BIAS_BYTES > 0 ? HALF : 32) / 32;  // bias values per lane
      float bv[NBV];
      if (use_bias) {  // loads in flight across the accumulator wait
        const float* bp = args.bias + (long long)bidx * args.N;
#pragma unroll
        for (int i = 0; i < NBV; ++i) {
          const int c = lane + 32 * i;
          bv[i] = (c < nch * CW && col_base + c < args.N) ? __ldg(bp + col_base + c) : 0.0f;
        }
      }
      int32_t gidx[2] = {-1, -1};
      if (EPI == MOE_EPI_GATHER_ADD && lane < nvalid) {
#pragma unroll
        for (int i = 0; i < 2; ++i)
          if (i < args.gk) gidx[i] = args.gidx[(orow0 + lane) * args.gk + i];
      }
      // GATHER_ADD: this lane's gathered 64-byte row pieces of chunk cc go to
      // aux buffer [i][cc] (swizzled like the staging tiles); every chunk of the
      // tile is requested up front, one cp.async group per chunk (4 groups)
      auto gather_prefetch = [&](int cc) {
        const int nn = col_base + cc * CW;
        if (nn + CW <= args.N) {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (gidx[i] < 0) continue;
            const __nv_bfloat16* src =
                reinterpret_cast<const __nv_bfloat16*>(args.gsrc) + (long long)gidx[i] * args.N + nn;
            const uint32_t dst = smem_u32(auxb + (i * 4 + cc) * STG);
#pragma unroll
            for (int j = 0; j < 4; ++j) cp_async16(dst + sw64(lane, j), src + j * 8);
          }
        }
        cp_async_commit();
      };
      if (EPI == MOE_EPI_GATHER_ADD) {
        static_assert(EPI != MOE_EPI_GATHER_ADD || (BN / 2) / C_::CW <= 4, "gather chunks");
        if (MOE_COOP_GATHER && col_base + nch * CW <= args.N) {
          // lanes cooperate per row: a warp instruction copies 2 (4) whole
          // gathered row pieces of 256 (128) contiguous bytes instead of 32
          // rows' 16-byte pieces -- coalesced reads of the scattered rows.
          // One cp.async group for the tile (+3 empty ones: same waits below)
          const int ppr = nch * 4, rpi = 32 / ppr;  // 16-byte pieces per row, rows per step
          const int q = lane % ppr, cq = q >> 2, jq = q & 3;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (i >= args.gk) break;
            for (int r0 = 0; r0 < 32; r0 += rpi) {
              const int r = r0 + lane / ppr;
              const int gi = __shfl_sync(0xffffffffu, gidx[i], r);
              if (gi >= 0) {
                const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(args.gsrc) +
                                           (long long)gi * args.N + col_base + q * 8;
                cp_async16(smem_u32(auxb + (i * 4 + cq) * STG) + sw64(r, jq), src);
              }
            }
          }
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) cp_async_commit();
        } else {
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            if (cc < nch) gather_prefetch(cc);
            else cp_async_commit();
          }
        }
      }
      const bool has_k = num_kblocks(g) > 0;
      const uint32_t acc = tcount & 1;
      mbar_wait(&tfull[acc], (tcount >> 1) & 1);
      tc_fence_after();
      if (use_bias) {
        __syncwarp();  // the previous tile's reads of the slice are done
#pragma unroll
        for (int i = 0; i < NBV; ++i) bsm[lane + 32 * i] = bv[i];
        __syncwarp();
      }
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + tcol;
#pragma unroll 1
      for (int c = 0; c < nch; ++c) {
        __syncwarp();
        float f[CW];
        {
          uint32_t v[CW];
          if constexpr (CW == 32) tmem_ld_32x32b_x32(t_row + c * CW, v);
          else tmem_ld_32x32b_x16(t_row + c * CW, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < CW; ++i) f[i] = has_k ? __uint_as_float(v[i]) : 0.0f;
        }
        const int n0 = col_base + c * CW;
        if (EPI == MOE_EPI_DGELU && lane == 0 && c + 1 < nch && n0 + CW < args.N) {
          mbar_arrive_expect_tx(&ab[(c + 1) & 1], STG);
          tma_load_2d(auxb + ((c + 1) & 1) * STG, &tmAux, &ab[(c + 1) & 1], n0 + CW, (int)orow0);
        }
        if (n0 >= args.N) continue;
        if (EPI == MOE_EPI_DGELU) {
          mbar_wait(&ab[c & 1], aph[c & 1]);
          aph[c & 1] ^= 1;
        }
        if (nvalid == 0) continue;
        uint8_t* const stg = stg_base + (C_::NBUF == 2 ? (nst & 1) : 0) * STG;
        uint8_t* const stg2 = stg_base + (C_::NBUF + (C_::NBUF == 2 ? (nst & 1) : 0)) * STG;
        const int ncols = min(CW, args.N - n0);
        const bool full_tile = nvalid == 32 && ncols == CW && !args.c_direct;
        const bool row_ok = lane < nvalid;
        if (EPI == MOE_EPI_ATOMIC_ADD) {
          if (row_ok) {
            float* Cp = reinterpret_cast<float*>(args.C);
            const long long m = orow0 + lane;
#pragma unroll
            for (int i = 0; i < CW; ++i) {
              if (i >= ncols) continue;
              const long long idx = args.transpose_c ? (long long)(n0 + i) * args.ldc + m
                                                     : m * args.ldc + n0 + i;
              atomicAdd(Cp + idx, f[i]);
            }
          }
          continue;
        }
        if (use_bias) {
          const float4* b4p = reinterpret_cast<const float4*>(bsm + c * CW);
#pragma unroll
          for (int i = 0; i < CW; i += 4) {
            const float4 b4 = b4p[i / 4];  // same address in every lane: broadcast
            const float2 lo = __fadd2_rn(make_float2(f[i], f[i + 1]), make_float2(b4.x, b4.y));
            const float2 hi = __fadd2_rn(make_float2(f[i + 2], f[i + 3]), make_float2(b4.z, b4.w));
            f[i] = lo.x;
            f[i + 1] = lo.y;
            f[i + 2] = hi.x;
            f[i + 3] = hi.y;
          }
        }
        float f2[CW];
        if (EPI == MOE_EPI_GELU) {
#pragma unroll
          for (int i = 0; i < CW; i += 2) {
            float2 a2, g2;
            gelu_and_grad_x2(make_float2(f[i], f[i + 1]), a2, g2);
            f[i] = a2.x;
            f[i + 1] = a2.y;
            f2[i] = g2.x;
            f2[i + 1] = g2.y;
          }
        }
        if (EPI == MOE_EPI_DGELU) {
          const uint8_t* ax = auxb + (c & 1) * STG;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint4 hv = *reinterpret_cast<const uint4*>(ax + sw64(lane, j));
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float2 m = __fmul2_rn(make_float2(f[j * 8 + 2 * i], f[j * 8 + 2 * i + 1]),
                                          bf16x2_to_float2(hw[i]));
              f[j * 8 + 2 * i] = m.x;
              f[j * 8 + 2 * i + 1] = m.y;
            }
          }
        }
        if (EPI == MOE_EPI_GATHER_ADD) {
          // chunk c's group done (the later chunks' may still be in flight)
          if (c == 0) cp_async_wait<3>();
          else if (c == 1) cp_async_wait<2>();
          else if (c == 2) cp_async_wait<1>();
          else cp_async_wait<0>();
          if (MOE_COOP_GATHER) __syncwarp();  // other lanes' copies of this lane's row
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (gidx[i] < 0) continue;
            if (ncols == CW) {
              const uint8_t* gb = auxb + (i * 4 + c) * STG;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const uint4 hv = *reinterpret_cast<const uint4*>(gb + sw64(lane, j));
                const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const float2 a2 = __fadd2_rn(make_float2(f[j * 8 + 2 * u], f[j * 8 + 2 * u + 1]),
                                               bf16x2_to_float2(hw[u]));
                  f[j * 8 + 2 * u] = a2.x;
                  f[j * 8 + 2 * u + 1] = a2.y;
                }
              }
            } else {
              const __nv_bfloat16* src = reinterpret_cast<const __nv_bfloat16*>(args.gsrc) +
                                         (long long)gidx[i] * args.N + n0;
#pragma unroll
              for (int u = 0; u < CW; ++u)
                if (u < ncols) f[u] += bf2f(src[u]);
            }
          }
        }
        if (REMOTE) {
          // return all-to-all fused into the epilogue: rows go straight to the
          // source rank's buffer over NVLink
          const int pl = src_of(row0 + lane);                    // this lane's row
          const int sl = (ro.me + pl) % ro.P;
          const int offl = __shfl_sync(0xffffffffu, rexcl, pl);
          const int p0 = __shfl_sync(0xffffffffu, pl, 0);
          const int p1 = __shfl_sync(0xffffffffu, pl, max(nvalid - 1, 0));
          const int off0 = __shfl_sync(0xffffffffu, rexcl, p0);
          const int s0 = (ro.me + p0) % ro.P;
          if (full_tile && p0 == p1) {
            if (lane == 0) {
              if (C_::NBUF == 2) bulk_wait_read1();
              else bulk_wait_read0();
            }
            __syncwarp();
            stage_row<CF32>(stg, lane, f);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&ro.maps[s0], stg, n0, (int)(rexp * ro.Cs + row0 - off0));
              bulk_commit();
            }
            ++nst;
          } else if (row_ok) {
            uint8_t* dst = ro.peers[sl] + ro.home_off;
            store_row_direct<CF32>(dst, (rexp * ro.Cs + row0 + lane - offl) * args.ldc + n0,
                                   ncols, f);
          }
          continue;
        }
        const bool want_colsum = EPI == MOE_EPI_DGELU && args.colsum != nullptr;
        if (full_tile || want_colsum) {
          if (lane == 0) {  // the store that last used this buffer has read it
            if (C_::NBUF == 2) bulk_wait_read1();
            else bulk_wait_read0();
          }
          __syncwarp();
          if (!row_ok) {
#pragma unroll
            for (int i = 0; i < CW; ++i) f[i] = 0.0f;
          }
          stage_row<CF32>(stg, lane, f);
          if (EPI == MOE_EPI_GELU) stage_row<CF32>(stg2, lane, f2);
          fence_proxy_async_smem();
          __syncwarp();
          if (full_tile && lane == 0) {
            tma_store_2d(&tmC, stg, n0, (int)orow0);
            if (EPI == MOE_EPI_GELU) tma_store_2d(&tmC2, stg2, n0, (int)orow0);
            bulk_commit();
          }
          if (full_tile) ++nst;
        }
        if (!full_tile && row_ok) {
          const long long off = (orow0 + lane) * args.ldc + n0;
          store_row_direct<CF32>(args.C, off, ncols, f, !args.c_direct);
          if (EPI == MOE_EPI_GELU) store_row_direct<CF32>(args.C2, off, ncols, f2);
        }
        if (want_colsum && !CF32) {
          // column sums of the stored (bf16-rounded) values, rows >= nvalid are zero
          // lane = (row parity, column pair): 16 x 4-byte reads per lane,
          // even/odd rows sit in opposite bank halves
          const uint32_t cp = lane & 15, rp = lane >> 4;
          float2 s = make_float2(0.f, 0.f);
#pragma unroll
          for (int r = 0; r < 16; ++r) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(
                stg + sw64(2 * r + rp, cp >> 2) + (cp & 3) * 4);
            s = __fadd2_rn(s, bf16x2_to_float2(w));
          }
          s.x += __shfl_xor_sync(0xffffffffu, s.x, 16);
          s.y += __shfl_xor_sync(0xffffffffu, s.y, 16);
          // this warp's 32-row block of group g owns its partial row: plain
          // stores, summed in block order afterwards (deterministic)
          float* cs = args.colsum + ((long long)g * args.cs_maxch + row0 / 32) * args.N + n0 + 2 * cp;
          if (rp == 0 && 2 * (int)cp < ncols) cs[0] = s.x;
          if (rp == 0 && 2 * (int)cp + 1 < ncols) cs[1] = s.y;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster_relaxed(mapa_shared(tempty0 + acc * 8, lead));
        else mbar_arrive(&tempty[acc]);
      }
    }
    if (lane == 0) bulk_wait0();
    if (REMOTE) __threadfence_system();  // remote rows visible before the signal kernel
  }

  __syncthreads();
  if (CG == 2) cluster_sync_all();  // the leader's MMAs into our TMEM are long complete
  if (warp == 10) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_2sm(tmem_base, C_::TMEM_COLS);
    else tmem_dealloc(tmem_base, C_::TMEM_COLS);
  }
}

// ------------------------------------------------------------------ host ----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  require(fn != nullptr, MOE_ERR_CUDA, "tma: cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 2D map over a row-major [outer][inner] matrix with row stride `ld` elements.
static CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                            uint32_t box_inner, uint32_t box_outer, bool f32 = false,
                            CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  const uint64_t es = f32 ? 4 : 2;
  const cuuint64_t dims[2] = {inner, outer ? outer : 1};
  const cuuint64_t strides[1] = {ld * es};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  require((reinterpret_cast<uintptr_t>(base) & 15) == 0, MOE_ERR_INVALID_ARGUMENT,
          "gemm: operand base must be 16-byte aligned");
  require((ld * es) % 16 == 0, MOE_ERR_INVALID_ARGUMENT,
          "gemm: operand row stride must be a multiple of 16 bytes");
  const CUresult r = encode_fn()(
      &m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, MOE_ERR_CUDA,
          "tma: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

template <int BN, bool A_MN, bool B_MN, int KIND, int EPI, bool CF32, int CG = 1,
          bool REMOTE = false>
static void launch(const moe_gemm_problem_t& p, cudaStream_t st,
                   const RemoteRows* remote = nullptr) {
  using C_ = Cfg<BN, EPI, CF32, CG, KIND>;
  constexpr int BH = BN / CG;
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN, KIND, EPI, CF32, CG, REMOTE>;
  // the smem opt-in is per device: remember which devices were configured
  static std::atomic<uint64_t> configured{0};
  int dev = 0;
  MOE_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(configured.load(std::memory_order_acquire) & bit)) {
    MOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM));
    configured.fetch_or(bit, std::memory_order_acq_rel);
  }
  CUtensorMap ta, tb, tcm, tc2, tax, tah;
  const bool split = p.split_terms == 6;
  // split-fp32: the maps span the three stacked planes
  const uint64_t np = split ? 3 : 1;
  uint64_t a_plane = 0, b_plane = 0;
  if (KIND == 0) {
    const uint64_t lda = p.lda ? p.lda : p.K;
    a_plane = p.a_rows;
    ta = make_map(p.A, p.K, np * p.a_rows, lda, 64, BM);
    tah = CG == 2 ? make_map(p.A, p.K, np * p.a_rows, lda, 64, 64) : ta;  // multicast halves
    if (!B_MN) {
      const uint64_t ldb = p.ldb ? p.ldb : p.K;
      const uint64_t rows = p.b_rows ? p.b_rows : (uint64_t)p.num_b * p.N;
      b_plane = rows;
      tb = make_map(p.B, p.K, np * rows, ldb, 64, BH);
    } else {
      const uint64_t ldb = p.ldb ? p.ldb : p.N;
      const uint64_t rows = p.b_rows ? p.b_rows : (uint64_t)p.num_b * p.K;
      b_plane = rows;
      tb = make_map(p.B, p.N, np * rows, ldb, 64, 64);
    }
  } else {
    const uint64_t lda = p.lda ? p.lda : p.M;
    const uint64_t ldb = p.ldb ? p.ldb : p.N;
    a_plane = p.a_rows;
    b_plane = p.b_rows ? p.b_rows : p.a_rows;
    ta = make_map(p.A, p.M, np * p.a_rows, lda, 64, 64);
    tah = ta;
    tb = make_map(p.B, p.N, np * b_plane, ldb, 64, 64);
  }
  const uint64_t c_rows = p.c_rows ? p.c_rows : (KIND == 0 ? p.a_rows : (uint64_t)p.num_b * p.M);
  tcm = tc2 = tax = ta;
  const uint64_t c_es = CF32 ? 4 : 2;
  const bool c_direct = (p.ldc * c_es) % 16 != 0 || (reinterpret_cast<uintptr_t>(p.C) & 15) != 0;
  require(!c_direct || (EPI == MOE_EPI_STORE && !REMOTE), MOE_ERR_INVALID_ARGUMENT,
          "gemm.ldc: rows must be 16-byte aligned for this epilogue");
  if (EPI != MOE_EPI_ATOMIC_ADD && !c_direct) {
    tcm = make_map(p.C, p.N, c_rows, p.ldc, C_::CW, 32, CF32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (EPI == MOE_EPI_GELU)
      tc2 = make_map(p.C2, p.N, c_rows, p.ldc, C_::CW, 32, CF32, CU_TENSOR_MAP_SWIZZLE_64B);
    if (EPI == MOE_EPI_DGELU)
      tax = make_map(p.aux, p.N, c_rows, p.ldc, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
  }
  Args a;
  a.groups = (int)p.groups;
  a.M = (int)p.M;
  a.N = (int)p.N;
  a.K = (int)p.K;
  a.gm = p.m;
  a.ga = p.a_row;
  a.gc = p.c_row;
  a.gb = p.b;
  a.C = p.C;
  a.C2 = p.C2;
  a.bias = p.bias;
  a.colsum = p.colsum_ws;
  a.cs_maxch = (int)((p.colsum_max_m + 31) / 32);
  a.gsrc = p.gather_src;
  a.gidx = p.gather_idx;
  a.gk = (int)p.gather_k;
  a.ldc = (long long)p.ldc;
  a.transpose_c = p.transpose_c;
  a.num_b = (int)p.num_b;
  a.c_direct = c_direct ? 1 : 0;
  a.terms = split ? 6 : 1;
  a.a_plane = (long long)a_plane;
  a.b_plane = (long long)b_plane;
  a.k_begin = (int)p.k_begin;
  a.k_len = (int)(p.k_len ? p.k_len : p.K - p.k_begin);
  a.gkb = p.k_begin_g;
  RemoteOut ro;  // remote descriptor (copied into the launch parameters)
  std::memset(&ro, 0, sizeof(ro));
  if (REMOTE) {
    require(remote != nullptr && remote->P <= 8, MOE_ERR_LOGIC, "gemm: remote rows descriptor");
    for (uint32_t q = 0; q < remote->P; ++q)
      ro.maps[q] = make_map(remote->peers_host[q] + remote->home_off, p.N,
                            (uint64_t)remote->E * remote->Cs, p.ldc, C_::CW, 32, CF32,
                            CU_TENSOR_MAP_SWIZZLE_64B);
    ro.peers = remote->peers_dev;
    ro.home_off = remote->home_off;
    ro.cnt = remote->cnt;
    ro.P = (int)remote->P;
    ro.me = (int)remote->me;
    ro.E = (int)remote->E;
    ro.El = (int)remote->El;
    ro.Cs = (long long)remote->Cs;
  }
  const int budget = gemm_cta_budget();
  const int grid = budget > 0 ? std::min(budget, num_sms()) : num_sms();
  if (CG == 1) {
    launch_pdl(kern, grid, THREADS, C_::SMEM, st, ta, tb, tcm, tc2, tax, tah, a, ro);
  } else {
    cudaLaunchConfig_t cfg = {};
    // multicast mode needs an even number of column blocks (the two pairs of a
    // cluster take consecutive ones) and whole quads of CTAs
    const int nblk_n = (int)((p.N + BN - 1) / BN);
    // (A/B on one B200, 64 experts: ffn2 / dgrad-ffn1 -2 to -3%, c2 step -0.7
    // to -1%, c3 -0.3 to -1.4%, the dense equivalent -3%; the GeLU / GeLU'
    // epilogue GEMMs, the fp32-output ones (c1 +1%) and the weight gradients
    // are not operand-bound enough to gain: pair mode for them)
    const bool mc = !REMOTE && gemm_multicast_enabled() && nblk_n % 2 == 0 &&
                    (grid & 3) == 0 && KIND == 0 && EPI == MOE_EPI_STORE && !CF32;
    cfg.gridDim = dim3((unsigned)std::max(2, grid & ~1));
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = C_::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[3];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (mc) {
      attr[na].id = cudaLaunchAttributePreferredClusterDimension;
      attr[na].val.preferredClusterDim.x = 4;
      attr[na].val.preferredClusterDim.y = 1;
      attr[na].val.preferredClusterDim.z = 1;
      ++na;
    }
    if (pdl_enabled()) {
      attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[na].val.programmaticStreamSerializationAllowed = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    MOE_CUDA(cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, tc2, tax, tah, a, ro));
  }
  MOE_LAUNCH_CHECK("tc_gemm_kernel");
  count_launch();
}

}  // namespace tc

bool gemm_multicast_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MOE_GEMM_MC");
    return !(e && e[0] == '0');
  }();
  return on;
}

int& gemm_cta_budget() {
  thread_local int budget = 0;
  return budget;
}

void tc_grouped_gemm(const moe_gemm_problem_t& p, cudaStream_t st, const RemoteRows* remote) {
  using namespace tc;
  if (remote != nullptr) {
    arg_check(p.kind == MOE_GEMM_RAGGED_M && p.epilogue == MOE_EPI_STORE &&
                  p.dtype_c == MOE_DTYPE_BF16,
              "gemm.remote: only bf16 RAGGED_M STORE GEMMs write to peers");
    if (p.b_mn_major) launch<256, false, true, 0, MOE_EPI_STORE, false, 2, true>(p, st, remote);
    else launch<256, false, false, 0, MOE_EPI_STORE, false, 2, true>(p, st, remote);
    return;
  }
  arg_check(p.groups >= 1 && p.groups <= MAX_GROUPS, "gemm.groups: must be in [1, 1024]");
  arg_check(p.dtype_ab == MOE_DTYPE_BF16, "gemm.dtype_ab: tcgen05 path needs bf16");
  arg_check(p.split_terms == 0 || p.split_terms == 1 ||
                (p.split_terms == 6 && p.dtype_c == MOE_DTYPE_F32 && p.epilogue == MOE_EPI_STORE),
            "gemm.split_terms: 0/1, or 6 (three bf16 planes per operand, fp32 STORE)");
  arg_check(p.kind == MOE_GEMM_RAGGED_K ||
                (p.k_begin % BK == 0 && p.k_len % BK == 0 && p.k_begin + p.k_len <= p.K),
            "gemm.k_begin/k_len: multiples of 64 inside [0, K]");
  arg_check(!p.k_begin_g || (p.kind == MOE_GEMM_RAGGED_M && p.k_len > 0),
            "gemm.k_begin_g: per-group K starts need RAGGED_M and k_len");
  const bool f32 = p.dtype_c == MOE_DTYPE_F32;
  if (p.kind == MOE_GEMM_RAGGED_M) {
    arg_check(p.K % BK == 0, "gemm.K: must be a multiple of 64");
    arg_check(p.N % 8 == 0 || p.epilogue == MOE_EPI_STORE,
              "gemm.N: must be a multiple of 8 (any N for STORE)");
    arg_check(!p.transpose_c, "gemm.transpose_c: only for RAGGED_K atomic");
    const bool bmn = p.b_mn_major != 0;
    if (p.N <= 64 && !bmn && p.epilogue == MOE_EPI_STORE) {
      if (f32) launch<64, false, false, 0, MOE_EPI_STORE, true>(p, st);
      else launch<64, false, false, 0, MOE_EPI_STORE, false>(p, st);
      return;
    }
    switch (p.epilogue) {
      case MOE_EPI_STORE:
        if (bmn) {
          if (f32) launch<256, false, true, 0, MOE_EPI_STORE, true, 2>(p, st);
          else launch<256, false, true, 0, MOE_EPI_STORE, false, 2>(p, st);
        } else {
          if (f32) launch<256, false, false, 0, MOE_EPI_STORE, true, 2>(p, st);
          else launch<256, false, false, 0, MOE_EPI_STORE, false, 2>(p, st);
        }
        return;
      case MOE_EPI_GELU:
        arg_check(!bmn && !f32, "gemm.epilogue: GELU needs K-major B and bf16 C");
        launch<256, false, false, 0, MOE_EPI_GELU, false, 2>(p, st);
        return;
      case MOE_EPI_DGELU: {
        arg_check(bmn && !f32, "gemm.epilogue: DGELU needs MN-major B and bf16 C");
        arg_check(!p.colsum || (p.colsum_ws && p.colsum_max_m >= 1),
                  "gemm.colsum_ws: DGELU column sums need colsum_ws / colsum_max_m");
        moe_gemm_problem_t q = p;
        if (!p.colsum) q.colsum_ws = nullptr;
        launch<256, false, true, 0, MOE_EPI_DGELU, false, 2>(q, st);
        if (p.colsum)
          seg_colsum(p.groups, p.m, p.b, p.num_b, p.N, 32, (uint32_t)((p.colsum_max_m + 31) / 32),
                     p.colsum_ws, p.colsum, st);
        return;
      }
      case MOE_EPI_GATHER_ADD:
        arg_check(bmn && !f32 && p.gather_src && p.gather_idx && p.gather_k >= 1 &&
                      p.gather_k <= 2,
                  "gemm.epilogue: GATHER_ADD needs MN-major B, bf16 C, gather_src/idx, k<=2");
        launch<256, false, true, 0, MOE_EPI_GATHER_ADD, false, 2>(p, st);
        return;
      default:
        fail(MOE_ERR_INVALID_ARGUMENT, "gemm.epilogue: unsupported for RAGGED_M");
    }
  } else {
    arg_check(p.M % BM == 0, "gemm.M: RAGGED_K needs M a multiple of 128");
    arg_check(p.N % 8 == 0 || p.epilogue == MOE_EPI_ATOMIC_ADD,
              "gemm.N: must be a multiple of 8 (any N for ATOMIC_ADD)");
    arg_check(f32, "gemm.dtype_c: RAGGED_K writes fp32");
    if (p.epilogue == MOE_EPI_ATOMIC_ADD) {
      if (p.N <= 64) launch<64, true, true, 1, MOE_EPI_ATOMIC_ADD, true>(p, st);
      else launch<256, true, true, 1, MOE_EPI_ATOMIC_ADD, true>(p, st);
      return;
    }
    arg_check(p.epilogue == MOE_EPI_STORE && !p.transpose_c,
              "gemm.epilogue: RAGGED_K supports STORE or ATOMIC_ADD");
    if (p.N <= 64) {  // narrow outputs (the split-K gate wgrad: N = E padded to 64)
      launch<64, true, true, 1, MOE_EPI_STORE, true>(p, st);
      return;
    }
    if (p.M % 256 == 0) launch<256, true, true, 1, MOE_EPI_STORE, true, 2>(p, st);
    else launch<256, true, true, 1, MOE_EPI_STORE, true, 1>(p, st);
  }
}

}  // namespace moe
