// K5 — grouped expert GEMM on 5th-generation tensor cores (sm_100a).
//
// One persistent, warp-specialised kernel per shape class:
//   warp 0      TMA producer (one lane): A/B tiles -> 128B-swizzled smem ring
//   warp 1      MMA issuer  (one lane): tcgen05.mma 128xBNx16, fp32 accum in TMEM
//   warp 2      TMEM allocator (2 x BN columns: double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld 32 lanes x 32 columns -> bias/GeLU/GeLU'
//               -> bf16/fp32 stores (or fp32 atomics for split-K)
// Work items are read from device-side group tables (no host sync on routing
// counts — the paper's CPU-side scheduling overhead):
//   RAGGED_M : group g = one (source, expert) slice of m[g] rows; tiles =
//              ceil(m/128) x ceil(N/BN); B = the expert's weight (K- or MN-major)
//   RAGGED_K : weight gradients; a segment = consecutive groups of one output,
//              K runs over the groups' rows (zero-padded to 64), A/B MN-major.
// The reference has no expert compute at all (cost model only:
// prefetch_cache.cpp:86-95, ring_offload.hpp:21); DESIGN.md §K5.
#include <cuda.h>

#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace moe {

namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int THREADS = 256;
constexpr int MAX_GROUPS = 1024;

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (BN == 256) ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int TMEM_COLS = 2 * BN;
  // smem: stages | barriers | tmem holder | tables
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int BAR_BYTES = (2 * STAGES + 4) * 8;
  static constexpr int HOLD_OFF = BAR_OFF + BAR_BYTES;
  static constexpr int TAB_OFF = ((HOLD_OFF + 16 + 15) / 16) * 16;
  static constexpr int SMEM = TAB_OFF + (MAX_GROUPS + 1) * 4 + 1024;  // + alignment slack
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
  const __nv_bfloat16* aux;
  const float* bias;
  long long ldc;
  int transpose_c;
  int num_b;
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

template <int BN, bool A_MN, bool B_MN, int KIND, int EPI, bool CF32>
__global__ void __launch_bounds__(THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const Args args) {
  using C_ = Cfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C_::BAR_OFF);
  uint64_t* empty = full + C_::STAGES;
  uint64_t* tfull = empty + C_::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_hold = reinterpret_cast<uint32_t*>(smem + C_::HOLD_OFF);
  int* tab = reinterpret_cast<int*>(smem + C_::TAB_OFF);  // [MAX_GROUPS+1]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int G = args.groups;
  const int nblk_n = (args.N + BN - 1) / BN;

  // ---- setup ---------------------------------------------------------
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C_::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    tmem_alloc(tmem_hold, C_::TMEM_COLS);
    tc_fence_before();
  }
  // Work tables: RAGGED_M -> tab = exclusive prefix of tiles per group;
  // RAGGED_K -> tab = first group of each segment (segment = output run,
  // or single group in atomic split-K mode).
  int* scratch = reinterpret_cast<int*>(smem);  // stage 0 is free during setup
  if (KIND == 0) {
    for (int g = threadIdx.x; g < G; g += THREADS) {
      const int m = args.gm[g];
      scratch[g] = ((m + BM - 1) / BM) * nblk_n;
    }
  } else {
    for (int g = threadIdx.x; g < G; g += THREADS) {
      const bool start = (EPI == MOE_EPI_ATOMIC_ADD) || g == 0 || args.gb[g] != args.gb[g - 1];
      scratch[g] = start ? 1 : 0;
    }
  }
  __syncthreads();
  if (warp == 3) {
    if (KIND == 0) {
      warp_scan_smem(scratch, G, tab);
    } else {
      // positions of segment starts: exclusive scan of flags, then compact
      int* pos = scratch + MAX_GROUPS + 1;
      warp_scan_smem(scratch, G, pos);
      __syncwarp();
      for (int g = lane; g < G; g += 32)
        if (scratch[g]) tab[pos[g]] = g;
      if (lane == 0) tab[pos[G]] = G;  // sentinel: nseg = pos[G]
      if (lane == 0) tab[MAX_GROUPS] = pos[G];
    }
  }
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_hold;

  int total_work;
  int nseg = 0;
  const int mt = args.M / BM;  // RAGGED_K only
  if (KIND == 0) {
    total_work = tab[G];
  } else {
    nseg = tab[MAX_GROUPS];
    total_work = nseg * mt * nblk_n;
  }

  // decode a work item
  auto decode = [&](int w, int& g, int& mb, int& nb) {
    if (KIND == 0) {
      int lo = 0, hi = G;  // last g with tab[g] <= w
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (tab[mid] <= w) lo = mid; else hi = mid;
      }
      // skip empty groups with equal prefix
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
    if (KIND == 0) return args.K / BK;
    int n = 0;
    for (int q = tab[g]; q < tab[g + 1]; ++q) n += (args.gm[q] + BK - 1) / BK;
    return n;
  };

  constexpr uint32_t IDESC = umma_idesc_bf16(BM, BN, A_MN, B_MN);

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      uint32_t it = 0;
      for (int w = blockIdx.x; w < total_work; w += gridDim.x) {
        int g, mb, nb;
        decode(w, g, mb, nb);
        if (KIND == 0) {
          const int arow = args.ga[g] + mb * BM;
          const int brow = args.gb[g] * (B_MN ? args.K : args.N);
          const int nkb = args.K / BK;
          for (int kb = 0; kb < nkb; ++kb, ++it) {
            const int s = it % C_::STAGES;
            mbar_wait(&empty[s], ((it / C_::STAGES) & 1) ^ 1);
            uint8_t* sA = smem + s * C_::STAGE_BYTES;
            uint8_t* sB = sA + C_::A_BYTES;
            mbar_arrive_expect_tx(&full[s], C_::STAGE_BYTES);
            tma_load_2d(sA, &tmA, &full[s], kb * BK, arow);  // A K-major box {64,128}
            if (!B_MN) {
              tma_load_2d(sB, &tmB, &full[s], kb * BK, brow + nb * BN);
            } else {
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_2d(sB + j * 8192, &tmB, &full[s], nb * BN + j * 64, brow + kb * BK);
            }
          }
        } else {
          for (int q = tab[g]; q < tab[g + 1]; ++q) {
            const int rows = args.gm[q];
            const int r0 = args.ga[q];
            for (int kb = 0; kb * BK < rows; ++kb, ++it) {
              const int s = it % C_::STAGES;
              mbar_wait(&empty[s], ((it / C_::STAGES) & 1) ^ 1);
              uint8_t* sA = smem + s * C_::STAGE_BYTES;
              uint8_t* sB = sA + C_::A_BYTES;
              mbar_arrive_expect_tx(&full[s], C_::STAGE_BYTES);
              const int row = r0 + kb * BK;
#pragma unroll
              for (int j = 0; j < BM / 64; ++j)
                tma_load_2d(sA + j * 8192, &tmA, &full[s], mb * BM + j * 64, row);
#pragma unroll
              for (int j = 0; j < BN / 64; ++j)
                tma_load_2d(sB + j * 8192, &tmB, &full[s], nb * BN + j * 64, row);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      uint32_t it = 0, tcount = 0;
      for (int w = blockIdx.x; w < total_work; w += gridDim.x, ++tcount) {
        int g, mb, nb;
        decode(w, g, mb, nb);
        const int nkb = num_kblocks(g);
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
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t da = A_MN ? umma_desc_sw128(aBase + kk * 2048, 8192, 1024)
                                     : umma_desc_sw128(aBase + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? umma_desc_sw128(bBase + kk * 2048, 8192, 1024)
                                     : umma_desc_sw128(bBase + kk * 32, 16, 1024);
            tc_mma_bf16(d_tmem, da, db, IDESC, (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue =================
    const int ew = warp - 4;          // TMEM lanes 32*ew .. 32*ew+31
    const int r = ew * 32 + lane;     // row within the tile
    uint32_t tcount = 0;
    for (int w = blockIdx.x; w < total_work; w += gridDim.x, ++tcount) {
      int g, mb, nb;
      decode(w, g, mb, nb);
      const uint32_t acc = tcount & 1;
      mbar_wait(&tfull[acc], (tcount >> 1) & 1);
      tc_fence_after();
      const bool has_k = num_kblocks(g) > 0;
      int m = mb * BM + r;
      bool row_ok;
      long long out_row;
      int bidx;
      if (KIND == 0) {
        row_ok = m < args.gm[g];
        out_row = (long long)args.gc[g] + m;
        bidx = args.gb[g];
      } else {
        row_ok = m < args.M;
        bidx = args.gb[tab[g]];
        out_row = (long long)bidx * args.M + m;
      }
      const uint32_t t_row = tmem_base + ((uint32_t)(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        __syncwarp();
        uint32_t v[32];
        tmem_ld_32x32b_x32(t_row + c * 32, v);
        tmem_ld_wait();
        const int n0 = nb * BN + c * 32;
        if (!row_ok || n0 >= args.N) continue;
        float f[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) f[i] = has_k ? __uint_as_float(v[i]) : 0.0f;
        const bool full_cols = n0 + 32 <= args.N;
        if (args.bias != nullptr && EPI != MOE_EPI_ATOMIC_ADD && EPI != MOE_EPI_DGELU) {
          const float* bp = args.bias + (long long)bidx * args.N + n0;
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] += (full_cols || n0 + i < args.N) ? bp[i] : 0.0f;
        }
        if (EPI == MOE_EPI_ATOMIC_ADD) {
          float* Cp = reinterpret_cast<float*>(args.C);
          for (int i = 0; i < 32; ++i) {
            const int n = n0 + i;
            if (n >= args.N) break;
            const long long idx = args.transpose_c
                                      ? (long long)n * args.ldc + out_row
                                      : out_row * args.ldc + n;
            atomicAdd(Cp + idx, f[i]);
          }
          continue;
        }
        if (EPI == MOE_EPI_DGELU) {
          const __nv_bfloat16* hp = args.aux + out_row * args.ldc + n0;
          if (full_cols) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const uint4 hv = *reinterpret_cast<const uint4*>(hp + q * 8);
              const __nv_bfloat16* h8 = reinterpret_cast<const __nv_bfloat16*>(&hv);
#pragma unroll
              for (int i = 0; i < 8; ++i) f[q * 8 + i] *= gelu_grad_f(bf2f(h8[i]));
            }
          } else {
            for (int i = 0; i < 32; ++i)
              if (n0 + i < args.N) f[i] *= gelu_grad_f(bf2f(hp[i]));
          }
        }
        if (EPI == MOE_EPI_GELU) {
          __nv_bfloat16* c2 = reinterpret_cast<__nv_bfloat16*>(args.C2) + out_row * args.ldc + n0;
          if (full_cols) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 o;
              o.x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
              o.y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
              o.z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
              o.w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
              *reinterpret_cast<uint4*>(c2 + q * 8) = o;
            }
          } else {
            for (int i = 0; i < 32; ++i)
              if (n0 + i < args.N) c2[i] = f2bf(f[i]);
          }
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = gelu_f(f[i]);
        }
        if (CF32) {
          float* cp = reinterpret_cast<float*>(args.C) + out_row * args.ldc + n0;
          if (full_cols) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              *reinterpret_cast<float4*>(cp + q * 4) =
                  make_float4(f[q * 4], f[q * 4 + 1], f[q * 4 + 2], f[q * 4 + 3]);
          } else {
            for (int i = 0; i < 32; ++i)
              if (n0 + i < args.N) cp[i] = f[i];
          }
        } else {
          __nv_bfloat16* cp = reinterpret_cast<__nv_bfloat16*>(args.C) + out_row * args.ldc + n0;
          if (full_cols) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 o;
              o.x = pack_bf16x2(f[q * 8 + 0], f[q * 8 + 1]);
              o.y = pack_bf16x2(f[q * 8 + 2], f[q * 8 + 3]);
              o.z = pack_bf16x2(f[q * 8 + 4], f[q * 8 + 5]);
              o.w = pack_bf16x2(f[q * 8 + 6], f[q * 8 + 7]);
              *reinterpret_cast<uint4*>(cp + q * 8) = o;
            }
          } else {
            for (int i = 0; i < 32; ++i)
              if (n0 + i < args.N) cp[i] = f2bf(f[i]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C_::TMEM_COLS);
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

// bf16 2D map over a row-major [outer][inner] matrix with row stride `ld`
// elements, 128B swizzle, zero OOB fill.
static CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                            uint32_t box_inner, uint32_t box_outer) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t es[2] = {1, 1};
  require((reinterpret_cast<uintptr_t>(base) & 15) == 0, MOE_ERR_INVALID_ARGUMENT,
          "gemm: operand base must be 16-byte aligned");
  require((ld * 2) % 16 == 0, MOE_ERR_INVALID_ARGUMENT,
          "gemm: operand row stride must be a multiple of 16 bytes");
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base),
                                 dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  require(r == CUDA_SUCCESS, MOE_ERR_CUDA, "tma: cuTensorMapEncodeTiled failed (" +
                                               std::to_string((int)r) + ")");
  return m;
}

template <int BN, bool A_MN, bool B_MN, int KIND, int EPI, bool CF32>
static void launch(const moe_gemm_problem_t& p, cudaStream_t st) {
  using C_ = Cfg<BN>;
  auto kern = tc_gemm_kernel<BN, A_MN, B_MN, KIND, EPI, CF32>;
  static bool attr = false;
  if (!attr) {
    MOE_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C_::SMEM));
    attr = true;
  }
  CUtensorMap ta, tb;
  if (KIND == 0) {
    const uint64_t lda = p.lda ? p.lda : p.K;
    ta = make_map(p.A, p.K, p.a_rows, lda, 64, BM);
    if (!B_MN) {
      const uint64_t ldb = p.ldb ? p.ldb : p.K;
      const uint64_t rows = p.b_rows ? p.b_rows : (uint64_t)p.num_b * p.N;
      tb = make_map(p.B, p.K, rows, ldb, 64, BN);
    } else {
      const uint64_t ldb = p.ldb ? p.ldb : p.N;
      const uint64_t rows = p.b_rows ? p.b_rows : (uint64_t)p.num_b * p.K;
      tb = make_map(p.B, p.N, rows, ldb, 64, 64);
    }
  } else {
    const uint64_t lda = p.lda ? p.lda : p.M;
    const uint64_t ldb = p.ldb ? p.ldb : p.N;
    ta = make_map(p.A, p.M, p.a_rows, lda, 64, 64);
    tb = make_map(p.B, p.N, p.b_rows ? p.b_rows : p.a_rows, ldb, 64, 64);
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
  a.aux = reinterpret_cast<const __nv_bfloat16*>(p.aux);
  a.bias = p.bias;
  a.ldc = (long long)p.ldc;
  a.transpose_c = p.transpose_c;
  a.num_b = (int)p.num_b;
  const int grid = num_sms();
  kern<<<grid, THREADS, C_::SMEM, st>>>(ta, tb, a);
  MOE_LAUNCH_CHECK("tc_gemm_kernel");
  count_launch();
}

}  // namespace tc

void tc_grouped_gemm(const moe_gemm_problem_t& p, cudaStream_t st) {
  using namespace tc;
  arg_check(p.groups >= 1 && p.groups <= MAX_GROUPS, "gemm.groups: must be in [1, 1024]");
  arg_check(p.dtype_ab == MOE_DTYPE_BF16, "gemm.dtype_ab: tcgen05 path needs bf16");
  if (p.kind == MOE_GEMM_RAGGED_M) {
    arg_check(p.K % BK == 0, "gemm.K: must be a multiple of 64");
    arg_check(p.N % 8 == 0, "gemm.N: must be a multiple of 8");
    arg_check(!p.transpose_c, "gemm.transpose_c: only for RAGGED_K atomic");
    const bool f32 = p.dtype_c == MOE_DTYPE_F32;
    const bool bmn = p.b_mn_major != 0;
    if (p.N <= 64 && !bmn && p.epilogue == MOE_EPI_STORE) {
      if (f32) launch<64, false, false, 0, MOE_EPI_STORE, true>(p, st);
      else launch<64, false, false, 0, MOE_EPI_STORE, false>(p, st);
      return;
    }
    switch (p.epilogue) {
      case MOE_EPI_STORE:
        if (bmn) {
          if (f32) launch<256, false, true, 0, MOE_EPI_STORE, true>(p, st);
          else launch<256, false, true, 0, MOE_EPI_STORE, false>(p, st);
        } else {
          if (f32) launch<256, false, false, 0, MOE_EPI_STORE, true>(p, st);
          else launch<256, false, false, 0, MOE_EPI_STORE, false>(p, st);
        }
        return;
      case MOE_EPI_GELU:
        arg_check(!bmn && !f32, "gemm.epilogue: GELU needs K-major B and bf16 C");
        launch<256, false, false, 0, MOE_EPI_GELU, false>(p, st);
        return;
      case MOE_EPI_DGELU:
        arg_check(bmn && !f32, "gemm.epilogue: DGELU needs MN-major B and bf16 C");
        launch<256, false, true, 0, MOE_EPI_DGELU, false>(p, st);
        return;
      default:
        fail(MOE_ERR_INVALID_ARGUMENT, "gemm.epilogue: unsupported for RAGGED_M");
    }
  } else {
    arg_check(p.M % BM == 0, "gemm.M: RAGGED_K needs M a multiple of 128");
    arg_check(p.N % 8 == 0, "gemm.N: must be a multiple of 8");
    arg_check(p.dtype_c == MOE_DTYPE_F32, "gemm.dtype_c: RAGGED_K writes fp32");
    if (p.epilogue == MOE_EPI_ATOMIC_ADD) {
      if (p.N <= 64) launch<64, true, true, 1, MOE_EPI_ATOMIC_ADD, true>(p, st);
      else launch<256, true, true, 1, MOE_EPI_ATOMIC_ADD, true>(p, st);
      return;
    }
    arg_check(p.epilogue == MOE_EPI_STORE && !p.transpose_c,
              "gemm.epilogue: RAGGED_K supports STORE or ATOMIC_ADD");
    launch<256, true, true, 1, MOE_EPI_STORE, true>(p, st);
  }
}

}  // namespace moe
