/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the SE-MoE MoE-layer hot path (arXiv 2205.10034) as the
 * reference (`/root/reference/proj`, "moesim") defines it where it exists, and
 * as DESIGN.md Appendix A defines it where the reference has no arithmetic.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or the
 * reported CPU baseline.  The product path (paper_2205_10034_b200/csrc) never
 * links or calls it.
 *
 * Parity status:
 *   - SplitMix64 / substream_seed  : pinned (rng.hpp:19-42, golden vectors from
 *                                    the compiled reference in tests/golden/).
 *   - gen_trace / imbalance_ratio  : pinned (workload.cpp:19-66, golden vectors).
 *   - alltoall_flat, fuse/split    : pinned (collectives.cpp:10-21, 88-118).
 *   - ring schedule + timing       : pinned (ring_offload.cpp:31-117,
 *                                    sim_engine.cpp:36-60, topology.cpp:73-84).
 *   - gating / capacity / aux loss / dispatch / expert FFN / combine and their
 *     backward: PARITY UNPINNED — the reference declares them out of scope
 *     (SPEC.md:15,153,156); semantics follow DESIGN.md Appendix A (GShard /
 *     Switch convention) and are fixed there.
 *
 * All floating arithmetic here accumulates in double.  Build with
 * -ffp-contract=off so the input generators match the device generators bit for
 * bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_INVALID 1
#define ORACLE_ERR_RANGE 2
#define ORACLE_ERR_CONFIG 3

/* ---------------------------------------------------------------- rng ---- */
/* rng.hpp:23-31 — SplitMix64 step. */
static inline uint64_t sm64_next(uint64_t* state) {
  *state += 0x9E3779B97F4A7C15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
/* rng.hpp:32 — uniform double in [0,1) with 53 random bits. */
static inline double sm64_u01(uint64_t* state) {
  return (double)(sm64_next(state) >> 11) * 0x1.0p-53;
}

uint64_t oracle_splitmix64_next(uint64_t* state) { return sm64_next(state); }

/* rng.hpp:40-42 */
uint64_t oracle_substream_seed(uint64_t seed, uint64_t step, uint64_t rank) {
  return seed ^ (0x9E3779B97F4A7C15ull * (step + 1)) ^ (0xC2B2AE3D27D4EB4Full * (rank + 1));
}

/* Synthetic tensor fill used by every harness: element i
 * is lo + (hi - lo) * u_i where u_i is the i-th draw of SplitMix64(seed),
 * computed in double and rounded to float. */
void oracle_fill_uniform(uint64_t seed, uint64_t n, double lo, double hi, float* out) {
  uint64_t s = seed;
  const double span = hi - lo;
  for (uint64_t i = 0; i < n; ++i) {
    const double u = sm64_u01(&s);
    out[i] = (float)(lo + span * u);
  }
}

/* float -> bf16 -> float, round-to-nearest-even (NaN preserved). */
static inline float bf16_round(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) {
    u |= 0x00400000u;
    u &= 0xffff0000u;
  } else {
    const uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    u &= 0xffff0000u;
  }
  float r;
  memcpy(&r, &u, 4);
  return r;
}

void oracle_round_bf16(uint64_t n, float* data) {
  for (uint64_t i = 0; i < n; ++i) data[i] = bf16_round(data[i]);
}

/* ----------------------------------------------------------- workload ---- */
/* workload.cpp:19-53 — Zipf (e+1)^-skew CDF, one SplitMix64 draw per token,
 * expert = upper_bound(cdf, u), counts[step][rank][expert]. */
int oracle_gen_trace(uint64_t seed, uint32_t steps, uint32_t ranks, uint32_t experts,
                     uint64_t tokens, double skew, uint64_t* counts) {
  if (experts == 0) return ORACLE_ERR_CONFIG;
  if (skew < 0.0) return ORACLE_ERR_CONFIG;
  double* cdf = (double*)malloc(sizeof(double) * experts);
  double acc = 0.0;
  for (uint32_t e = 0; e < experts; ++e) {
    acc += pow((double)(e + 1), -skew);
    cdf[e] = acc;
  }
  for (uint32_t e = 0; e < experts; ++e) cdf[e] /= acc;
  cdf[experts - 1] = 1.0;
  memset(counts, 0, sizeof(uint64_t) * (size_t)steps * ranks * experts);
  for (uint32_t s = 0; s < steps; ++s) {
    for (uint32_t r = 0; r < ranks; ++r) {
      uint64_t st = oracle_substream_seed(seed, s, r);
      uint64_t* row = counts + ((size_t)s * ranks + r) * experts;
      for (uint64_t t = 0; t < tokens; ++t) {
        const double u = sm64_u01(&st);
        /* upper_bound: first index with cdf[i] > u */
        uint32_t lo = 0, hi = experts;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) / 2;
          if (cdf[mid] > u) hi = mid; else lo = mid + 1;
        }
        row[lo < experts - 1 ? lo : experts - 1] += 1;
      }
    }
  }
  free(cdf);
  return ORACLE_OK;
}

/* workload.cpp:55-66 — max expert total / mean expert total. */
int oracle_imbalance_ratio(uint32_t steps, uint32_t ranks, uint32_t experts,
                           const uint64_t* counts, double* out) {
  uint64_t total = 0, max_total = 0;
  for (uint32_t e = 0; e < experts; ++e) {
    uint64_t t = 0;
    for (uint32_t s = 0; s < steps; ++s)
      for (uint32_t r = 0; r < ranks; ++r) t += counts[((size_t)s * ranks + r) * experts + e];
    total += t;
    if (t > max_total) max_total = t;
  }
  if (total == 0) return ORACLE_ERR_CONFIG;
  const double mean = (double)total / (double)experts;
  *out = (double)max_total / mean;
  return ORACLE_OK;
}

/* -------------------------------------------------------- collectives ---- */
/* collectives.cpp:10-21 — out[i][j] = in[j][i] over an R x R ragged chunk
 * matrix.  Chunks are passed flattened: lens[src*R+dst], data concatenated in
 * row-major (src, dst) order; the output uses the same convention. */
int oracle_alltoall_flat(uint64_t ranks, uint64_t n_chunks, const uint64_t* lens,
                         const uint8_t* data, uint64_t* out_lens, uint8_t* out_data) {
  if (n_chunks != ranks * ranks) return ORACLE_ERR_INVALID;
  uint64_t* in_off = (uint64_t*)malloc(sizeof(uint64_t) * (n_chunks + 1));
  in_off[0] = 0;
  for (uint64_t i = 0; i < n_chunks; ++i) in_off[i + 1] = in_off[i] + lens[i];
  uint64_t o = 0;
  for (uint64_t dst = 0; dst < ranks; ++dst) {
    for (uint64_t src = 0; src < ranks; ++src) {
      const uint64_t c = src * ranks + dst; /* out.at(dst, src) = in.at(src, dst) */
      out_lens[dst * ranks + src] = lens[c];
      memcpy(out_data + o, data + in_off[c], lens[c]);
      o += lens[c];
    }
  }
  free(in_off);
  return ORACLE_OK;
}

/* topology.cpp:61-71 route(): hop classes [nvlink,pcie,ssd_io,tor,leaf,spin]
 * between two GPUs given as (node index, local rank). */
static void oracle_route_hops(uint64_t na, uint64_t la, uint64_t nb, uint64_t lb, uint64_t* hops,
                              uint64_t* transfers) {
  if (na == nb && la == lb) return;
  *transfers += 1;
  if (na == nb) {
    hops[0] += 1;
  } else if (la == lb) {
    hops[3] += 2;
    hops[4] += 1;
  } else {
    hops[3] += 2;
    hops[4] += 2;
    hops[5] += 1;
  }
}

/* collectives.cpp:31-79 — two-phase rail-aware all-to-all.  Delivery is the
 * flat transpose (the chunks only travel through holders); the stats count
 * phase 1 (src -> holder on src's node with dst's local rank) and phase 2
 * (holder -> dst) hops.  stats: phase1_hops[6], phase2_hops[6], p1, p2. */
int oracle_alltoall_hierarchical(uint32_t clusters, uint32_t nodes, uint32_t gpus, uint64_t ranks,
                                 uint64_t n_chunks, const uint64_t* lens, const uint8_t* data,
                                 uint64_t* out_lens, uint8_t* out_data, uint64_t* stats) {
  if (clusters == 0 || nodes == 0 || gpus == 0) return ORACLE_ERR_CONFIG;
  if (n_chunks != ranks * ranks) return ORACLE_ERR_INVALID;
  if (ranks != (uint64_t)clusters * nodes * gpus) return ORACLE_ERR_INVALID;
  memset(stats, 0, 14 * sizeof(uint64_t));
  for (uint64_t s = 0; s < ranks; ++s)
    for (uint64_t d = 0; d < ranks; ++d) {
      /* node index = cluster * nodes + node identifies the node uniquely */
      const uint64_t ns = s / gpus, ls = s % gpus, nd = d / gpus, ld = d % gpus;
      oracle_route_hops(ns, ls, ns, ld, stats, &stats[12]);
      oracle_route_hops(ns, ld, nd, ld, stats + 6, &stats[13]);
    }
  return oracle_alltoall_flat(ranks, n_chunks, lens, data, out_lens, out_data);
}

/* collectives.cpp:88-98 — concatenate, index = (slice_id, offset, length). */
int oracle_fuse_slices(uint64_t n, const uint64_t* lens, const uint8_t* data, uint8_t* blob,
                       uint64_t* index /* n x 3 */) {
  if (n == 0) return ORACLE_ERR_INVALID;
  uint64_t off = 0;
  for (uint64_t i = 0; i < n; ++i) {
    index[3 * i + 0] = i;
    index[3 * i + 1] = off;
    index[3 * i + 2] = lens[i];
    memcpy(blob + off, data + off, lens[i]);
    off += lens[i];
  }
  return ORACLE_OK;
}

/* collectives.cpp:100-118 — validate contiguity + coverage, then split. */
int oracle_split_blob(uint64_t blob_len, const uint8_t* blob, uint64_t n, const uint64_t* index,
                      uint8_t* out) {
  uint64_t expect = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (index[3 * i + 1] != expect) return ORACLE_ERR_INVALID;
    expect += index[3 * i + 2];
  }
  if (expect != blob_len) return ORACLE_ERR_INVALID;
  uint64_t o = 0;
  for (uint64_t i = 0; i < n; ++i) {
    memcpy(out + o, blob + index[3 * i + 1], index[3 * i + 2]);
    o += index[3 * i + 2];
  }
  return ORACLE_OK;
}

/* --------------------------------------------------------------- ring ---- */
/* ring_offload.cpp:31-50 — ops as (kind, layer, slot, waits_release_of or -1);
 * kind 0 = load, 1 = compute, 2 = release.  Returns the op count through
 * *n_ops; ops must hold 3 * (slots + 2 * layers) int64. */
int oracle_ring_schedule(uint32_t layers, uint32_t ring_slots, int64_t* ops, uint64_t* n_ops,
                         uint32_t* slots_out, int* clamped) {
  if (layers < 1 || ring_slots == 0) return ORACLE_ERR_CONFIG;
  const uint32_t K = ring_slots < layers ? ring_slots : layers;
  *clamped = ring_slots > layers;
  *slots_out = K;
  uint64_t n = 0;
#define PUT(k, l, s, w) do { ops[4*n+0]=(k); ops[4*n+1]=(l); ops[4*n+2]=(s); ops[4*n+3]=(w); ++n; } while (0)
  for (uint32_t i = 0; i < K; ++i) PUT(0, i, i % K, -1);
  for (uint32_t i = 0; i < layers; ++i) {
    PUT(1, i, i % K, -1);
    PUT(2, i, i % K, -1);
    if (i + K < layers) PUT(0, i + K, (i + K) % K, i);
  }
#undef PUT
  *n_ops = n;
  return ORACLE_OK;
}

/* topology.cpp:73-84 for a one-hop path: lat + ceil(bytes * 1e9 / bw). */
static int64_t transfer_ns(uint64_t bytes, uint64_t bw, int64_t lat) {
  if (bytes == 0) return lat;
  const unsigned __int128 num = (unsigned __int128)bytes * 1000000000u;
  return lat + (int64_t)((num - 1) / bw + 1);
}

/* ring_offload.cpp:52-106 restated on the FIFO-stream semantics of
 * sim_engine.cpp:36-52: loads serialise on the h2d stream, computes and
 * zero-time releases on the compute stream.  Writes per-layer
 * load/compute start/end (ns) and the summary metrics. */
int oracle_ring_simulate(uint32_t layers, uint32_t ring_slots, uint64_t expert_bytes,
                         uint64_t dense_bytes, const int64_t* compute_ns, uint64_t pcie_bw,
                         int64_t pcie_lat, int64_t* load_start, int64_t* load_end,
                         int64_t* comp_start, int64_t* comp_end, int64_t* makespan,
                         int64_t* stall, int64_t* copy_ns, uint64_t* peak_bytes,
                         uint64_t* baseline_bytes) {
  if (layers < 1 || ring_slots == 0) return ORACLE_ERR_CONFIG;
  const uint32_t K = ring_slots < layers ? ring_slots : layers;
  const int64_t c = transfer_ns(expert_bytes, pcie_bw, pcie_lat);
  int64_t h2d_free = 0, comp_free = 0, total = 0, end = 0;
  int64_t* release_end = (int64_t*)calloc(layers, sizeof(int64_t));
  for (uint32_t i = 0; i < K; ++i) {
    load_start[i] = h2d_free;
    load_end[i] = h2d_free + c;
    h2d_free = load_end[i];
  }
  for (uint32_t i = 0; i < layers; ++i) {
    const int64_t s = load_end[i] > comp_free ? load_end[i] : comp_free;
    comp_start[i] = s;
    comp_end[i] = s + compute_ns[i];
    comp_free = comp_end[i];
    release_end[i] = comp_free; /* zero-duration release right after compute */
    total += compute_ns[i];
    if (i + K < layers) {
      const uint32_t j = i + K;
      const int64_t ls = h2d_free > release_end[i] ? h2d_free : release_end[i];
      load_start[j] = ls;
      load_end[j] = ls + c;
      h2d_free = load_end[j];
    }
  }
  for (uint32_t i = 0; i < layers; ++i) {
    if (comp_end[i] > end) end = comp_end[i];
    if (load_end[i] > end) end = load_end[i];
  }
  free(release_end);
  *makespan = end;
  *stall = end - total;
  *copy_ns = c;
  *peak_bytes = dense_bytes + (uint64_t)K * expert_bytes;
  *baseline_bytes = dense_bytes + (uint64_t)layers * expert_bytes;
  return ORACLE_OK;
}

/* ------------------------------------------------------------ routing ---- */
/* DESIGN.md Appendix A (builder-owned semantics; not in the reference).
 *  top-1 e1 = argmax logits (NaN treated as -inf, ties to the lowest index);
 *  top-2 e2 = argmax over e != e1; p = softmax(logits) max-subtracted;
 *  k=1: g1 = p[e1]; k=2: g_i = p[e_i]/(p[e1]+p[e2]);
 *  pos1[t] = #{t'<t: e1[t']=e1[t]};
 *  pos2[t] = count1[e2[t]] + #{t'<t: e2[t']=e2[t]};
 *  keep = pos < C;  l_aux = E * sum_e mean_t(p[t,e]) * count1[e]/T.
 * Outputs: expert[T*k], gate[T*k] (double), pos[T*k], keep[T*k],
 * count1[E], count2[E], kept[E] = min(count1+count2, C), aux. */
static inline int lt_nan_low(float a, float b) { /* a < b with NaN read as -inf */
  const float x = isnan(a) ? -INFINITY : a;
  const float y = isnan(b) ? -INFINITY : b;
  return x < y;
}

int oracle_route(uint64_t T, uint32_t E, uint32_t k, uint64_t C, const float* logits,
                 int32_t* expert, double* gate, int32_t* pos, uint8_t* keep, int32_t* count1,
                 int32_t* count2, int32_t* kept, double* aux, double* probs_out /* nullable T*E */) {
  if (E == 0 || (k != 1 && k != 2) || (k == 2 && E < 2)) return ORACLE_ERR_CONFIG;
  double* psum = (double*)calloc(E, sizeof(double));
  double* p = (double*)malloc(sizeof(double) * E);
  memset(count1, 0, sizeof(int32_t) * E);
  memset(count2, 0, sizeof(int32_t) * E);
  for (uint64_t t = 0; t < T; ++t) {
    const float* L = logits + t * E;
    uint32_t e1 = 0;
    for (uint32_t e = 1; e < E; ++e)
      if (lt_nan_low(L[e1], L[e])) e1 = e;
    uint32_t e2 = 0;
    if (k == 2) {
      e2 = (e1 == 0) ? 1 : 0;
      for (uint32_t e = 0; e < E; ++e)
        if (e != e1 && lt_nan_low(L[e2], L[e])) e2 = e;
    }
    const double m = (double)L[e1];
    double z = 0.0;
    for (uint32_t e = 0; e < E; ++e) {
      p[e] = exp((double)L[e] - m);
      z += p[e];
    }
    for (uint32_t e = 0; e < E; ++e) {
      p[e] /= z;
      psum[e] += p[e];
      if (probs_out) probs_out[t * E + e] = p[e];
    }
    expert[t * k] = (int32_t)e1;
    if (k == 1) {
      gate[t] = p[e1];
    } else {
      const double s = p[e1] + p[e2];
      expert[t * 2 + 1] = (int32_t)e2;
      gate[t * 2] = p[e1] / s;
      gate[t * 2 + 1] = p[e2] / s;
    }
    pos[t * k] = count1[e1]++;
  }
  if (k == 2) {
    for (uint64_t t = 0; t < T; ++t) {
      const int32_t e2 = expert[t * 2 + 1];
      pos[t * 2 + 1] = count1[e2] + count2[e2]++;
    }
  }
  for (uint64_t i = 0; i < T * k; ++i) keep[i] = (uint64_t)pos[i] < C;
  double a = 0.0;
  for (uint32_t e = 0; e < E; ++e) {
    const int64_t tot = (int64_t)count1[e] + count2[e];
    kept[e] = (int32_t)(tot < (int64_t)C ? tot : (int64_t)C);
    a += (psum[e] / (double)T) * ((double)count1[e] / (double)T);
  }
  *aux = T ? (double)E * a : 0.0;
  free(psum);
  free(p);
  return ORACLE_OK;
}

/* ---------------------------------------------------------- MoE layer ---- */
static inline double gelu(double h) { return 0.5 * h * (1.0 + erf(h * 0.70710678118654752440)); }
static inline double gelu_grad(double h) {
  return 0.5 * (1.0 + erf(h * 0.70710678118654752440)) +
         h * 0.39894228040143267794 * exp(-0.5 * h * h);
}
static inline double rnd(double v, int bf16) { return bf16 ? (double)bf16_round((float)v) : (double)(float)v; }

/* Forward of one MoE layer on one source shard (DESIGN.md Appendix A §8).
 *   x[T,d], wg[E,d], bg[E] (nullable), w1[E,dff,d], b1[E,dff], w2[E,d,dff], b2[E,d]
 *   logits_in (nullable): when given, routing uses these fp32 logits (the
 *   GPU's), after the caller checked them against logits_out.
 * emulate_bf16 = 1 rounds every stored intermediate to bf16 at the same points
 * the bf16 device path stores them; 0 rounds to fp32.
 * Outputs: logits_out[T,E] (float, fp64-accumulated), routing arrays, y[T,d]
 * (double), and per kept slot the H/A rows are not exposed.  Returns 0. */
int oracle_moe_forward(uint64_t T, uint32_t d, uint32_t dff, uint32_t E, uint32_t k, uint64_t C,
                       int emulate_bf16, const float* x, const float* wg, const float* bg,
                       const float* w1, const float* b1, const float* w2, const float* b2,
                       const float* logits_in, float* logits_out, int32_t* expert, double* gate,
                       int32_t* pos, uint8_t* keep, int32_t* count1, int32_t* count2,
                       int32_t* kept, double* aux, double* y) {
  /* logits = x wg^T + bg, fp64 accumulation, stored fp32 */
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)T; ++t) {
    for (uint32_t e = 0; e < E; ++e) {
      double acc = 0.0;
      const float* xr = x + (uint64_t)t * d;
      const float* wr = wg + (uint64_t)e * d;
      for (uint32_t i = 0; i < d; ++i) acc += (double)xr[i] * (double)wr[i];
      if (bg) acc += (double)bg[e];
      logits_out[(uint64_t)t * E + e] = (float)acc;
    }
  }
  const float* L = logits_in ? logits_in : logits_out;
  int rc = oracle_route(T, E, k, C, L, expert, gate, pos, keep, count1, count2, kept, aux, NULL);
  if (rc) return rc;
  memset(y, 0, sizeof(double) * T * d);
  /* per token-choice expert FFN; kept slots only */
#pragma omp parallel
  {
    double* h = (double*)malloc(sizeof(double) * dff);
#pragma omp for schedule(dynamic, 4)
    for (int64_t t = 0; t < (int64_t)T; ++t) {
      for (uint32_t i = 0; i < k; ++i) {
        const uint64_t c = (uint64_t)t * k + i;
        if (!keep[c]) continue;
        const uint32_t e = (uint32_t)expert[c];
        const float* xr = x + (uint64_t)t * d;
        const float* W1 = w1 + (uint64_t)e * dff * d;
        const float* W2 = w2 + (uint64_t)e * d * dff;
        for (uint32_t j = 0; j < dff; ++j) {
          double acc = 0.0;
          const float* wr = W1 + (uint64_t)j * d;
          for (uint32_t q = 0; q < d; ++q) acc += (double)xr[q] * (double)wr[q];
          acc += (double)b1[(uint64_t)e * dff + j];
          h[j] = rnd(gelu(acc), emulate_bf16); /* A = act(H) as stored */
        }
        const double g = gate[c];
        for (uint32_t o = 0; o < d; ++o) {
          double acc = 0.0;
          const float* wr = W2 + (uint64_t)o * dff;
          for (uint32_t j = 0; j < dff; ++j) acc += h[j] * (double)wr[j];
          acc += (double)b2[(uint64_t)e * d + o];
          y[(uint64_t)t * d + o] += g * rnd(acc, emulate_bf16); /* Y stored, then combined */
        }
      }
    }
    free(h);
  }
  return ORACLE_OK;
}

/* Backward of oracle_moe_forward given the routing it produced.
 *   dy[T,d]; d_aux = upstream gradient of l_aux.
 * Outputs (double): dx[T,d], dwg[E,d], dbg[E], dw1[E,dff,d], db1[E,dff],
 * dw2[E,d,dff], db2[E,d], dlogits[T,E].
 * Gate gradient (DESIGN.md Appendix A §10):
 *   dg_i = keep_i * <dy_t, Y_i>;  k=1: dlogit = dg1 * p1 * (onehot(e1) - p);
 *   k=2: with g1 = sigmoid(l_e1 - l_e2): dl_e1 = (dg1-dg2) g1 g2 = -dl_e2;
 *   aux: dl[t,:] += d_aux * p_t * (a - <p_t, a>), a_e = E*count1_e/T^2. */
int oracle_moe_backward(uint64_t T, uint32_t d, uint32_t dff, uint32_t E, uint32_t k, uint64_t C,
                        int emulate_bf16, const float* x, const float* wg, const float* bg,
                        const float* w1, const float* b1, const float* w2, const float* b2,
                        const float* logits, const int32_t* expert, const double* gate,
                        const uint8_t* keep, const int32_t* count1, const float* dy, double d_aux,
                        double* dx, double* dwg, double* dbg, double* dw1, double* db1,
                        double* dw2, double* db2, double* dlogits) {
  (void)C;
  (void)bg;
  (void)b2;
  const int B = emulate_bf16;
  memset(dx, 0, sizeof(double) * T * d);
  memset(dwg, 0, sizeof(double) * (uint64_t)E * d);
  memset(dbg, 0, sizeof(double) * E);
  memset(dw1, 0, sizeof(double) * (uint64_t)E * dff * d);
  memset(db1, 0, sizeof(double) * (uint64_t)E * dff);
  memset(dw2, 0, sizeof(double) * (uint64_t)E * d * dff);
  memset(db2, 0, sizeof(double) * (uint64_t)E * d);
  double* dgate = (double*)calloc(T * k, sizeof(double));

  /* Expert backward, parallel over experts (each thread owns dw1/dw2 of e). */
#pragma omp parallel
  {
    double* hpre = (double*)malloc(sizeof(double) * dff);
    double* act = (double*)malloc(sizeof(double) * dff);
    double* dyv = (double*)malloc(sizeof(double) * d);
    double* dh = (double*)malloc(sizeof(double) * dff);
#pragma omp for schedule(dynamic, 1)
    for (int64_t e = 0; e < (int64_t)E; ++e) {
      const float* W1 = w1 + (uint64_t)e * dff * d;
      const float* W2 = w2 + (uint64_t)e * d * dff;
      double* dW1 = dw1 + (uint64_t)e * dff * d;
      double* dW2 = dw2 + (uint64_t)e * d * dff;
      for (uint64_t c = 0; c < T * k; ++c) {
        if (!keep[c] || expert[c] != (int32_t)e) continue;
        const uint64_t t = c / k;
        const float* xr = x + t * d;
        for (uint32_t j = 0; j < dff; ++j) {
          double acc = 0.0;
          const float* wr = W1 + (uint64_t)j * d;
          for (uint32_t q = 0; q < d; ++q) acc += (double)xr[q] * (double)wr[q];
          acc += (double)b1[(uint64_t)e * dff + j];
          hpre[j] = acc;
          act[j] = rnd(gelu(acc), B);
        }
        /* Y (as stored) for dgate */
        double dg = 0.0;
        for (uint32_t o = 0; o < d; ++o) {
          double acc = 0.0;
          const float* wr = W2 + (uint64_t)o * dff;
          for (uint32_t j = 0; j < dff; ++j) acc += act[j] * (double)wr[j];
          acc += (double)b2[(uint64_t)e * d + o];
          dg += (double)dy[t * d + o] * rnd(acc, B);
        }
        dgate[c] = dg;
        const double g = gate[c];
        for (uint32_t o = 0; o < d; ++o) dyv[o] = rnd(g * (double)dy[t * d + o], B); /* dY stored */
        for (uint32_t o = 0; o < d; ++o) {
          db2[(uint64_t)e * d + o] += dyv[o];
          double* row = dW2 + (uint64_t)o * dff;
          for (uint32_t j = 0; j < dff; ++j) row[j] += dyv[o] * act[j];
        }
        for (uint32_t j = 0; j < dff; ++j) {
          double acc = 0.0;
          for (uint32_t o = 0; o < d; ++o) acc += dyv[o] * (double)W2[(uint64_t)o * dff + j];
          /* gelu'(h) as stored by the forward epilogue (rounded), then dH stored */
          dh[j] = rnd(acc * rnd(gelu_grad(hpre[j]), B), B);
          db1[(uint64_t)e * dff + j] += dh[j];
        }
        for (uint32_t j = 0; j < dff; ++j) {
          double* row = dW1 + (uint64_t)j * d;
          const double v = dh[j];
          for (uint32_t q = 0; q < d; ++q) row[q] += v * (double)xr[q];
        }
        /* dX_e = dH W1, stored then combined */
        for (uint32_t q = 0; q < d; ++q) {
          double acc = 0.0;
          for (uint32_t j = 0; j < dff; ++j) acc += dh[j] * (double)W1[(uint64_t)j * d + q];
          dyv[q] = rnd(acc, B);
        }
        /* accumulate into dx: tokens can hit two experts -> serialise */
#pragma omp critical
        for (uint32_t q = 0; q < d; ++q) dx[t * d + q] += dyv[q];
      }
    }
    free(hpre);
    free(act);
    free(dyv);
    free(dh);
  }

  /* routing backward */
  const double inv_t2 = T ? 1.0 / ((double)T * (double)T) : 0.0;
  double* p = (double*)malloc(sizeof(double) * E);
  for (uint64_t t = 0; t < T; ++t) {
    const float* L = logits + t * E;
    double m = -INFINITY;
    for (uint32_t e = 0; e < E; ++e)
      if (!isnan(L[e]) && (double)L[e] > m) m = (double)L[e];
    double z = 0.0;
    for (uint32_t e = 0; e < E; ++e) {
      p[e] = exp((double)L[e] - m);
      z += p[e];
    }
    double pa = 0.0;
    for (uint32_t e = 0; e < E; ++e) {
      p[e] /= z;
      pa += p[e] * (double)E * (double)count1[e] * inv_t2;
    }
    double* dl = dlogits + t * E;
    for (uint32_t e = 0; e < E; ++e)
      dl[e] = d_aux * p[e] * ((double)E * (double)count1[e] * inv_t2 - pa);
    if (k == 1) {
      const uint32_t e1 = (uint32_t)expert[t];
      const double dg = keep[t] ? dgate[t] : 0.0;
      for (uint32_t e = 0; e < E; ++e) dl[e] += dg * p[e1] * ((e == e1 ? 1.0 : 0.0) - p[e]);
    } else {
      const uint32_t e1 = (uint32_t)expert[2 * t], e2 = (uint32_t)expert[2 * t + 1];
      const double dg1 = keep[2 * t] ? dgate[2 * t] : 0.0;
      const double dg2 = keep[2 * t + 1] ? dgate[2 * t + 1] : 0.0;
      const double g1 = gate[2 * t], g2 = gate[2 * t + 1];
      const double v = (dg1 - dg2) * g1 * g2;
      dl[e1] += v;
      dl[e2] -= v;
    }
    for (uint32_t e = 0; e < E; ++e) {
      const double g = rnd(dl[e], B); /* dlogits stored bf16 for the gate GEMMs */
      dbg[e] += dl[e];
      const float* xr = x + t * d;
      double* row = dwg + (uint64_t)e * d;
      for (uint32_t q = 0; q < d; ++q) row[q] += g * (double)xr[q];
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < (int64_t)T; ++t) {
    const double* dl = dlogits + (uint64_t)t * E;
    for (uint32_t q = 0; q < d; ++q) {
      double acc = 0.0;
      for (uint32_t e = 0; e < E; ++e) acc += rnd(dl[e], B) * (double)wg[(uint64_t)e * d + q];
      dx[(uint64_t)t * d + q] += acc;
    }
  }
  free(p);
  free(dgate);
  return ORACLE_OK;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* torchrun exports OMP_NUM_THREADS=1 to every rank; the CPU arm resets it */
void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}
