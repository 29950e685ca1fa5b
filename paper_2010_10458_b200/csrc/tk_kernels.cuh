// tk_kernels.cuh — sm_100a kernels of the MSTopK + sparse-aggregation hot path.
//
// All kernels are HBM/L2-bandwidth bound streaming passes (no contraction, no tensor cores).
// Layout: the gradient is cut into TILE = 4096-element tiles (16 KB of fp32); a CTA of 256
// threads (8 warps) owns one tile; warp w owns the 512 contiguous elements [w*512, w*512+512)
// of its tile, as 4 chunks of 128 elements; in chunk c lane l holds elements 4l..4l+3 through
// one 128-bit load, so every warp-wide load is a fully coalesced 512-byte transaction.
//
// Citations: P:n = PAPER.md line n.  Q<n> = numbered reading in DESIGN.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tk {

constexpr int TILE = 4096;          // elements per tile (power of two: aligned pairwise subtrees, Q3)
constexpr int THREADS = 256;        // 8 warps
constexpr int WARPS = THREADS / 32;
constexpr int WARP_SPAN = TILE / WARPS;  // 512
constexpr int CHUNKS = WARP_SPAN / 128;  // 4
constexpr int TMAX = 15;            // max candidates per count pass (4 bisection levels)
constexpr int NMAX = 52;            // max MSTopK samplings (Q5)
constexpr uint32_t INF_BITS = 0x7F800000u;

// Device-resident MSTopK control block (Alg. 1 l.4-6 state + the trial log).
struct Ctrl {
  double abar;        // Alg. 1 l.2
  double U;           // (double) u, Alg. 1 l.3
  uint32_t umax_bits;
  uint32_t nonfinite;
  double lo, hi;      // Alg. 1's l, r
  uint32_t k1, k2;
  double thres1, thres2;
  uint32_t key1, key2;
  int32_t prov1, prov2;  // where the per-tile counts of key1/key2 live: pass*TMAX + slot, -1 unset
  uint32_t it;           // trials done
  uint32_t ncand;        // candidates of the pass about to run
  uint32_t cand_key[TMAX];
  uint32_t totals[TMAX];
  double cand_ratio[TMAX];
  double cand_t[TMAX];
  uint32_t ticket;
  uint32_t need;
  uint64_t len2;
  uint64_t rand;
  uint64_t step;
  double ratio_log[NMAX];
  double thres_log[NMAX];
  uint32_t key_log[NMAX];
  uint32_t nnz_log[NMAX];
};

struct SearchParams {
  uint64_t n;        // vector length MSTopK runs on (d, or d/n for HiTopKComm)
  uint64_t k;        // number of elements to select
  uint32_t ntiles;
  uint32_t n_iters;  // N
  uint32_t levels;   // bisection levels per count pass
  uint32_t rank;
  uint64_t seed;
  uint32_t rand_mode;
};

// ------------------------------------------------------------------------------------------
// SplitMix64 window hash (Q10), implemented independently of the oracle.
__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t magnitude_bits(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }

// threshold of a bisection ratio: thres = a-bar + ratio * (u - a-bar), fp64, three RN ops (Q4)
__device__ __forceinline__ double threshold_of(double abar, double U, double ratio) {
  return __dadd_rn(abar, __dmul_rn(ratio, __dsub_rn(U, abar)));
}
// smallest fp32 >= t, as bits: a >= t  <=>  bits(a) >= key for finite a >= 0 (Q4)
__device__ __forceinline__ uint32_t key_of(double t) {
  if (!(t > 0.0)) return 0u;
  return __float_as_uint(__double2float_ru(t));
}

// Candidates of one count pass: the 2^lev - 1 ratios of the next lev bisection levels below
// the current [lo, hi], in ascending order.  All ratios are dyadic with <= 52 significant bits,
// so lo + (hi-lo)*m/2^lev is exact and equals the sequential l + (r-l)/2 of Alg. 1 l.8 (Q5).
__device__ void make_candidates(Ctrl* c, int lev) {
  const int T = (1 << lev) - 1;
  const double w = __dsub_rn(c->hi, c->lo);
  const double inv = 1.0 / (double)(1 << lev);
  for (int m = 1; m <= T; ++m) {
    double ratio = __dadd_rn(c->lo, __dmul_rn(w, (double)m * inv));
    double t = threshold_of(c->abar, c->U, ratio);
    c->cand_ratio[m - 1] = ratio;
    c->cand_t[m - 1] = t;
    c->cand_key[m - 1] = key_of(t);
    c->totals[m - 1] = 0u;
  }
  c->ncand = (uint32_t)T;
}

// Replay lev levels of Alg. 1 l.8-23 over the candidates' exact counts (totals[]).
__device__ void replay_levels(Ctrl* c, const uint32_t* totals, int lev, int pass, uint64_t k) {
  int m = 1 << (lev - 1);
  int stepm = m >> 1;
  for (int l = 0; l < lev; ++l) {
    const int s = m - 1;
    const uint32_t nnz = totals[s];
    const double ratio = c->cand_ratio[s];
    const double t = c->cand_t[s];
    const uint32_t key = c->cand_key[s];
    const uint32_t it = c->it;
    c->ratio_log[it] = ratio;
    c->thres_log[it] = t;
    c->key_log[it] = key;
    c->nnz_log[it] = nnz;
    c->it = it + 1;
    if ((uint64_t)nnz <= k) {            // l.11
      c->hi = ratio;                     // l.12
      if (nnz > c->k1) {                 // l.13
        c->k1 = nnz; c->thres1 = t; c->key1 = key; c->prov1 = pass * TMAX + s;
      }
      m -= stepm;
    } else {                             // l.17
      c->lo = ratio;                     // l.18
      if (nnz < c->k2) {                 // l.19
        c->k2 = nnz; c->thres2 = t; c->key2 = key; c->prov2 = pass * TMAX + s;
      }
      m += stepm;
    }
    stepm >>= 1;
  }
}

// Alg. 1 l.27 window: R = len(iota2) - (k - k1) + 1 >= 1 (Q8, Q9); rand uniform on [0, R).
__device__ void finish_window(Ctrl* c, const SearchParams& sp) {
  const uint64_t k1 = c->k1;
  const uint64_t cnt2 = (c->prov2 >= 0) ? (uint64_t)c->k2 : sp.n;  // count(a >= thres2)
  const uint64_t len2 = cnt2 - k1;
  const uint64_t need = sp.k - k1;
  const uint64_t R = len2 - need + 1;
  c->len2 = len2;
  c->need = (uint32_t)need;
  uint64_t r = 0;
  if (sp.rand_mode == 0) {
    uint64_t h = sm64(sp.seed);
    h = sm64(h ^ c->step);
    h = sm64(h ^ (uint64_t)sp.rank);
    h = sm64(h ^ 0ull);
    r = __umul64hi(h, R);
  }
  c->rand = r;
}

// ------------------------------------------------------------------------------------------
// K1: error feedback + |acc| statistics (Alg. 1 l.1-3; EF per BASELINE north_star, Q14).
//   acc = fl32(g + r) written in place into r (EF = 1) or acc = g (EF = 0, nothing written).
//   Per tile: canonical fp64 pairwise sum of |acc| (aligned 4096-leaf subtree, Q3) and the max
//   of |acc| bits (max of non-negative floats == max of their bit patterns).
// HBM: 12 B/elem with EF (read g, read r, write acc), 4 B/elem without.
template <bool EF>
__global__ void __launch_bounds__(THREADS) k_ef_stats(const float* __restrict__ g, float* __restrict__ r,
                                                      uint64_t n, double* __restrict__ tile_sum,
                                                      uint32_t* __restrict__ tile_max) {
  __shared__ double s_sum[WARPS];
  __shared__ uint32_t s_max[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t tile_base = (uint64_t)blockIdx.x * TILE;
  const uint64_t wbase = tile_base + (uint64_t)warp * WARP_SPAN + 4 * lane;
  float4 acc[CHUNKS];
  if (tile_base + TILE <= n) {
    float4 gv[CHUNKS], rv[CHUNKS];
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) gv[c] = __ldcs(reinterpret_cast<const float4*>(g + wbase + c * 128));
    if (EF) {
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c) rv[c] = *reinterpret_cast<const float4*>(r + wbase + c * 128);
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c) {
        acc[c].x = __fadd_rn(gv[c].x, rv[c].x);
        acc[c].y = __fadd_rn(gv[c].y, rv[c].y);
        acc[c].z = __fadd_rn(gv[c].z, rv[c].z);
        acc[c].w = __fadd_rn(gv[c].w, rv[c].w);
        *reinterpret_cast<float4*>(r + wbase + c * 128) = acc[c];
      }
    } else {
#pragma unroll
      for (int c = 0; c < CHUNKS; ++c) acc[c] = gv[c];
    }
  } else {
#pragma unroll
    for (int c = 0; c < CHUNKS; ++c) {
      float v[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t i = wbase + c * 128 + e;
        float x = 0.0f;
        if (i < n) {
          x = g[i];
          if (EF) {
            x = __fadd_rn(x, r[i]);
            r[i] = x;
          }
        }
        v[e] = x;
      }
      acc[c] = make_float4(v[0], v[1], v[2], v[3]);
    }
  }
  // pairwise tree: 4 leaves per lane -> 128 per chunk (xor shuffles) -> 512 per warp -> 4096
  double cs[CHUNKS];
  uint32_t mx = 0;
#pragma unroll
  for (int c = 0; c < CHUNKS; ++c) {
    const uint32_t b0 = magnitude_bits(acc[c].x), b1 = magnitude_bits(acc[c].y);
    const uint32_t b2 = magnitude_bits(acc[c].z), b3 = magnitude_bits(acc[c].w);
    mx = max(mx, max(max(b0, b1), max(b2, b3)));
    double s = __dadd_rn(__dadd_rn((double)__uint_as_float(b0), (double)__uint_as_float(b1)),
                         __dadd_rn((double)__uint_as_float(b2), (double)__uint_as_float(b3)));
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
    cs[c] = s;
  }
  const double ws = __dadd_rn(__dadd_rn(cs[0], cs[1]), __dadd_rn(cs[2], cs[3]));
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    s_sum[warp] = ws;
    s_max[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double t = __dadd_rn(__dadd_rn(__dadd_rn(s_sum[0], s_sum[1]), __dadd_rn(s_sum[2], s_sum[3])),
                               __dadd_rn(__dadd_rn(s_sum[4], s_sum[5]), __dadd_rn(s_sum[6], s_sum[7])));
    uint32_t m = s_max[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) m = max(m, s_max[w]);
    tile_sum[blockIdx.x] = t;
    tile_max[blockIdx.x] = m;
  }
}

// K1f: finalize a-bar and u over the tile partials (one CTA of 1024 threads) and emit the first
// pass's candidate thresholds.  The tree over tiles is the canonical pairwise tree over
// L = max(next_pow2(ntiles), 1024) leaves (extra zero leaves never change a pairwise sum of
// non-negative values, so this equals PW over next_pow2(d) element leaves, Q3).
constexpr int FIN_THREADS = 1024;
__global__ void __launch_bounds__(FIN_THREADS) k_finalize(const double* __restrict__ tile_sum,
                                                          const uint32_t* __restrict__ tile_max,
                                                          Ctrl* __restrict__ c, SearchParams sp,
                                                          uint64_t step, int first_levels) {
  __shared__ double s_v[FIN_THREADS];
  __shared__ uint32_t s_m[32];
  const int tid = threadIdx.x;
  uint32_t L = 1024;
  while (L < sp.ntiles) L <<= 1;
  const uint32_t G = L / FIN_THREADS;  // leaves per thread (power of two)
  // in-thread canonical pairwise sum of leaves [tid*G, tid*G + G) with a binary-counter stack
  double stk[32];
  uint32_t mx = 0;
  for (uint32_t i = 0; i < G; ++i) {
    const uint32_t leaf = tid * G + i;
    double v = 0.0;
    if (leaf < sp.ntiles) {
      v = tile_sum[leaf];
      mx = max(mx, tile_max[leaf]);
    }
    int lvl = 0;
    uint32_t cnt = i;
    while (cnt & 1u) {
      v = __dadd_rn(stk[lvl], v);
      ++lvl;
      cnt >>= 1;
    }
    stk[lvl] = v;
  }
  int top = 0;
  while ((1u << top) < G) ++top;
  s_v[tid] = stk[top];
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((tid & 31) == 0) s_m[tid >> 5] = mx;
  __syncthreads();
  for (int s = FIN_THREADS / 2; s >= 1; s >>= 1) {
    double v = 0.0;
    if (tid < s) v = __dadd_rn(s_v[2 * tid], s_v[2 * tid + 1]);
    __syncthreads();
    if (tid < s) s_v[tid] = v;
    __syncthreads();
  }
  if (tid == 0) {
    uint32_t m = s_m[0];
    for (int w = 1; w < 32; ++w) m = max(m, s_m[w]);
    const double S = s_v[0];
    c->abar = __ddiv_rn(S, (double)sp.n);                 // Alg. 1 l.2
    c->umax_bits = m;                                     // Alg. 1 l.3
    c->U = (double)__uint_as_float(m);
    c->nonfinite = (m >= INF_BITS) ? 1u : 0u;
    c->lo = 0.0; c->hi = 1.0;                             // l.4
    c->k1 = 0u; c->k2 = (uint32_t)sp.n;                   // l.5
    c->thres1 = 0.0; c->thres2 = 0.0;                     // l.6
    c->key1 = INF_BITS; c->key2 = 0u;                     // Q8 / Q9 sentinels
    c->prov1 = -1; c->prov2 = -1;
    c->it = 0u;
    c->ticket = 0u;
    c->step = step;
    make_candidates(c, first_levels);
  }
}

// K2: count pass (Alg. 1 l.10) for T = 2^lev - 1 candidate thresholds at once (speculative
// bisection: lev levels per read of the data).  nnz_j = #{i : bits|acc_i| >= key_j}.
// Per-tile u16 counts are kept (the selection's prefix sums reuse them); the last CTA to finish
// replays the lev levels of Alg. 1 l.11-23 on the exact totals and emits the next candidates.
// HBM/L2: 4 B/elem.
template <int T>
__global__ void __launch_bounds__(THREADS) k_count(const float* __restrict__ acc, Ctrl* __restrict__ c,
                                                   SearchParams sp, uint16_t* __restrict__ tile_counts,
                                                   int pass, int lev, int next_lev) {
  __shared__ uint32_t s_cnt[WARPS][T];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t key[T];
#pragma unroll
  for (int s = 0; s < T; ++s) key[s] = (int32_t)c->cand_key[s];
  uint32_t cnt[T];
#pragma unroll
  for (int s = 0; s < T; ++s) cnt[s] = 0;
  const uint64_t tile_base = (uint64_t)blockIdx.x * TILE;
  const uint64_t wbase = tile_base + (uint64_t)warp * WARP_SPAN + 4 * lane;
  const uint32_t* a32 = reinterpret_cast<const uint32_t*>(acc);
  if (tile_base + TILE <= sp.n) {
    uint4 v[CHUNKS];
#pragma unroll
    for (int ch = 0; ch < CHUNKS; ++ch) v[ch] = *reinterpret_cast<const uint4*>(a32 + wbase + ch * 128);
#pragma unroll
    for (int ch = 0; ch < CHUNKS; ++ch) {
      const int32_t a0 = (int32_t)(v[ch].x & 0x7FFFFFFFu), a1 = (int32_t)(v[ch].y & 0x7FFFFFFFu);
      const int32_t a2 = (int32_t)(v[ch].z & 0x7FFFFFFFu), a3 = (int32_t)(v[ch].w & 0x7FFFFFFFu);
#pragma unroll
      for (int s = 0; s < T; ++s)
        cnt[s] += (uint32_t)(a0 >= key[s]) + (uint32_t)(a1 >= key[s]) + (uint32_t)(a2 >= key[s]) +
                  (uint32_t)(a3 >= key[s]);
    }
  } else {
#pragma unroll
    for (int ch = 0; ch < CHUNKS; ++ch) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint64_t i = wbase + ch * 128 + e;
        const int32_t a = (i < sp.n) ? (int32_t)(a32[i] & 0x7FFFFFFFu) : -1;  // padding never counts
#pragma unroll
        for (int s = 0; s < T; ++s) cnt[s] += (uint32_t)(a >= key[s]);
      }
    }
  }
#pragma unroll
  for (int s = 0; s < T; ++s) {
    const uint32_t w = __reduce_add_sync(0xffffffffu, cnt[s]);
    if (lane == 0) s_cnt[warp][s] = w;
  }
  __syncthreads();
  if (threadIdx.x < T) {
    const int s = threadIdx.x;
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) tot += s_cnt[w][s];
    tile_counts[(size_t)(pass * TMAX + s) * sp.ntiles + blockIdx.x] = (uint16_t)tot;
    atomicAdd(&c->totals[s], tot);
  }
  // last-CTA-done ticket: the controller runs once all counts are in
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t prev = atomicAdd(&c->ticket, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    // read the totals through L2 (volatile: the CTA's L1 may hold the line from the key load)
    volatile uint32_t* tv = c->totals;
    uint32_t tot[T];
#pragma unroll
    for (int s = 0; s < T; ++s) tot[s] = tv[s];
    replay_levels(c, tot, lev, pass, sp.k);
    c->ticket = 0u;
    if (next_lev > 0) {
      make_candidates(c, next_lev);
    } else {
      finish_window(c, sp);
    }
  }
}

// K3: exclusive prefix over tiles of the class-1 (a >= thres1) and class-2 (thres2 <= a < thres1)
// counts, read back from the saved per-tile counts of the trials that set thres1 / thres2.
constexpr int SCAN_THREADS = 1024;
__global__ void __launch_bounds__(SCAN_THREADS) k_scan(const Ctrl* __restrict__ c, SearchParams sp,
                                                       const uint16_t* __restrict__ tile_counts,
                                                       uint32_t* __restrict__ pre1, uint32_t* __restrict__ pre2) {
  __shared__ uint32_t s1[SCAN_THREADS], s2[SCAN_THREADS];
  const int tid = threadIdx.x;
  const int32_t p1 = c->prov1, p2 = c->prov2;
  const uint32_t nt = sp.ntiles;
  const uint32_t per = (nt + SCAN_THREADS - 1) / SCAN_THREADS;
  const uint32_t b = tid * per, e = min(nt, b + per);
  auto tile_valid = [&](uint32_t t) -> uint32_t {
    const uint64_t lo = (uint64_t)t * TILE;
    const uint64_t hi = min(sp.n, lo + TILE);
    return (uint32_t)(hi - lo);
  };
  uint32_t a1 = 0, a2 = 0;
  for (uint32_t t = b; t < e; ++t) {
    const uint32_t c1 = (p1 >= 0) ? tile_counts[(size_t)p1 * nt + t] : 0u;
    const uint32_t call = (p2 >= 0) ? tile_counts[(size_t)p2 * nt + t] : tile_valid(t);
    a1 += c1;
    a2 += call - c1;
  }
  s1[tid] = a1;
  s2[tid] = a2;
  __syncthreads();
  // Hillis-Steele inclusive scan over thread totals
  for (int off = 1; off < SCAN_THREADS; off <<= 1) {
    uint32_t v1 = 0, v2 = 0;
    if (tid >= off) { v1 = s1[tid - off]; v2 = s2[tid - off]; }
    __syncthreads();
    s1[tid] += v1;
    s2[tid] += v2;
    __syncthreads();
  }
  uint32_t r1 = s1[tid] - a1, r2 = s2[tid] - a2;
  for (uint32_t t = b; t < e; ++t) {
    const uint32_t c1 = (p1 >= 0) ? tile_counts[(size_t)p1 * nt + t] : 0u;
    const uint32_t call = (p2 >= 0) ? tile_counts[(size_t)p2 * nt + t] : tile_valid(t);
    pre1[t] = r1;
    pre2[t] = r2;
    r1 += c1;
    r2 += call - c1;
  }
}

// K4: stable ascending-index compaction (Alg. 1 l.25-29, Q11) with fused residual write-back.
//   class 1: bits >= key1 (iota1; empty when k1 == 0, Q8)
//   class 2: key2 <= bits < key1 (iota2); the window keeps class-2 ranks [rand, rand + k - k1)
//   output position of a kept element i = #class1 before i + clamp(#class2 before i - rand, 0, need)
// Warp ballots + popc give in-warp ranks; warp totals are scanned through shared memory.
// HBM/L2: 4 B/elem read + 8 B per selected pair + one 4-byte residual zero per selected pair.
__global__ void __launch_bounds__(THREADS) k_select(const float* __restrict__ acc, const Ctrl* __restrict__ c,
                                                    SearchParams sp, const uint32_t* __restrict__ pre1,
                                                    const uint32_t* __restrict__ pre2, uint32_t* __restrict__ idx_out,
                                                    float* __restrict__ val_out, float* __restrict__ r_zero) {
  __shared__ uint32_t s_w1[WARPS], s_w2[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t key1 = (c->prov1 >= 0) ? (int32_t)c->key1 : (int32_t)INF_BITS;
  const int32_t key2 = (c->prov2 >= 0) ? (int32_t)c->key2 : 0;
  const uint32_t rnd = (uint32_t)c->rand, need = c->need;
  const uint64_t tile_base = (uint64_t)blockIdx.x * TILE;
  const uint64_t wbase = tile_base + (uint64_t)warp * WARP_SPAN + 4 * lane;
  const uint32_t* a32 = reinterpret_cast<const uint32_t*>(acc);
  uint4 v[CHUNKS];
  if (tile_base + TILE <= sp.n) {
#pragma unroll
    for (int ch = 0; ch < CHUNKS; ++ch) v[ch] = *reinterpret_cast<const uint4*>(a32 + wbase + ch * 128);
  } else {
#pragma unroll
    for (int ch = 0; ch < CHUNKS; ++ch) {
      const uint64_t i = wbase + ch * 128;
      // padding (i >= n) is excluded by the explicit validity test below
      v[ch].x = (i + 0 < sp.n) ? a32[i + 0] : 0u;
      v[ch].y = (i + 1 < sp.n) ? a32[i + 1] : 0u;
      v[ch].z = (i + 2 < sp.n) ? a32[i + 2] : 0u;
      v[ch].w = (i + 3 < sp.n) ? a32[i + 3] : 0u;
    }
  }
  // class flags per element, packed: bit e = class-1 flag of element e, bit 4+e = class-2 flag
  uint32_t flags[CHUNKS];
  uint32_t n1 = 0, n2 = 0;
#pragma unroll
  for (int ch = 0; ch < CHUNKS; ++ch) {
    uint32_t f = 0;
    const uint32_t w4[4] = {v[ch].x, v[ch].y, v[ch].z, v[ch].w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint64_t i = wbase + ch * 128 + e;
      const int32_t a = (int32_t)(w4[e] & 0x7FFFFFFFu);
      const bool valid = i < sp.n;
      const bool f1 = valid && (a >= key1);
      const bool f2 = valid && !f1 && (a >= key2);
      f |= ((uint32_t)f1 << e) | ((uint32_t)f2 << (4 + e));
    }
    flags[ch] = f;
    n1 += __popc(f & 0xFu);
    n2 += __popc(f >> 4);
  }
  const uint32_t wn1 = __reduce_add_sync(0xffffffffu, n1);
  const uint32_t wn2 = __reduce_add_sync(0xffffffffu, n2);
  if (lane == 0) {
    s_w1[warp] = wn1;
    s_w2[warp] = wn2;
  }
  __syncthreads();
  uint32_t b1 = pre1[blockIdx.x], b2 = pre2[blockIdx.x];
  for (int w = 0; w < warp; ++w) {
    b1 += s_w1[w];
    b2 += s_w2[w];
  }
  if (wn1 == 0 && (wn2 == 0 || b2 >= rnd + need || b2 + wn2 <= rnd)) {
    // nothing of this warp can be selected: no class-1 element, and its class-2 ranks miss the window
    return;
  }
#pragma unroll
  for (int ch = 0; ch < CHUNKS; ++ch) {
    const uint32_t f = flags[ch];
    const uint32_t l1 = __popc(f & 0xFu), l2 = __popc(f >> 4);
    // warp exclusive scan of (l1, l2) packed in 16-bit halves (each <= 128)
    uint32_t packed = l1 | (l2 << 16);
    uint32_t incl = packed;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += o;
    }
    const uint32_t excl = incl - packed;
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t c1 = b1 + (excl & 0xFFFFu);
    uint32_t c2 = b2 + (excl >> 16);
    if (f) {
      const uint32_t w4[4] = {v[ch].x, v[ch].y, v[ch].z, v[ch].w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t i = (uint32_t)(wbase + ch * 128 + e);
        if (f & (1u << e)) {
          const uint32_t after = (c2 > rnd) ? min(c2 - rnd, need) : 0u;
          const uint32_t pos = c1 + after;
          idx_out[pos] = i;
          val_out[pos] = __uint_as_float(w4[e]);
          if (r_zero) r_zero[i] = 0.0f;
          ++c1;
        } else if (f & (1u << (4 + e))) {
          if (c2 >= rnd && c2 < rnd + need) {
            const uint32_t pos = c1 + (c2 - rnd);
            idx_out[pos] = i;
            val_out[pos] = __uint_as_float(w4[e]);
            if (r_zero) r_zero[i] = 0.0f;
          }
          ++c2;
        }
      }
    }
    b1 += tot & 0xFFFFu;
    b2 += tot >> 16;
  }
}

// ------------------------------------------------------------------------------------------
// Decompression (Alg. 2 l.15-20): out = +0; for p in rank order: out[idx_p] += val_p (fp32 RN).
// Tile-owner design: CTA t owns out[t*TILE, (t+1)*TILE) in shared memory, applies the ranks'
// pairs that fall in its tile in rank order (barrier between ranks; indices within one rank are
// distinct so one rank's adds never collide), then writes the tile once, coalesced.  No global
// atomics, no read-modify-write of out: HBM 4 B/elem write + 8 B per gathered pair.

// tile_ranges: start[p][t] = first j with idx_p[j] >= t*TILE (lower bound), t in [0, ntiles].
__global__ void k_tile_ranges(const uint32_t* __restrict__ gathered, uint32_t nchunks, uint64_t k, uint64_t n,
                              uint32_t ntiles, uint32_t* __restrict__ starts) {
  const uint64_t tot = (uint64_t)nchunks * (k + 1);
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < tot; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = (uint32_t)(g / (k + 1));
    const uint64_t j = g % (k + 1);
    const uint32_t* idx = gathered + (size_t)p * 2 * k;
    const uint32_t tj = (j < k) ? min((uint32_t)(idx[j] / TILE), ntiles) : ntiles;
    const int64_t tp = (j > 0) ? (int64_t)min((uint32_t)(idx[j - 1] / TILE), ntiles) : -1;
    for (int64_t t = tp + 1; t <= (int64_t)tj; ++t) starts[(size_t)p * (ntiles + 1) + t] = (uint32_t)j;
  }
  (void)n;
}

__global__ void __launch_bounds__(THREADS) k_decompress(const uint32_t* __restrict__ gathered, uint32_t nchunks,
                                                        uint64_t k, uint64_t n, uint32_t ntiles,
                                                        const uint32_t* __restrict__ starts, float* __restrict__ out) {
  __shared__ __align__(16) float s_tile[TILE];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t t = blockIdx.x;
  const uint64_t lo = (uint64_t)t * TILE;
  // prefetch up to 32 pairs of rank p = warp (the common case: ~rho*TILE pairs per rank per tile)
  uint32_t pre_i = 0xFFFFFFFFu;
  float pre_v = 0.0f;
  uint32_t my_s = 0, my_e = 0;
  if (warp < (int)nchunks) {
    const uint32_t* st = starts + (size_t)warp * (ntiles + 1);
    my_s = st[t];
    my_e = st[t + 1];
    if (my_e < my_s) my_e = my_s;
    const uint32_t j = my_s + lane;
    if (j < my_e) {
      const uint32_t* ch = gathered + (size_t)warp * 2 * k;
      pre_i = ch[j];
      pre_v = __uint_as_float(ch[k + j]);
    }
  }
  float4* s4 = reinterpret_cast<float4*>(s_tile);
  for (int q = threadIdx.x; q < TILE / 4; q += THREADS) s4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  for (uint32_t p = 0; p < nchunks; ++p) {
    if (p < WARPS) {
      if (warp == (int)p) {
        if (pre_i != 0xFFFFFFFFu && pre_i >= lo && pre_i - lo < TILE)
          s_tile[pre_i - lo] = __fadd_rn(s_tile[pre_i - lo], pre_v);
        const uint32_t* ch = gathered + (size_t)p * 2 * k;
        for (uint32_t j = my_s + 32 + lane; j < my_e; j += 32) {
          const uint32_t i = ch[j];
          if (i >= lo && i - lo < TILE) s_tile[i - lo] = __fadd_rn(s_tile[i - lo], __uint_as_float(ch[k + j]));
        }
      }
    } else {
      const uint32_t* st = starts + (size_t)p * (ntiles + 1);
      const uint32_t s = st[t];
      uint32_t e = st[t + 1];
      if (e < s) e = s;
      const uint32_t* ch = gathered + (size_t)p * 2 * k;
      for (uint32_t j = s + threadIdx.x; j < e; j += THREADS) {
        const uint32_t i = ch[j];
        if (i >= lo && i - lo < TILE) s_tile[i - lo] = __fadd_rn(s_tile[i - lo], __uint_as_float(ch[k + j]));
      }
    }
    __syncthreads();
  }
  if (lo + TILE <= n) {
    for (int q = threadIdx.x; q < TILE / 4; q += THREADS) __stcs(reinterpret_cast<float4*>(out + lo) + q, s4[q]);
  } else {
    for (int q = threadIdx.x; q < TILE; q += THREADS)
      if (lo + q < n) out[lo + q] = s_tile[q];
  }
}

}  // namespace tk
