// tk_kernels.cuh — sm_100a kernels of the MSTopK + sparse-aggregation hot path.
//
// All kernels are HBM/L2-bandwidth bound streaming passes (no contraction, so no tensor cores).
// They are persistent: the grid is (#SMs x resident CTAs), every warp works independently on
// its own contiguous work unit with fully coalesced 128-bit loads (lane l of a warp holds
// elements 4l..4l+3 of each 128-element chunk), and block barriers appear only where a result
// needs the whole CTA.  The last CTA to finish a pass (ticket) runs the scalar control of
// Alg. 1 on the device, so an iteration never returns to the host.
//
// Citations: P:n = PAPER.md line n.  Q<n> = numbered reading in DESIGN.md.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tk {

constexpr int TILE = 4096;          // elements per pairwise-sum tile (power of two, Q3) / output tile
constexpr int THREADS = 256;        // 8 warps per CTA
constexpr int WARPS = THREADS / 32;
constexpr int ROUND = 512;          // elements one warp touches per round (4 chunks of 128)
constexpr int TMAX = 15;            // max candidates per count pass (4 bisection levels)
constexpr int NMAX = 52;            // max MSTopK samplings (Q5)
constexpr uint32_t INF_BITS = 0x7F800000u;
constexpr uint32_t NO_INDEX = 0xFFFFFFFFu;

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
  int32_t prov1, prov2;  // slot (pass*TMAX + candidate) whose per-warp counts are key1's / key2's; -1 unset
  uint32_t it;           // trials done
  uint32_t ncand;        // candidates of the pass about to run
  uint32_t cand_key[16];
  uint32_t totals[16];
  double cand_ratio[16];
  double cand_t[16];
  uint32_t ticket;
  uint32_t cap_ok;       // 1: passes >= 1 and the selection run on the compacted entries (see k_count)
  uint32_t cmp_key;      // key above which the first count pass compacts elements
  double cmp_ratio;      // its bisection ratio
  double prev_lo;        // final l of the previous compression (predicts the bracket; perf only)
  uint32_t overflow;     // set by a warp whose compacted entries exceeded the capacity
  uint32_t need;
  uint64_t len2;
  uint64_t rand;
  uint64_t step;
  double ratio_log[NMAX];
  double thres_log[NMAX];
  uint32_t key_log[NMAX];
  uint32_t nnz_log[NMAX];
};

// Per-launch parameters of the MSTopK kernels.  The count and selection kernels share one
// partition of [0, n) into W contiguous warp slabs of S elements (S a multiple of ROUND).
struct SearchParams {
  uint64_t n;        // vector length MSTopK runs on (d, or d/n for HiTopKComm)
  uint64_t k;        // number of elements to select
  uint32_t W;        // warp slabs (= gridDim.x * WARPS of the count / select launches)
  uint64_t S;        // slab length
  uint32_t rank;
  uint32_t rand_mode;
  uint64_t seed;
};

// Compacted entries of the first count pass: warp w keeps, in ascending index order, every
// element of its slab with |acc| >= the pass's lowest candidate key (idx[w*C + j], bits[w*C + j],
// j < cnt[w]).  When the bisection's bracket after that pass lies above that key, no later trial
// threshold and no selected element can lie below it, so the later passes and the selection read
// only these entries instead of the whole vector (exact: same counts, same sets).
struct Compact {
  uint32_t* idx;
  uint32_t* bits;
  uint32_t* cnt;
  uint32_t C;  // capacity per warp (multiple of 4)
};

// ------------------------------------------------------------------------------------------
// scalar control (runs in one thread of the last CTA of a pass)

// SplitMix64 finaliser chain (Q10), implemented independently of the oracle.
__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// thres = a-bar + ratio * (u - a-bar): fp64, three separate round-to-nearest ops (Alg. 1 l.9, Q4)
__device__ __forceinline__ double threshold_of(double abar, double U, double ratio) {
  return __dadd_rn(abar, __dmul_rn(ratio, __dsub_rn(U, abar)));
}
// smallest fp32 >= t, as bits: a >= t  <=>  bits(a) >= key for finite a >= 0 (Q4)
__device__ __forceinline__ uint32_t key_of(double t) {
  if (!(t > 0.0)) return 0u;
  return __float_as_uint(__double2float_ru(t));
}

// Candidates of one count pass: the 2^lev - 1 ratios of the next lev bisection levels below the
// current [lo, hi], ascending.  Every ratio is dyadic with <= 52 significant bits, so
// lo + (hi-lo)*m/2^lev is exact and equals the sequential l + (r-l)/2 of Alg. 1 l.8 (Q5).
__device__ void make_candidates(Ctrl* c, int lev) {
  const int T = (1 << lev) - 1;
  const double w = __dsub_rn(c->hi, c->lo);
  const double inv = ldexp(1.0, -lev);
  for (int m = 1; m <= T; ++m) {
    const double ratio = __dadd_rn(c->lo, __dmul_rn(w, (double)m * inv));
    const double t = threshold_of(c->abar, c->U, ratio);
    c->cand_ratio[m - 1] = ratio;
    c->cand_t[m - 1] = t;
    c->cand_key[m - 1] = key_of(t);
    c->totals[m - 1] = 0u;
  }
  c->ncand = (uint32_t)T;
}

// Replay lev levels of Alg. 1 l.8-23 on the candidates' exact counts.
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

// last-CTA-done ticket: true in every thread of the CTA that finished last (resets the ticket)
__device__ __forceinline__ bool last_cta(uint32_t* ticket) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// The last CTA runs the scalar control on a shared-memory copy of the control block (one
// coalesced load and store by the whole CTA instead of a chain of dependent global accesses).
__device__ __forceinline__ void ctrl_to_smem(Ctrl* s, const Ctrl* g) {
  static_assert(sizeof(Ctrl) % 4 == 0, "Ctrl must be a whole number of words");
  for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(s)[i] = __ldcg(reinterpret_cast<const uint32_t*>(g) + i);
  __syncthreads();
}
__device__ __forceinline__ void ctrl_to_global(Ctrl* g, const Ctrl* s) {
  __syncthreads();
  for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(g)[i] = reinterpret_cast<const uint32_t*>(s)[i];
}

// block-wide exclusive scan of one u32 per thread (THREADS threads); returns the block total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* s_warp, uint32_t& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += o;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t base = 0;
  total = 0;
#pragma unroll
  for (int w = 0; w < WARPS; ++w) {
    const uint32_t x = s_warp[w];
    if (w < warp) base += x;
    total += x;
  }
  __syncthreads();
  return base + incl - v;
}

// ------------------------------------------------------------------------------------------
// K1: error feedback + |acc| statistics (Alg. 1 l.1-3; EF per BASELINE north_star, Q14).
//   acc = fl32(g + r) written in place into r (EF) or acc = g (no EF, nothing written).
//   The canonical fp64 pairwise tree of |acc| (Q3) is built bottom-up with no global atomics
//   inside the stream: a 512-element unit is one warp round (lane: 4 leaves; xor-shuffle tree:
//   128-leaf chunks; chunks: 512), each warp owns an aligned power-of-two run of units and folds
//   them with a binary-counter stack, each CTA owns an aligned power-of-two run of warps' runs
//   (tree over its 8 warps), and the last CTA folds the CTA partials (zero-padded to a power of
//   two, Q3) into a-bar, u and the first pass's candidate thresholds.
// HBM: 12 B/elem with EF (read g, read r, write acc), 4 B/elem without.
__device__ __forceinline__ double lane_quad_sum(float4 v) {
  return __dadd_rn(__dadd_rn((double)fabsf(v.x), (double)fabsf(v.y)),
                   __dadd_rn((double)fabsf(v.z), (double)fabsf(v.w)));
}
__device__ __forceinline__ uint32_t quad_max_bits(float4 v) {
  const uint32_t a = __float_as_uint(v.x) & 0x7FFFFFFFu, b = __float_as_uint(v.y) & 0x7FFFFFFFu;
  const uint32_t c = __float_as_uint(v.z) & 0x7FFFFFFFu, d = __float_as_uint(v.w) & 0x7FFFFFFFu;
  return max(max(a, b), max(c, d));
}

__device__ void stats_finalize(Ctrl* c, const SearchParams& sp, double S, uint32_t m, uint64_t step,
                               int first_levels) {
  c->prev_lo = c->lo;
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
  c->step = step;
  make_candidates(c, first_levels);
  // compaction key of the first count pass: the highest of its candidates at or below the
  // bracket the previous compression ended in (any choice is exact; a good one keeps few elements)
  int ms = 0;
  for (int q = 1; q < (int)c->ncand; ++q)
    if (c->cand_ratio[q] <= c->prev_lo) ms = q;
  c->cmp_key = c->cand_key[ms];
  c->cmp_ratio = c->cand_ratio[ms];
}

// HiTopKComm step 1 fused into K1 (Eq. 4; reading Q20): with NP > 0 the gradient of
// this GPU's segment is the ordered reduce-scatter sum_{q=0..NP-1} g_q[segment], read directly
// from the row peers' memory (CUDA IPC peer pointers over NVLink) and added in ascending row rank,
// left to right, in fp32 round-to-nearest - bit-exact, unlike a reduce-scatter whose order the
// library chooses.
struct Peers {
  const float* p[8];  // row peers' gradient + segment offset, in row-rank order
};

template <int NP>
__device__ __forceinline__ void load_g(const float* g, const Peers& pr, uint64_t base, float4* gv) {
  if (NP == 0) {
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) gv[ch] = __ldcs(reinterpret_cast<const float4*>(g + base + ch * 128));
  } else {
    float4 pv[NP > 0 ? NP : 1][4];
#pragma unroll
    for (int q = 0; q < NP; ++q)
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) pv[q][ch] = __ldcs(reinterpret_cast<const float4*>(pr.p[q] + base + ch * 128));
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      float4 a = pv[0][ch];
#pragma unroll
      for (int q = 1; q < NP; ++q)
        a = make_float4(__fadd_rn(a.x, pv[q][ch].x), __fadd_rn(a.y, pv[q][ch].y), __fadd_rn(a.z, pv[q][ch].z),
                        __fadd_rn(a.w, pv[q][ch].w));
      gv[ch] = a;
    }
  }
}
template <int NP>
__device__ __forceinline__ float load_g1(const float* g, const Peers& pr, uint64_t i) {
  if (NP == 0) return g[i];
  float a = pr.p[0][i];
#pragma unroll
  for (int q = 1; q < NP; ++q) a = __fadd_rn(a, pr.p[q][i]);
  return a;
}

template <bool EF, int NP>
__device__ __forceinline__ void ef_load(const float* g, const Peers& pr, const float* r, uint64_t base, float4* gv,
                                        float4* rv) {
  load_g<NP>(g, pr, base, gv);
  if (EF) {
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) rv[ch] = __ldcs(reinterpret_cast<const float4*>(r + base + ch * 128));
  }
}

template <bool EF, int NP>
__global__ void __launch_bounds__(THREADS, 4) k_ef_stats(const float* __restrict__ g, Peers pr, float* __restrict__ r,
                                                         SearchParams sp, uint32_t units_per_warp,
                                                         double* __restrict__ cta_sum, uint32_t* __restrict__ cta_max,
                                                         Ctrl* __restrict__ c, uint64_t step, int first_levels) {
  __shared__ double s_ws[WARPS];
  __shared__ uint32_t s_wm[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n = sp.n;
  const uint64_t u0 = ((uint64_t)blockIdx.x * WARPS + warp) * units_per_warp;
  double stk[24];
  uint32_t mx = 0;
  for (uint32_t i = 0; i < units_per_warp; ++i) {
    const uint64_t u = u0 + i;
    const uint64_t base = u * ROUND + 4 * lane;
    float4 acc[4];
    if ((u + 1) * ROUND <= n) {
      float4 rv[4];
      ef_load<EF, NP>(g, pr, r, base, acc, rv);
      if (EF) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          acc[ch] = make_float4(__fadd_rn(acc[ch].x, rv[ch].x), __fadd_rn(acc[ch].y, rv[ch].y),
                                __fadd_rn(acc[ch].z, rv[ch].z), __fadd_rn(acc[ch].w, rv[ch].w));
          *reinterpret_cast<float4*>(r + base + ch * 128) = acc[ch];
        }
      }
    } else {
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        float v[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint64_t idx = base + ch * 128 + e;
          float x = 0.0f;  // zero leaves beyond n (padding of the canonical tree)
          if (idx < n) {
            x = load_g1<NP>(g, pr, idx);
            if (EF) {
              x = __fadd_rn(x, r[idx]);
              r[idx] = x;
            }
          }
          v[e] = x;
        }
        acc[ch] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
    double cs[4];
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      mx = max(mx, quad_max_bits(acc[ch]));
      double s = lane_quad_sum(acc[ch]);
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
      cs[ch] = s;
    }
    double v = __dadd_rn(__dadd_rn(cs[0], cs[1]), __dadd_rn(cs[2], cs[3]));  // 512-leaf subtree
    int lvl = 0;
    for (uint32_t cnt = i; cnt & 1u; cnt >>= 1) v = __dadd_rn(stk[lvl++], v);  // binary-counter stack
    stk[lvl] = v;
  }
  int top = 0;
  while ((1u << top) < units_per_warp) ++top;
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    s_ws[warp] = stk[top];
    s_wm[warp] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cta_sum[blockIdx.x] = __dadd_rn(__dadd_rn(__dadd_rn(s_ws[0], s_ws[1]), __dadd_rn(s_ws[2], s_ws[3])),
                                    __dadd_rn(__dadd_rn(s_ws[4], s_ws[5]), __dadd_rn(s_ws[6], s_ws[7])));
    uint32_t m = s_wm[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) m = max(m, s_wm[w]);
    cta_max[blockIdx.x] = m;
  }
  if (!last_cta(&c->ticket)) return;
  // ---- last CTA: canonical tree over the CTA partials, zero-padded to Lp = 2^j >= THREADS ----
  __shared__ double s_v[THREADS];
  __shared__ uint32_t s_m[WARPS];
  const int tid = threadIdx.x;
  uint32_t Lp = THREADS;
  while (Lp < gridDim.x) Lp <<= 1;
  const uint32_t G = Lp / THREADS;  // <= 8 for grids up to 2048 CTAs
  double leaf[8];
  uint32_t m2 = 0;
#pragma unroll
  for (uint32_t q = 0; q < 8; ++q) {
    const uint32_t li = tid * G + q;
    leaf[q] = 0.0;
    if (q < G && li < gridDim.x) {
      leaf[q] = __ldcg(cta_sum + li);
      m2 = max(m2, __ldcg(cta_max + li));
    }
  }
  double st2[4];
#pragma unroll
  for (uint32_t q = 0; q < 8; ++q) {
    if (q < G) {
      double v = leaf[q];
      int lvl = 0;
      for (uint32_t cnt = q; cnt & 1u; cnt >>= 1) v = __dadd_rn(st2[lvl++], v);
      st2[lvl] = v;
    }
  }
  int top2 = 0;
  while ((1u << top2) < G) ++top2;
  s_v[tid] = st2[top2];
  m2 = __reduce_max_sync(0xffffffffu, m2);
  if (lane == 0) s_m[warp] = m2;
  __syncthreads();
  for (int h = THREADS / 2; h >= 1; h >>= 1) {
    double v = 0.0;
    if (tid < h) v = __dadd_rn(s_v[2 * tid], s_v[2 * tid + 1]);
    __syncthreads();
    if (tid < h) s_v[tid] = v;
    __syncthreads();
  }
  __shared__ Ctrl sc;
  ctrl_to_smem(&sc, c);
  if (tid == 0) {
    uint32_t m = s_m[0];
    for (int w = 1; w < WARPS; ++w) m = max(m, s_m[w]);
    sc.ticket = 0u;
    stats_finalize(&sc, sp, s_v[0], m, step, first_levels);
  }
  ctrl_to_global(c, &sc);
}

// ------------------------------------------------------------------------------------------
// K2: count pass (Alg. 1 l.10) resolving LEV bisection levels per read of the data: the
// T = 2^LEV - 1 candidate keys are sorted, so each element's bucket b = #{s : key_s <= bits}
// is found by a LEV-step binary search, and buckets are counted in packed 8-bit fields of a
// 64-bit register (flushed every 15 rounds).  nnz_s = sum_{b > s} bucket_b exactly.
// Per-warp-slab counts are kept (the selection's prefix sums reuse them); the last CTA replays
// the LEV levels of Alg. 1 l.11-23 and emits the next candidates, or after the last pass
// computes the window (l.27) and the slab prefix sums of the two selection classes.
// HBM/L2: 4 B/elem.
template <int LEV>
__device__ __forceinline__ uint32_t bucket_of(int32_t a, int32_t root, const int32_t* s_key) {
  uint32_t b = (a >= root) ? (1u << (LEV - 1)) : 0u;
#pragma unroll
  for (int l = LEV - 2; l >= 0; --l) {
    const int32_t kk = s_key[b + (1u << l) - 1];
    b += (a >= kk) ? (1u << l) : 0u;
  }
  return b;
}

// Exclusive prefix over the W warp slabs of the class-1 (a >= thres1) and class-2
// (thres2 <= a < thres1) counts, taken from the per-slab counts of the trials that set thres1 /
// thres2.  Chunks of 8*THREADS slabs are staged through shared memory with coalesced loads.
__device__ __noinline__ void scan_slabs(const Ctrl* c, const SearchParams& sp, const uint32_t* __restrict__ wcnt,
                                        uint32_t* __restrict__ pre1, uint32_t* __restrict__ pre2) {
  constexpr int PER = 8;
  constexpr int CH = PER * THREADS;
  __shared__ uint32_t s_c1[CH], s_ca[CH];
  __shared__ uint32_t s_w[2][WARPS];
  const int32_t p1 = c->prov1, p2 = c->prov2;
  const uint32_t W = sp.W;
  uint32_t carry1 = 0, carry2 = 0;
  for (uint32_t c0 = 0; c0 < W; c0 += CH) {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const uint32_t w = c0 + i * THREADS + threadIdx.x;
      uint32_t x1 = 0u, xa = 0u;
      if (w < W) {
        if (p1 >= 0) x1 = __ldcg(wcnt + (size_t)p1 * W + w);
        if (p2 >= 0) {
          xa = __ldcg(wcnt + (size_t)p2 * W + w);
        } else {
          const uint64_t lo = min(sp.n, (uint64_t)w * sp.S);
          xa = (uint32_t)(min(sp.n, lo + sp.S) - lo);
        }
      }
      s_c1[i * THREADS + threadIdx.x] = x1;
      s_ca[i * THREADS + threadIdx.x] = xa;
    }
    __syncthreads();
    uint32_t a1 = 0, a2 = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const uint32_t x1 = s_c1[threadIdx.x * PER + i];
      a1 += x1;
      a2 += s_ca[threadIdx.x * PER + i] - x1;
    }
    uint32_t t1, t2;
    uint32_t r1 = carry1 + block_excl_scan(a1, s_w[0], t1);
    uint32_t r2 = carry2 + block_excl_scan(a2, s_w[1], t2);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const uint32_t w = c0 + threadIdx.x * PER + i;
      const uint32_t x1 = s_c1[threadIdx.x * PER + i];
      const uint32_t x2 = s_ca[threadIdx.x * PER + i] - x1;
      if (w < W) {
        pre1[w] = r1;
        pre2[w] = r2;
      }
      r1 += x1;
      r2 += x2;
    }
    carry1 += t1;
    carry2 += t2;
    __syncthreads();
  }
}

template <int LEV, bool FIRST>
__global__ void __launch_bounds__(THREADS, 3) k_count(const float* __restrict__ acc, Ctrl* __restrict__ c,
                                                      SearchParams sp, uint32_t* __restrict__ wcnt,
                                                      uint32_t* __restrict__ pre1, uint32_t* __restrict__ pre2,
                                                      Compact cp, int pass, int next_lev) {
  constexpr int T = (1 << LEV) - 1;
  constexpr int NB = 1 << LEV;  // buckets
  // Full-vector mode: LEV <= 2 compares every element against the T keys directly
  // (count_s += a >= key_s); LEV >= 3 gives the bucket search only to elements inside
  // [key_0, key_{T-1}) (the others are below every key or counted in `above`).
  // Compacted mode (passes >= 1 when c->cap_ok): direct compares over the warp's entries.
  constexpr bool BRACKET = LEV >= 3;
  __shared__ int32_t s_key[16];
  __shared__ uint32_t s_cnt[WARPS][T];
  __shared__ uint32_t s_bkt[WARPS][NB];  // per-warp bucket totals (flushed from packed registers)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < T) s_key[threadIdx.x] = (int32_t)c->cand_key[threadIdx.x];
  if (lane < NB) s_bkt[warp][lane] = 0u;
  const bool cap_mode = !FIRST && c->cap_ok != 0u;
  const int32_t kcmp = (int32_t)c->cmp_key;
  __syncthreads();
  int32_t kr[T], km1[T];  // keys and keys - 1 (a >= k  <=>  (k - 1 - a) < 0, no overflow for a, k >= 0)
#pragma unroll
  for (int s = 0; s < T; ++s) {
    kr[s] = s_key[s];
    km1[s] = kr[s] - 1;
  }
  const int32_t root = kr[(1 << (LEV - 1)) - 1];
  const int32_t kmin = kr[0], kmax = kr[T - 1];
  const uint32_t width = (uint32_t)(kmax - kmin);
  const uint32_t gw = blockIdx.x * WARPS + warp;
  const uint64_t lo = min(sp.n, (uint64_t)gw * sp.S);
  const uint64_t hi = min(sp.n, lo + sp.S);
  const uint32_t* a32 = reinterpret_cast<const uint32_t*>(acc);
  uint32_t direct[T];  // count_s (direct mode)
  uint32_t ge[T];      // this warp's nnz per candidate
  uint32_t above = 0;
  uint64_t pk0 = 0, pk1 = 0;  // packed 8-bit bucket counters of in-bracket elements (buckets 0-7, 8-15)
  int since_flush = 0;
  uint32_t ncomp = 0;         // FIRST: compacted entries of this warp so far
  auto flush = [&]() {
#pragma unroll
    for (int b = 1; b < NB; ++b) {
      const uint64_t w = (b < 8) ? pk0 : pk1;
      const uint32_t t = __reduce_add_sync(0xffffffffu, (uint32_t)((w >> (8 * (b & 7))) & 0xFFu));
      if (lane == 0) s_bkt[warp][b] += t;
    }
    pk0 = 0;
    pk1 = 0;
    since_flush = 0;
  };
  auto add_bucket = [&](int32_t a) {
    const uint32_t b = bucket_of<LEV>(a, root, s_key);
    if (LEV <= 3) {
      pk0 += 1ull << (8 * b);
    } else {
      const uint64_t inc = 1ull << (8 * (b & 7));
      if (b & 8) pk1 += inc; else pk0 += inc;
    }
  };
  auto direct_one = [&](uint32_t bits) {
    const int32_t a = (int32_t)(bits & 0x7FFFFFFFu);
#pragma unroll
    for (int s = 0; s < T; ++s) direct[s] += (uint32_t)(km1[s] - a) >> 31;  // IADD3 + LEA.HI
  };

  if (cap_mode) {
    // ---- compacted entries of this warp: direct compares ----
#pragma unroll
    for (int s = 0; s < T; ++s) direct[s] = 0;
    const uint32_t ne = min(__ldcg(cp.cnt + gw), cp.C);
    const uint32_t* eb = cp.bits + (size_t)gw * cp.C;
    for (uint32_t j0 = 0; j0 < ne; j0 += 128) {
      const uint32_t j = j0 + 4 * lane;
      if (j + 4 <= ne) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(eb + j));
        direct_one(q.x); direct_one(q.y); direct_one(q.z); direct_one(q.w);
      } else {
        for (uint32_t t = j; t < ne && t < j + 4; ++t) direct_one(__ldcg(eb + t));
      }
    }
#pragma unroll
    for (int s = 0; s < T; ++s) ge[s] = __reduce_add_sync(0xffffffffu, direct[s]);
  } else {
    if (!BRACKET) {
#pragma unroll
      for (int s = 0; s < T; ++s) direct[s] = 0;
    }
    // ---- whole slab ----
    auto one = [&](uint32_t bits, uint32_t& inb, int j) {
      const int32_t a = (int32_t)(bits & 0x7FFFFFFFu);
      if (!BRACKET) {
        direct_one(bits);
      } else {
        above += (a >= kmax) ? 1u : 0u;
        inb |= ((uint32_t)(a - kmin) < width) ? (1u << j) : 0u;
      }
    };
    // rare path: bucket search for the in-bracket elements of a round (re-read through L1/L2 by
    // index, so the round's registers need not stay live)
    auto slow = [&](uint64_t rbase, uint32_t inb) {
      if (BRACKET && __any_sync(0xffffffffu, inb != 0u)) {
#pragma unroll 1
        for (uint32_t m = inb; m; m &= m - 1u) {
          const int j = __ffs(m) - 1;
          const uint32_t bits = __ldg(a32 + rbase + 4 * lane + (j >> 2) * 128 + (j & 3));
          add_bucket((int32_t)(bits & 0x7FFFFFFFu));
        }
      }
    };
    // FIRST: append the round's elements >= the compaction key to the warp's entries, in index
    // order (chunk, lane, element); one packed warp scan covers the four chunks
    const int32_t kcmp1 = kcmp - 1;
    auto compact = [&](const uint4* v, uint64_t rbase, uint32_t valid) {
      uint32_t m = 0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        m |= ((uint32_t)(kcmp1 - (int32_t)(v[ch].x & 0x7FFFFFFFu)) >> 31) << (4 * ch);
        m |= ((uint32_t)(kcmp1 - (int32_t)(v[ch].y & 0x7FFFFFFFu)) >> 31) << (4 * ch + 1);
        m |= ((uint32_t)(kcmp1 - (int32_t)(v[ch].z & 0x7FFFFFFFu)) >> 31) << (4 * ch + 2);
        m |= ((uint32_t)(kcmp1 - (int32_t)(v[ch].w & 0x7FFFFFFFu)) >> 31) << (4 * ch + 3);
      }
      m &= valid;
      if (!__any_sync(0xffffffffu, m != 0u)) return;
      // per-chunk counts of this lane (<= 4 each) packed in bytes; warp sums stay <= 128
      uint32_t packed = 0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) packed |= (uint32_t)__popc((m >> (4 * ch)) & 0xFu) << (8 * ch);
      uint32_t incl = packed;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - packed;
      uint32_t* oi = cp.idx + (size_t)gw * cp.C;
      uint32_t* ob = cp.bits + (size_t)gw * cp.C;
      uint32_t chunk_base = ncomp;
      const uint32_t i0 = (uint32_t)(rbase + 4 * lane);
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        uint32_t pos = chunk_base + ((excl >> (8 * ch)) & 0xFFu);
        const uint32_t mc = (m >> (4 * ch)) & 0xFu;
        const uint32_t vv[4] = {v[ch].x, v[ch].y, v[ch].z, v[ch].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if ((mc >> e) & 1u) {
            if (pos < cp.C) {
              oi[pos] = i0 + ch * 128 + e;
              ob[pos] = vv[e];
            }
            ++pos;
          }
        }
        chunk_base += (tot >> (8 * ch)) & 0xFFu;
      }
      ncomp = chunk_base;
    };
    auto consume = [&](const uint4* v, uint64_t rbase) {
      uint32_t inb = 0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        one(v[ch].x, inb, 4 * ch);
        one(v[ch].y, inb, 4 * ch + 1);
        one(v[ch].z, inb, 4 * ch + 2);
        one(v[ch].w, inb, 4 * ch + 3);
      }
      slow(rbase, inb);
      if (FIRST) compact(v, rbase, 0xFFFFu);
      if (BRACKET && ++since_flush == 15) flush();
    };
    // software pipeline, two rounds deep: while round i is counted, the 128-bit loads of rounds
    // i+1 and i+2 are in flight (8 per lane)
    uint4 va[4], vb[4];
    auto load_round = [&](uint64_t b, uint4* dst) {
      const uint64_t e0 = b + 4 * lane;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) dst[ch] = *reinterpret_cast<const uint4*>(a32 + e0 + ch * 128);
    };
    const uint64_t nfull = (hi - lo) / ROUND;  // full rounds of this slab
    uint64_t base = lo;
    if (nfull > 0) load_round(base, va);
    if (nfull > 1) load_round(base + ROUND, vb);
    for (uint64_t i = 0; i < nfull; i += 2) {
      consume(va, base);
      if (i + 2 < nfull) load_round(base + 2 * ROUND, va);
      if (i + 1 < nfull) {
        consume(vb, base + ROUND);
        if (i + 3 < nfull) load_round(base + 3 * ROUND, vb);
      }
      base += 2 * ROUND;
    }
    base = lo + nfull * ROUND;
    if (base < hi) {  // ragged tail round (end of the vector only)
      const uint64_t e0 = base + 4 * lane;
      uint32_t inb = 0, valid = 0;
      uint4 v[4];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint64_t i = e0 + (j >> 2) * 128 + (j & 3);
        const uint32_t bits = (i < hi) ? a32[i] : 0u;
        if (i < hi) {
          one(bits, inb, j);
          valid |= 1u << j;
        }
        uint32_t* vj = reinterpret_cast<uint32_t*>(&v[j >> 2]) + (j & 3);
        *vj = bits;
      }
      slow(base, inb);
      if (FIRST) compact(v, base, valid);
    }
    if (BRACKET) flush();
    if (FIRST && lane == 0) {
      cp.cnt[gw] = ncomp;
      if (ncomp > cp.C) atomicOr(&c->overflow, 1u);
    }
    __syncwarp();
    if (BRACKET) {
      uint32_t run = __reduce_add_sync(0xffffffffu, above);
#pragma unroll
      for (int b = NB - 1; b >= 1; --b) {
        run += s_bkt[warp][b];
        ge[b - 1] = run;
      }
    } else {
#pragma unroll
      for (int s = 0; s < T; ++s) ge[s] = __reduce_add_sync(0xffffffffu, direct[s]);
    }
  }
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < T; ++s) {
      wcnt[(size_t)(pass * TMAX + s) * sp.W + gw] = ge[s];
      s_cnt[warp][s] = ge[s];
    }
  }
  __syncthreads();
  if (threadIdx.x < T) {
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) tot += s_cnt[w][threadIdx.x];
    atomicAdd(&c->totals[threadIdx.x], tot);
  }
  if (!last_cta(&c->ticket)) return;
  __shared__ uint32_t s_tot[16];
  __shared__ Ctrl sc;
  if (threadIdx.x < T) s_tot[threadIdx.x] = __ldcg(&c->totals[threadIdx.x]);
  ctrl_to_smem(&sc, c);
  if (threadIdx.x == 0) {
    const double lo_key_ratio = sc.cmp_ratio;
    replay_levels(&sc, s_tot, LEV, pass, sp.k);
    sc.ticket = 0u;
    if (FIRST) {
      // compacted mode is exact iff every later threshold (and thres2) lies above the compaction
      // key: the bracket's lower end must have reached its ratio, and nothing overflowed
      sc.cap_ok = (sc.lo >= lo_key_ratio && sc.overflow == 0u) ? 1u : 0u;
      sc.overflow = 0u;
    }
    if (next_lev > 0) make_candidates(&sc, next_lev); else finish_window(&sc, sp);
  }
  __syncthreads();
  if (next_lev == 0) scan_slabs(&sc, sp, wcnt, pre1, pre2);
  ctrl_to_global(c, &sc);
}

// ------------------------------------------------------------------------------------------
// K4: stable ascending-index compaction (Alg. 1 l.25-29, Q11) with fused residual write-back.
//   class 1: bits >= key1 (iota1; empty when k1 == 0, Q8)
//   class 2: key2 <= bits < key1 (iota2); the window keeps class-2 ranks [rand, rand + k - k1)
//   output position of a kept element i = #class1 before i + clamp(#class2 before i - rand, 0, need)
// Each warp walks its slab (same partition as the count passes) in ascending order from the
// slab's exclusive prefix counts; rounds without any class-1/2 element cost a ballot only, and a
// slab that provably holds no kept element is not read at all.
// HBM/L2: <= 4 B/elem read + 8 B per selected pair + a 4-byte residual zero per selected pair.
__global__ void __launch_bounds__(THREADS, 3) k_select(const float* __restrict__ acc, const Ctrl* __restrict__ c,
                                                       SearchParams sp, const uint32_t* __restrict__ wcnt,
                                                       const uint32_t* __restrict__ pre1, const uint32_t* __restrict__ pre2,
                                                       uint32_t* __restrict__ idx_out, float* __restrict__ val_out,
                                                       float* __restrict__ r_zero, Compact cp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * WARPS + warp;
  const uint64_t lo = min(sp.n, (uint64_t)gw * sp.S);
  const uint64_t hi = min(sp.n, lo + sp.S);
  if (lo >= hi) return;
  const int32_t p1 = c->prov1, p2 = c->prov2;
  const int32_t key1 = (p1 >= 0) ? (int32_t)c->key1 : (int32_t)INF_BITS;
  const int32_t key2 = (p2 >= 0) ? (int32_t)c->key2 : 0;
  const uint32_t rnd = (uint32_t)c->rand, need = c->need;
  uint32_t b1 = pre1[gw], b2 = pre2[gw];
  {
    const uint32_t c1 = p1 >= 0 ? wcnt[(size_t)p1 * sp.W + gw] : 0u;
    const uint32_t call = p2 >= 0 ? wcnt[(size_t)p2 * sp.W + gw] : (uint32_t)(hi - lo);
    const uint32_t c2 = call - c1;
    if (c1 == 0 && (c2 == 0 || b2 >= rnd + need || b2 + c2 <= rnd)) return;  // nothing kept here
  }
  if (c->cap_ok) {
    // ---- compacted entries of this warp (ascending index order): 128 per iteration, lane l
    // holds entries 4l..4l+3 of the group, so (lane, e) order is index order ----
    const uint32_t ne = min(cp.cnt[gw], cp.C);
    const uint32_t* ei = cp.idx + (size_t)gw * cp.C;
    const uint32_t* eb = cp.bits + (size_t)gw * cp.C;
    for (uint32_t j0 = 0; j0 < ne; j0 += 128) {
      const uint32_t j = j0 + 4 * lane;
      uint32_t bb[4] = {0u, 0u, 0u, 0u}, ii[4] = {0u, 0u, 0u, 0u};
      if (j + 4 <= ne) {
        const uint4 q = __ldcg(reinterpret_cast<const uint4*>(eb + j));
        const uint4 x = __ldcg(reinterpret_cast<const uint4*>(ei + j));
        bb[0] = q.x; bb[1] = q.y; bb[2] = q.z; bb[3] = q.w;
        ii[0] = x.x; ii[1] = x.y; ii[2] = x.z; ii[3] = x.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (j + e < ne) { bb[e] = __ldcg(eb + j + e); ii[e] = __ldcg(ei + j + e); }
      }
      uint32_t fc1 = 0, fc2 = 0;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = j + e < ne;
        const int32_t a = (int32_t)(bb[e] & 0x7FFFFFFFu);
        const bool x1 = ok && a >= key1;
        const bool x2 = ok && !x1 && a >= key2;
        fc1 |= (uint32_t)x1 << e;
        fc2 |= (uint32_t)x2 << e;
      }
      const uint32_t packed = __popc(fc1) | (__popc(fc2) << 16);
      uint32_t incl = packed;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - packed;
      uint32_t q1 = b1 + (excl & 0xFFFFu);
      uint32_t q2 = b2 + (excl >> 16);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (fc1 & (1u << e)) {
          const uint32_t after = (q2 > rnd) ? min(q2 - rnd, need) : 0u;
          const uint32_t pos = q1 + after;
          idx_out[pos] = ii[e];
          val_out[pos] = __uint_as_float(bb[e]);
          if (r_zero) r_zero[ii[e]] = 0.0f;
          ++q1;
        } else if (fc2 & (1u << e)) {
          if (q2 >= rnd && q2 < rnd + need) {
            const uint32_t pos = q1 + (q2 - rnd);
            idx_out[pos] = ii[e];
            val_out[pos] = __uint_as_float(bb[e]);
            if (r_zero) r_zero[ii[e]] = 0.0f;
          }
          ++q2;
        }
      }
      b1 += tot & 0xFFFFu;
      b2 += tot >> 16;
    }
    return;
  }
  const uint32_t* a32 = reinterpret_cast<const uint32_t*>(acc);
  // rare path: a round holding class-1/2 elements.  cand: bit j = element j of the lane is >= key2
  auto emit = [&](uint64_t rbase, uint32_t cand) {
    const uint64_t e0 = rbase + 4 * lane;
    uint32_t f1 = 0;  // class-1 bits (subset of cand); class 2 = cand & ~f1
#pragma unroll 1
    for (uint32_t m = cand; m; m &= m - 1u) {
      const int j = __ffs(m) - 1;
      const uint32_t bits = __ldg(a32 + e0 + (j >> 2) * 128 + (j & 3));
      if ((int32_t)(bits & 0x7FFFFFFFu) >= key1) f1 |= 1u << j;
    }
    const uint32_t f2 = cand & ~f1;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {  // chunk order, then lane order, then element order = index order
      const uint32_t fc1 = (f1 >> (4 * ch)) & 0xFu, fc2 = (f2 >> (4 * ch)) & 0xFu;
      const uint32_t packed = __popc(fc1) | (__popc(fc2) << 16);
      uint32_t incl = packed;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - packed;
      uint32_t q1 = b1 + (excl & 0xFFFFu);
      uint32_t q2 = b2 + (excl >> 16);
#pragma unroll 1
      for (int e = 0; e < 4; ++e) {
        if (!((fc1 | fc2) & (1u << e))) continue;
        const uint32_t i = (uint32_t)(e0 + ch * 128 + e);
        if (fc1 & (1u << e)) {
          const uint32_t after = (q2 > rnd) ? min(q2 - rnd, need) : 0u;
          const uint32_t pos = q1 + after;
          idx_out[pos] = i;
          val_out[pos] = __uint_as_float(__ldg(a32 + i));
          if (r_zero) r_zero[i] = 0.0f;
          ++q1;
        } else {
          if (q2 >= rnd && q2 < rnd + need) {
            const uint32_t pos = q1 + (q2 - rnd);
            idx_out[pos] = i;
            val_out[pos] = __uint_as_float(__ldg(a32 + i));
            if (r_zero) r_zero[i] = 0.0f;
          }
          ++q2;
        }
      }
      b1 += tot & 0xFFFFu;
      b2 += tot >> 16;
    }
  };
  auto cand_of = [&](uint32_t bits, int j) -> uint32_t {
    return ((int32_t)(bits & 0x7FFFFFFFu) >= key2) ? (1u << j) : 0u;
  };
  auto consume = [&](const uint4* v, uint64_t rbase) {
    uint32_t cand = 0;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch)
      cand |= cand_of(v[ch].x, 4 * ch) | cand_of(v[ch].y, 4 * ch + 1) | cand_of(v[ch].z, 4 * ch + 2) |
              cand_of(v[ch].w, 4 * ch + 3);
    if (__any_sync(0xffffffffu, cand != 0u)) emit(rbase, cand);
  };
  // software pipeline, two rounds deep (as in k_count)
  uint4 va[4], vb[4];
  auto load_round = [&](uint64_t b, uint4* dst) {
    const uint64_t e0 = b + 4 * lane;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) dst[ch] = *reinterpret_cast<const uint4*>(a32 + e0 + ch * 128);
  };
  const uint64_t nfull = (hi - lo) / ROUND;
  uint64_t base = lo;
  if (nfull > 0) load_round(base, va);
  if (nfull > 1) load_round(base + ROUND, vb);
  for (uint64_t i = 0; i < nfull; i += 2) {
    consume(va, base);
    if (i + 2 < nfull) load_round(base + 2 * ROUND, va);
    if (i + 1 < nfull) {
      consume(vb, base + ROUND);
      if (i + 3 < nfull) load_round(base + 3 * ROUND, vb);
    }
    base += 2 * ROUND;
  }
  base = lo + nfull * ROUND;
  if (base < hi) {  // ragged tail round (end of the vector only)
    const uint64_t e0 = base + 4 * lane;
    uint32_t cand = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint64_t i = e0 + (j >> 2) * 128 + (j & 3);
      if (i < hi) cand |= cand_of(a32[i], j);
    }
    if (__any_sync(0xffffffffu, cand != 0u)) emit(base, cand);
  }
}

// ------------------------------------------------------------------------------------------
// Decompression (Alg. 2 l.15-20): out = +0; for p in rank order: out[idx_p] += val_p (fp32 RN).
// Tile-owner design: a persistent CTA owns a contiguous run of 4096-element output tiles; per
// tile it zero-fills shared memory, applies the ranks' pairs falling in the tile in rank order
// (one barrier per rank; indices within one rank are distinct so its adds never collide), and
// writes the tile once with streaming 128-bit stores.  Each rank's cursor only moves forward
// (chunks are ascending), found once per CTA by a warp-cooperative 32-ary search.  No global
// atomics, no read-modify-write of out.  HBM: 4 B/elem write + 8 B per gathered pair.

// first j in [0, n) with a[j] >= target (n if none); all lanes of the warp participate
__device__ uint32_t warp_lower_bound(const uint32_t* a, uint32_t n, uint32_t target) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t pos = lo + lane * step;
    const uint32_t v = pos < hi ? __ldg(a + pos) : 0xFFFFFFFFu;
    const uint32_t m = __ballot_sync(0xffffffffu, v >= target);
    const uint32_t f = m ? (uint32_t)(__ffs(m) - 1) : 32u;
    if (f == 0) return lo;
    const uint32_t nlo = lo + (f - 1) * step + 1;
    const uint32_t nhi = (f < 32) ? min(hi, lo + f * step) : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint32_t pos = lo + lane;
  const uint32_t v = pos < hi ? __ldg(a + pos) : 0xFFFFFFFFu;
  const uint32_t m = __ballot_sync(0xffffffffu, pos < hi && v >= target);
  return m ? lo + (uint32_t)(__ffs(m) - 1) : hi;
}

__global__ void __launch_bounds__(THREADS) k_decompress(const uint32_t* __restrict__ gathered, uint32_t nchunks,
                                                        uint64_t k, uint64_t n, uint32_t ntiles, uint32_t tiles_per_cta,
                                                        float* __restrict__ out) {
  __shared__ __align__(16) float s_tile[TILE];
  extern __shared__ uint32_t s_cur[];  // [nchunks] per-rank cursors
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t t0 = blockIdx.x * tiles_per_cta;
  const uint32_t t1 = min(ntiles, t0 + tiles_per_cta);
  if (t0 >= t1) return;
  for (uint32_t p = warp; p < nchunks; p += WARPS) {
    const uint32_t j = warp_lower_bound(gathered + (size_t)p * 2 * k, (uint32_t)k, t0 * TILE);
    if (lane == 0) s_cur[p] = j;
  }
  __syncthreads();
  float4* s4 = reinterpret_cast<float4*>(s_tile);
  for (uint32_t t = t0; t < t1; ++t) {
    const uint32_t tlo = t * TILE, thi = tlo + TILE;
    // prefetch up to 32 pairs of rank p = warp (common case: ~rho*TILE pairs per rank per tile)
    uint32_t pi = NO_INDEX, cnt = 0, cur = 0;
    float pv = 0.0f;
    if (warp < (int)nchunks) {
      const uint32_t* ch = gathered + (size_t)warp * 2 * k;
      cur = s_cur[warp];
      const uint32_t j = cur + lane;
      if (j < k) {
        pi = __ldg(ch + j);
        pv = __uint_as_float(__ldg(ch + k + j));
      }
      cnt = __popc(__ballot_sync(0xffffffffu, pi < thi));
    }
    for (int q = threadIdx.x; q < TILE / 4; q += THREADS) s4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    for (uint32_t p = 0; p < nchunks; ++p) {
      if ((uint32_t)warp == (p & (WARPS - 1))) {
        const uint32_t* ch = gathered + (size_t)p * 2 * k;
        uint32_t c0;
        if (p < WARPS) {
          if (pi < thi) s_tile[pi - tlo] = __fadd_rn(s_tile[pi - tlo], pv);
          c0 = cur + cnt;
        } else {
          c0 = s_cur[p];
        }
        if (p >= WARPS || cnt == 32) {  // more pairs of this rank in this tile
          for (;;) {
            const uint32_t j = c0 + lane;
            const uint32_t i = j < k ? __ldg(ch + j) : NO_INDEX;
            const bool in = i < thi;
            if (in) s_tile[i - tlo] = __fadd_rn(s_tile[i - tlo], __uint_as_float(__ldg(ch + k + j)));
            const uint32_t m = __popc(__ballot_sync(0xffffffffu, in));
            c0 += m;
            if (m < 32) break;
          }
        }
        if (lane == 0) s_cur[p] = c0;
      }
      __syncthreads();
    }
    if ((uint64_t)thi <= n) {
      float4* o4 = reinterpret_cast<float4*>(out + tlo);
      for (int q = threadIdx.x; q < TILE / 4; q += THREADS) __stcs(o4 + q, s4[q]);
    } else {
      for (int q = threadIdx.x; q < TILE; q += THREADS)
        if ((uint64_t)tlo + q < n) out[tlo + q] = s_tile[q];
    }
    __syncthreads();  // s_tile is rewritten by the next tile
  }
}

}  // namespace tk
