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
#include <cstddef>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace tk {

#ifdef TK_PHASE_TRACE  // experiment builds only: per-CTA %globaltimer at every phase stamp / barrier arrival
__device__ uint64_t g_trace[2][32][2048];
#define TK_TRACE(slot)                                                                                   \
  do {                                                                                                   \
    if (threadIdx.x == 0 && blockIdx.x < 2048) {                                                         \
      uint64_t t_;                                                                                       \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                             \
      g_trace[0][(slot)][blockIdx.x] = t_;                                                               \
    }                                                                                                    \
  } while (0)
#else
#define TK_TRACE(slot) do { } while (0)
#endif

constexpr int TILE = 4096;          // elements per pairwise-sum tile (power of two, Q3) / output tile
constexpr int THREADS = 256;        // 8 warps per CTA
constexpr int WARPS = THREADS / 32;
constexpr int ROUND = 512;          // elements one warp touches per round (4 chunks of 128)
constexpr int TMAX = 15;            // max candidates per count pass (4 bisection levels)
constexpr int NMAX = 52;            // max MSTopK samplings (Q5)
constexpr uint32_t INF_BITS = 0x7F800000u;
constexpr uint32_t NO_INDEX = 0xFFFFFFFFu;
#ifdef TK_DEVICE_CHECKS
#define TK_DCHECK(cond, tag, a, b)                                                                     \
  do {                                                                                                 \
    if (!(cond)) {                                                                                     \
      printf("TK_DCHECK %s failed: blk %d thr %d a=%llu b=%llu\n", tag, (int)blockIdx.x, (int)threadIdx.x, \
             (unsigned long long)(a), (unsigned long long)(b));                                       \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define TK_DCHECK(cond, tag, a, b) do { } while (0)
#endif
// Global pass totals / histograms can be replicated HREP times (copy = CTA index mod HREP) to spread
// the CTAs' atomic adds over HREP addresses per bin; readers sum the copies.  One copy is fastest:
// the histogram pass adds only its non-empty bins (C2: ~1e5 adds over ~450 bins), and every CTA then
// reads the whole histogram after the barrier - measured at C2, 8 copies: 73.9 us per call, 4: 73.4,
// 2: 72.4, 1: 71.8 (the read of 8 copies costs 2 us more than the contention it saves).
#ifndef TK_HREP
#define TK_HREP 1
#endif
constexpr int HREP = TK_HREP;
// COUNT_HIST: up to HIST_LEV bisection levels (2^HIST_LEV - 1 candidate keys) per histogram pass
constexpr int HIST_LEV = 10;
constexpr int HIST_BINS = 1 << HIST_LEV;
constexpr int TOT_STRIDE = HIST_BINS;  // words per copy
constexpr int NPATH_CAND = 16;           // candidates with an explicit ratio / threshold (path, exact)

// Device-resident MSTopK control block (Alg. 1 l.4-6 state + the trial log).  Laid out as
//   [header: scalar state, incl. what the next call predicts from]  copied in by every CTA
//   [logs: trial log, phase stamps]                                  written back by CTA 0
//   [scratch: candidate keys of one pass]                            per call, never copied
struct Ctrl {
  // ---------------------------------------------------------------- header
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
  uint32_t cap_ok;       // 1: passes >= 1 and the selection run on the compacted entries (see k_count)
  uint32_t cmp_key;      // key above which the first count pass compacts elements
  double cmp_ratio;      // its bisection ratio
  double prev_lo;        // final l of the previous compression (predicts the bracket; perf only)
  uint32_t need;
  uint32_t n_phase;
  uint64_t len2;
  uint64_t rand;
  uint64_t step;
  uint32_t n_compacted;  // entries kept by the compaction (all warps)
  uint32_t cand_tree;    // the candidates form a complete subtree (walked by index in replay)
  // exact selector (TK_SELECT_EXACT): bracket [xlo, xhi) of the k-th largest key T with
  // xcnt_lo = #{a >= xlo} >= k > xcnt_hi = #{a >= xhi}; prev_T = the previous call's T (0: none)
  uint32_t xlo, xhi, xcnt_lo, xcnt_hi;
  uint32_t prev_T, prev_dT;  // the previous call's T and how far T moved in that call
  uint32_t xretry;       // a whole-vector compaction retry was spent
  uint32_t xguess;       // exact: upper end of the first histogram pass's keys (0: xhi)
  uint32_t cmp_bottom;   // the entries sit at the bottom of the warp regions (ef-phase compaction)
  uint32_t ef_key;       // compaction key of the NEXT call's ef phase (0: none), set at the end of a call
  uint32_t ef_used;      // this call's selection ran on the ef-phase entries
  uint32_t prev_key2;    // MSTopK: the previous call's key2
  uint32_t mv_est;       // decaying maximum of the recent moves of key2 (exact selector: of T), in key units
  uint64_t nnz_lb;       // trials whose count was not taken (their key lay below the ef-phase key, so
                         // only "nnz > k" is known); cleared when exact_trial_counts counts them
  // prose search (TK_SELECT_PROSE, reading Q33): the next trial threshold pt and the bracket
  // [lo, hi] in THRESHOLD units (Alg. 1's bisection keeps lo, hi in ratio units); lo / hi are
  // only meaningful once set
  double pt;
  uint32_t lo_set, hi_set;
  // ---------------------------------------------------------------- logs
  double ratio_log[NMAX];
  double thres_log[NMAX];
  uint32_t key_log[NMAX];
  uint32_t nnz_log[NMAX];
  uint64_t phase_ns[12];  // %globaltimer at the phase boundaries of the last k_compress (CTA 0)
  // ---------------------------------------------------------------- per-call scratch
  double cand_ratio[NPATH_CAND];    // coordinate (ratio / threshold) of path candidates
  double cand_t[NPATH_CAND];        // and their thresholds
  uint32_t cand_key[HIST_BINS];     // candidate keys (ascending for a tree / histogram pass)
  double tree_t[HIST_BINS];         // tree candidates' thresholds, kept by make_candidates_par so the serial
  double tree_lo, tree_w, tree_scale;  // replay recomputes none; ratio of node m = lo + w * (m * scale)
};
constexpr int CTRL_HEADER_WORDS = (int)(offsetof(Ctrl, ratio_log) / 4);
constexpr int CTRL_KEEP_WORDS = (int)(offsetof(Ctrl, cand_ratio) / 4);
static_assert(offsetof(Ctrl, ratio_log) % 8 == 0 && offsetof(Ctrl, cand_ratio) % 8 == 0, "Ctrl layout");


// Per-launch parameters of the MSTopK kernels.  The count and selection kernels share one
// partition of [0, n) into W contiguous warp slabs of S elements (S a multiple of ROUND).
struct SearchParams {
  uint64_t n;        // vector length MSTopK runs on (d, or d/n for HiTopKComm)
  uint64_t k;        // number of elements to select
  uint32_t W;        // warp slabs (= gridDim.x * WARPS of the count / select launches)
  uint64_t S;        // slab length (one run of units_per_warp 512-element units)
  uint32_t R;        // runs: ceil(n / S) <= W
  uint32_t fold;     // 1: warp gw owns run gw and each CTA folds its 8 runs (R >= 7/8 W); 0: balanced map
  uint32_t rank;
  uint32_t rand_mode;
  uint64_t seed;
};

// Warp -> run map (monotone, balanced over the CTAs): CTA b owns runs [floor(b*R/G), floor((b+1)*R/G))
// - 0..8 consecutive runs - on its first warps; run j covers elements [j*S, (j+1)*S).  The runs must
// stay aligned power-of-two blocks of units for the canonical tree (Q3), so R = ceil(n/S) < W in
// general; leaving the W - R idle warps all in the last CTAs would idle whole SMs (measured: 2048 of
// 3552 warps busy at d = 2^27 ran the EF pass 2x slower), so they are spread over the CTAs instead.
// Each warp's subtree goes to run_sum[j]; stats_root folds the R run sums.
__device__ __forceinline__ int32_t warp_run_of(const SearchParams& sp, uint32_t gw) {
  // when almost every warp has a run (R >= 7/8 W, e.g. C2: 3125 / 3552) the identity map is kept:
  // each CTA's 8 runs are then one aligned subtree it folds itself, and stats_root reads only the
  // G CTA partials (measured: ~1 us faster at the root, and the idle warps cost ~0.5 us)
  if (sp.fold) return gw < sp.R ? (int32_t)gw : -1;
  const uint32_t G = sp.W / WARPS, b = gw / WARPS, w = gw % WARPS;
  const uint32_t j0 = b * sp.R / G, j1 = (b + 1) * sp.R / G;  // W * R < 2^32
  return j0 + w < j1 ? (int32_t)(j0 + w) : -1;
}

// Compacted entries of the first count pass: warp w keeps, in ascending index order, every
// element of its slab with |acc| >= the compaction key, at the top of its region
// (idx[w*C + C - cnt[w] + j], bits[...], j < cnt[w]).  When the bisection's bracket after that pass lies above that key, no later trial
// threshold and no selected element can lie below it, so the later passes and the selection read
// only these entries instead of the whole vector (exact: same counts, same sets).
struct Compact {
  uint32_t* idx;
  uint32_t* bits;
  uint32_t* cnt;
  uint32_t C;  // capacity per warp (multiple of 4)
};

// first entry of warp gw's compacted entries (ne of them): top of the region for the count
// pass's compaction, bottom for the ef phase's
__device__ __forceinline__ uint32_t entry_off(const Compact& cp, uint32_t ne, uint32_t bottom) {
  return bottom ? 0u : cp.C - ne;
}

// TK_AG_PUSH (fused all-gather): slot[q] = this rank's chunk of peer q's gathered buffer (q == me:
// the local one).  A pair travels as one 16-byte packet of two 8-byte words {idx, tag} and
// {val, tag}; tag = the step's sequence number.  Each 8-byte word is written and read as one
// single-copy-atomic access, so a reader that sees both tags equal to the step's sequence has the
// pair -- no fence, no flag, no counter (the "tag in every word" protocol).
struct PushOut {
  ulonglong2* slot[8];
  uint32_t np, me, tag;
};

__device__ __forceinline__ void st_ll(ulonglong2* p, uint32_t i, uint32_t v, uint32_t tag) {
  const uint64_t a = (uint64_t)i | ((uint64_t)tag << 32), b = (uint64_t)v | ((uint64_t)tag << 32);
  asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}

__device__ __forceinline__ ulonglong2 ld_ll(const ulonglong2* p) {
  ulonglong2 v;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
  return v;
}

// chunked pair sources of the decompression
struct PlainChunks {  // [nchunks][idx k | val k] u32
  const uint32_t* g;
  uint64_t k;
  __device__ __forceinline__ uint32_t idx(uint32_t p, uint32_t j) const { return __ldg(g + (size_t)p * 2 * k + j); }
  __device__ __forceinline__ void get(uint32_t p, uint32_t j, uint32_t& i, float& v) const {
    i = __ldg(g + (size_t)p * 2 * k + j);
    v = __uint_as_float(__ldg(g + (size_t)p * 2 * k + k + j));
  }
};

struct PlainChunks16 {  // FP16 wire: [nchunks][idx k | binary16 val k (padded to whole words)] (stride cw words)
  const uint32_t* g;
  uint64_t k, cw;
  __device__ __forceinline__ uint32_t idx(uint32_t p, uint32_t j) const { return __ldg(g + (size_t)p * cw + j); }
  __device__ __forceinline__ void get(uint32_t p, uint32_t j, uint32_t& i, float& v) const {
    i = __ldg(g + (size_t)p * cw + j);
    v = __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short*>(g + (size_t)p * cw + k) + j)));
  }
};

struct TaggedChunks {  // [nchunks][k] tagged packets, written by the peers during this step
  const ulonglong2* g;
  uint64_t k;
  uint32_t tag;
  uint32_t* err;        // sticky timeout flag (device word, reported by tk_get_stats)
  uint64_t timeout_ns;  // how long to wait for one packet before giving up
  // A packet that never arrives (a peer that died, or one that stalls longer than the timeout)
  // sets *err and yields NO_INDEX - which every consumer treats as "beyond this tile", so the
  // kernel finishes (memory-safe, result invalid) instead of trapping the CUDA context; once the
  // flag is set no further packet is waited for.
  __device__ __forceinline__ void get(uint32_t p, uint32_t j, uint32_t& i, float& v) const {
    const ulonglong2* a = g + (size_t)p * k + j;
    ulonglong2 x = ld_ll(a);
    if ((uint32_t)(x.x >> 32) != tag || (uint32_t)(x.y >> 32) != tag) {
      uint64_t t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      do {
        if (*reinterpret_cast<volatile uint32_t*>(err)) {
          i = NO_INDEX;
          v = 0.0f;
          return;
        }
        __nanosleep(64);
        x = ld_ll(a);
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > timeout_ns) {
          atomicExch(err, 1u);
          i = NO_INDEX;
          v = 0.0f;
          return;
        }
      } while ((uint32_t)(x.x >> 32) != tag || (uint32_t)(x.y >> 32) != tag);
    }
    i = (uint32_t)x.x;
    v = __uint_as_float((uint32_t)x.y);
  }
  __device__ __forceinline__ uint32_t idx(uint32_t p, uint32_t j) const {
    uint32_t i;
    float v;
    get(p, j, i, v);
    return i;
  }
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
// four consecutive u32 of the compacted entries (their start is only 4-byte aligned)
__device__ __forceinline__ uint4 ldcg4(const uint32_t* p) {
  return make_uint4(__ldcg(p), __ldcg(p + 1), __ldcg(p + 2), __ldcg(p + 3));
}

__device__ __forceinline__ uint32_t key_of(double t) {
  if (!(t > 0.0)) return 0u;
  return __float_as_uint(__double2float_ru(t));
}

// Selectors of the compression kernel: Alg. 1 (MSTopK), the exact top-k of Eq. 2 and
// MSTopK with the threshold search the prose of P:148 describes (reading Q33).
enum { SEL_MSTOPK = 0, SEL_EXACT = 1, SEL_PROSE = 2 };

// Prose search (Q33), one trial's outcome: nnz > k ("too many": the bracket's low end
// moves up to t) or nnz <= k (its high end moves down to t); then the next trial is 2t while no
// trial has had nnz <= k, t/2 while none has had nnz > k, else the fp64 midpoint of the bracket.
// fmax / fmin are exact; 2t and t/2 are exact in fp64 here (|t| between 2^-200 and 2^200).
__device__ __forceinline__ void prose_advance(double& t, double& lo, double& hi, uint32_t& lo_set, uint32_t& hi_set,
                                              bool gt) {
  if (gt) { lo = lo_set ? fmax(lo, t) : t; lo_set = 1u; }
  else    { hi = hi_set ? fmin(hi, t) : t; hi_set = 1u; }
  if (!hi_set) t = __dmul_rn(t, 2.0);
  else if (!lo_set) t = __dmul_rn(t, 0.5);
  else t = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), 0.5));
}

// Candidates of one count pass: the 2^lev - 1 trial keys of the next lev levels of the search
// tree below the current state, in in-order (= ascending threshold) order.
//   Alg. 1: the ratios lo + (hi-lo)*m/2^lev; every ratio is dyadic with <= 52 significant bits,
//   so this is exact and equals the sequential l + (r-l)/2 of Alg. 1 l.8 (Q5).
//   Prose: candidate m's threshold is found by walking from the root, taking at each node the
//   decision that leads toward m (left = nnz <= k = smaller thresholds), with the same fp64
//   operations the replay performs - so the keys are bit-identical to the trials' keys.
// Computed by the CTA's threads in parallel (candidate m-1 by thread m-1); the caller
// synchronises the CTA before and after.
template <int SEL>
__device__ __forceinline__ void make_candidates_par(Ctrl* c, int lev) {
  const int T = (1 << lev) - 1;  // <= 1023
  if constexpr (SEL == SEL_PROSE) {
    for (int m = (int)threadIdx.x + 1; m <= T; m += THREADS) {
      double t = c->pt, lo = c->lo, hi = c->hi;
      uint32_t ls = c->lo_set, hs = c->hi_set;
      int node = (T + 1) >> 1, half = node >> 1;
      while (node != m) {
        const bool gt = m > node;
        prose_advance(t, lo, hi, ls, hs, gt);
        node += gt ? half : -half;
        half >>= 1;
      }
      c->cand_key[m - 1] = key_of(t);
      c->tree_t[m - 1] = t;
    }
  } else {
    const double w = __dsub_rn(c->hi, c->lo);
    const double scale = __longlong_as_double((long long)(1023 - lev) << 52);  // 2^-lev, exact
    for (int m = (int)threadIdx.x + 1; m <= T; m += THREADS) {
      const double ratio = __dadd_rn(c->lo, __dmul_rn(w, (double)m * scale));
      const double t = threshold_of(c->abar, c->U, ratio);
      c->cand_key[m - 1] = key_of(t);
      c->tree_t[m - 1] = t;
    }
    if (threadIdx.x == 0) { c->tree_lo = c->lo; c->tree_w = w; c->tree_scale = scale; }
  }
  if (threadIdx.x == 0) {
    c->ncand = (uint32_t)T;
    c->cand_tree = 1u;
  }
}

// Replay lev levels of Alg. 1 l.8-23 on the candidates' exact counts.
template <int SEL>
__device__ __forceinline__ int replay_levels(Ctrl* c, const uint32_t* totals, int max_lev, int pass, uint64_t k) {
  // Alg. 1 l.8-23, one level at a time: the level's trial (Alg. 1: ratio l + (r-l)/2, exact, Q5;
  // prose: the state's next threshold) is looked up among the counted candidates; the replay
  // stops at the first level whose threshold was not counted (speculative candidate sets).
  // Returns the number of levels resolved.
  const int nc = (int)c->ncand;
  // a complete subtree (make_candidates_par: 2^L - 1 ascending candidates) is walked by index;
  // other sets (the first pass's path) are searched by their coordinate (ratio / threshold)
  const bool tree = ((nc + 1) & nc) == 0 && c->cand_tree;
  int m = (nc + 1) >> 1, stepm = m >> 1;  // tree walk: 1-based node index and half-width
  int l = 0;
  if (tree) {
    // node m of the complete subtree is exactly this level's trial (Alg. 1: its ratio is dyadic,
    // so lo + (hi-lo)*m/2^L equals the sequential midpoints, Q5; prose: the candidate walked the
    // same decisions): coordinate, threshold and key as make_candidates_par kept them.  The state
    // lives in registers for the walk (this serial chain is on the kernel's critical path).
    uint32_t it = c->it, k1 = c->k1, k2 = c->k2, key1 = c->key1, key2 = c->key2;
    double thres1 = c->thres1, thres2 = c->thres2, lo = c->lo, hi = c->hi;
    int32_t prov1 = c->prov1, prov2 = c->prov2;
    const double tlo = c->tree_lo, tw = c->tree_w, tscale = c->tree_scale;
    for (; l < max_lev && m >= 1 && m <= nc; ++l) {
      const int s = m - 1;
      const uint32_t nnz = totals[s], key = c->cand_key[s];
      const double t = c->tree_t[s];
      const double ratio = (SEL == SEL_PROSE) ? t : __dadd_rn(tlo, __dmul_rn(tw, (double)m * tscale));
      c->ratio_log[it] = (SEL == SEL_PROSE) ? __longlong_as_double(0x7FF8000000000000ll) : ratio;  // prose: no ratio
      c->thres_log[it] = t;
      c->key_log[it] = key;
      c->nnz_log[it] = nnz;
      ++it;
      const bool gt = (uint64_t)nnz > k;
      if (!gt) {                           // l.11
        hi = ratio;                        // l.12 (prose: the bracket, re-derived below)
        if (nnz > k1) { k1 = nnz; thres1 = t; key1 = key; prov1 = pass * TMAX + s; }  // l.13-15
        m -= stepm;
      } else {                             // l.17
        lo = ratio;                        // l.18
        if (nnz < k2) { k2 = nnz; thres2 = t; key2 = key; prov2 = pass * TMAX + s; }  // l.19-21
        m += stepm;
      }
      if constexpr (SEL == SEL_PROSE) prose_advance(c->pt, c->lo, c->hi, c->lo_set, c->hi_set, gt);
      stepm >>= 1;
    }
    c->it = it; c->k1 = k1; c->k2 = k2; c->key1 = key1; c->key2 = key2;
    c->thres1 = thres1; c->thres2 = thres2; c->prov1 = prov1; c->prov2 = prov2;
    if constexpr (SEL != SEL_PROSE) { c->lo = lo; c->hi = hi; }
    return l;
  }
  for (; l < max_lev; ++l) {
    double ratio, t;
    if constexpr (SEL == SEL_PROSE) {
      ratio = c->pt;  // the prose search's coordinate is the threshold itself
    } else {
      ratio = __dadd_rn(c->lo, __dmul_rn(__dsub_rn(c->hi, c->lo), 0.5));  // Alg. 1 l.8
    }
    int s = -1;
    if (tree) {
      // node m of the complete subtree is exactly this level's trial: its threshold and key
      // are recomputed by the same operations make_candidates_par used
      if (m >= 1 && m <= nc) s = m - 1;
      t = (SEL == SEL_PROSE) ? ratio : threshold_of(c->abar, c->U, ratio);
    } else {
      for (int q = 0; q < nc && q < NPATH_CAND; ++q)
        if (c->cand_ratio[q] == ratio) { s = q; break; }
      t = s >= 0 ? c->cand_t[s] : 0.0;
    }
    if (s < 0) break;
    const uint32_t nnz = totals[s];
    const uint32_t key = c->cand_key[s];
    const uint32_t it = c->it;
    c->ratio_log[it] = (SEL == SEL_PROSE) ? __longlong_as_double(0x7FF8000000000000ll) : ratio;  // prose: no ratio
    c->thres_log[it] = t;
    c->key_log[it] = key;
    c->nnz_log[it] = nnz;
    c->it = it + 1;
    const bool gt = (uint64_t)nnz > k;
    if (!gt) {                           // l.11
      if constexpr (SEL != SEL_PROSE) c->hi = ratio;  // l.12
      if (nnz > c->k1) {                 // l.13
        c->k1 = nnz; c->thres1 = t; c->key1 = key; c->prov1 = pass * TMAX + s;
      }
      m -= stepm;
    } else {                             // l.17
      if constexpr (SEL != SEL_PROSE) c->lo = ratio;  // l.18
      if (nnz < c->k2) {                 // l.19
        c->k2 = nnz; c->thres2 = t; c->key2 = key; c->prov2 = pass * TMAX + s;
      }
      m += stepm;
    }
    if constexpr (SEL == SEL_PROSE) prose_advance(c->pt, c->lo, c->hi, c->lo_set, c->hi_set, gt);
    stepm >>= 1;
  }
  return l;
}

// Speculative candidates of the first pass: the lev search nodes along the path toward `target`
// (the bracket the previous compression ended in, as a coordinate: ratio for Alg. 1, threshold
// for the prose search).  When the data take that path, one read of the vector resolves lev
// levels with lev keys; otherwise it resolves at least one.
template <int SEL>
__device__ __forceinline__ void make_candidates_path(Ctrl* c, int lev, double target) {
  if constexpr (SEL == SEL_PROSE) {
    double t = c->pt, lo = c->lo, hi = c->hi;
    uint32_t ls = c->lo_set, hs = c->hi_set;
    for (int q = 0; q < lev; ++q) {
      c->cand_ratio[q] = t;
      c->cand_t[q] = t;
      c->cand_key[q] = key_of(t);
      prose_advance(t, lo, hi, ls, hs, target >= t);
    }
  } else {
    double lo = c->lo, hi = c->hi;
    for (int q = 0; q < lev; ++q) {
      const double ratio = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), 0.5));
      const double t = threshold_of(c->abar, c->U, ratio);
      c->cand_ratio[q] = ratio;
      c->cand_t[q] = t;
      c->cand_key[q] = key_of(t);
      if (target >= ratio) lo = ratio; else hi = ratio;
    }
  }
  c->ncand = (uint32_t)lev;
  c->cand_tree = 0u;
}

// the search bracket's low end (as a coordinate) lies at or above x: every later trial does too
template <int SEL>
__device__ __forceinline__ bool bracket_low_at_least(const Ctrl* c, double x) {
  if constexpr (SEL == SEL_PROSE) return c->lo_set && c->lo >= x;
  return c->lo >= x;
}

// Alg. 1 l.27's random source (Q10): H = SplitMix64 chain over (seed, step, rank, 0); it does not
// depend on the data, so each launch computes it once, off the critical path.
__device__ __forceinline__ uint64_t window_hash(uint64_t seed, uint64_t step, uint32_t rank) {
  // sm64(sm64(sm64(sm64(seed) ^ step) ^ rank) ^ 0), as a loop (one copy of the code)
  uint64_t h = seed;
#pragma unroll 1
  for (int q = 0; q < 4; ++q) h = sm64(h ^ (q == 1 ? step : (q == 2 ? (uint64_t)rank : 0ull)));
  return h;
}

// Alg. 1 l.27 window: R = len(iota2) - (k - k1) + 1 >= 1 (Q8, Q9); rand uniform on [0, R):
// floor(H * R / 2^64).  (k1, k2 as counts; k2 counts a >= thres2, n when thres2 was never set.)
struct Window {
  uint64_t len2, need, rand;
};
__device__ __forceinline__ Window window_of(uint64_t k1, uint64_t cnt2, const SearchParams& sp, uint64_t H) {
  Window w;
  w.len2 = cnt2 - k1;
  w.need = sp.k - k1;
  const uint64_t R = w.len2 - w.need + 1;
  w.rand = (sp.rand_mode == 0) ? __umul64hi(H, R) : 0ull;
  return w;
}
__device__ __forceinline__ void finish_window(Ctrl* c, const SearchParams& sp, uint64_t H) {
  const Window w = window_of(c->k1, (c->prov2 >= 0) ? (uint64_t)c->k2 : sp.n, sp, H);
  c->len2 = w.len2;
  c->need = (uint32_t)w.need;
  c->rand = w.rand;
}

// The selection's inputs straight from a histogram pass that resolves ALL N levels (the fast
// search's single pass): every thread walks Alg. 1 l.8-21 over the pass's complete candidate
// subtree (node m's count is tot[m-1]; right iff nnz > k) from the reset state (l.4-6) and keeps
// only k1 / k2 and their candidates - the same decisions replay_levels takes, without its trial
// log, thresholds and bracket, which block 0 fills in after the selection (the control block it
// writes back is bit-identical).  ok: thres2 was set at or above the ef-phase key (the search was
// exact, see k_compress).
struct FastDecision {
  int32_t s1, s2;      // candidate index of thres1 / thres2 (-1: never set)
  uint32_t k1, k2;     // Alg. 1's k1, k2
  uint32_t key1, key2;
  Window w;
  bool ok;
};
__device__ __forceinline__ FastDecision fast_walk(const Ctrl* c, const uint32_t* tot, int lev, const SearchParams& sp,
                                                  uint32_t efk, uint64_t H) {
  FastDecision d;
  int m = 1 << (lev - 1), st = m >> 1;
  d.k1 = 0u;
  d.k2 = (uint32_t)sp.n;
  d.s1 = -1;
  d.s2 = -1;
#pragma unroll 1
  for (int l = 0; l < lev; ++l) {
    const int s = m - 1;
    const uint32_t nnz = tot[s];
    if ((uint64_t)nnz > sp.k) {           // l.17-21
      if (nnz < d.k2) { d.k2 = nnz; d.s2 = s; }
      m += st;
    } else {                              // l.11-15
      if (nnz > d.k1) { d.k1 = nnz; d.s1 = s; }
      m -= st;
    }
    st >>= 1;
  }
  d.key1 = d.s1 >= 0 ? c->cand_key[d.s1] : INF_BITS;
  d.key2 = d.s2 >= 0 ? c->cand_key[d.s2] : 0u;
  d.w = window_of(d.k1, d.s2 >= 0 ? (uint64_t)d.k2 : sp.n, sp, H);
  d.ok = d.s2 >= 0 && d.key2 >= efk;
  return d;
}

// The last CTA runs the scalar control on a shared-memory copy of the control block (one
// coalesced load and store by the whole CTA instead of a chain of dependent global accesses).
__device__ __forceinline__ void ctrl_to_smem(Ctrl* s, const Ctrl* g) {
  static_assert(sizeof(Ctrl) % 4 == 0, "Ctrl must be a whole number of words");
  for (int i = threadIdx.x; i < CTRL_HEADER_WORDS; i += blockDim.x)
    reinterpret_cast<uint32_t*>(s)[i] = __ldcg(reinterpret_cast<const uint32_t*>(g) + i);
  __syncthreads();
}
__device__ __forceinline__ void ctrl_to_global(Ctrl* g, const Ctrl* s) {
  __syncthreads();
  for (int i = threadIdx.x; i < CTRL_KEEP_WORDS; i += blockDim.x)
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
// Candidates of the whole-vector first count pass: the nodes along the path toward the bracket
// the previous compression ended in; the compaction key is the highest of them at or below that
// bracket (any choice is exact; a good one keeps few elements).  One thread.
template <int SEL>
__device__ __forceinline__ void first_pass_candidates(Ctrl* sc, int first_levels) {
  make_candidates_path<SEL>(sc, first_levels, sc->prev_lo);
  int ms = 0;
  for (int q = 1; q < (int)sc->ncand; ++q)
    if (sc->cand_ratio[q] <= sc->prev_lo && sc->cand_ratio[q] > sc->cand_ratio[ms]) ms = q;
  if (sc->cand_ratio[ms] > sc->prev_lo) {  // no candidate below the prediction: take the lowest
    for (int q = 1; q < (int)sc->ncand; ++q)
      if (sc->cand_ratio[q] < sc->cand_ratio[ms]) ms = q;
  }
  // the compaction key becomes candidate 0, so the first pass's compaction test is the same
  // compare as its count of that key (the replay finds candidates by coordinate, order-free)
  if (ms != 0) {
    const double r0 = sc->cand_ratio[0], t0 = sc->cand_t[0];
    const uint32_t k0 = sc->cand_key[0];
    sc->cand_ratio[0] = sc->cand_ratio[ms]; sc->cand_t[0] = sc->cand_t[ms]; sc->cand_key[0] = sc->cand_key[ms];
    sc->cand_ratio[ms] = r0; sc->cand_t[ms] = t0; sc->cand_key[ms] = k0;
  }
  sc->cmp_key = sc->cand_key[0];
  sc->cmp_ratio = sc->cand_ratio[0];
}

// Alg. 1 l.4-6: the search state before the first trial (prose: trial 1 at t = a-bar, no bracket)
template <int SEL>
__device__ __forceinline__ void search_reset(Ctrl* c, uint64_t n) {
  c->lo = 0.0; c->hi = 1.0;                             // l.4
  c->k1 = 0u; c->k2 = (uint32_t)n;                      // l.5
  c->thres1 = 0.0; c->thres2 = 0.0;                     // l.6
  c->key1 = INF_BITS; c->key2 = 0u;                     // Q8 / Q9 sentinels
  c->prov1 = -1; c->prov2 = -1;
  c->it = 0u;
  if constexpr (SEL == SEL_PROSE) {
    c->lo = 0.0; c->hi = 0.0;
    c->lo_set = 0u; c->hi_set = 0u;
    c->pt = c->abar;                                    // "we first use the average value"
  }
}

template <int SEL>
__device__ __forceinline__ void stats_finalize(Ctrl* c, const SearchParams& sp, double S, uint32_t m, uint64_t step) {
  // the previous call's final bracket low end predicts this call's (prose: 0 when never set)
  c->prev_lo = (SEL == SEL_PROSE && !c->lo_set) ? 0.0 : c->lo;
  c->abar = __ddiv_rn(S, (double)sp.n);                 // Alg. 1 l.2
  c->umax_bits = m;                                     // Alg. 1 l.3
  c->U = (double)__uint_as_float(m);
  c->nonfinite = (m >= INF_BITS) ? 1u : 0u;
  search_reset<SEL>(c, sp.n);
  c->step = step;
}

// HiTopKComm step 1 fused into K1 (Eq. 4; reading Q20): with NP > 0 the gradient of
// this GPU's segment is the ordered reduce-scatter sum_{q=0..NP-1} g_q[segment], read directly
// from the row peers' memory (CUDA IPC peer pointers over NVLink) and added in ascending row rank,
// left to right, in fp32 round-to-nearest - bit-exact, unlike a reduce-scatter whose order the
// library chooses.
struct Peers {
  const float* p[8];  // row peers' gradient + segment offset, in row-rank order
};

// The ef phase's unit is one warp round of 512 elements as four coalesced 128-element chunks:
// lane l holds elements 4l..4l+3 of each chunk (one 128-bit load per chunk per source).
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

// Entries the ef phase keeps: staged per warp in shared memory; a warp whose entries outgrow the
// staging buffer spills them, in order, to its global region (flushed > 0) - otherwise they stay in
// shared memory for the count, prefix and selection phases of the same CTA (no global round trip).
constexpr uint32_t SCAP = 256;
struct EfStage {
  uint32_t si[WARPS][SCAP];  // element index
  uint32_t sb[WARPS][SCAP];  // bits of acc
  uint32_t n[WARPS];         // entries of the warp
  uint32_t in_smem[WARPS];   // 1: all of them are in si/sb (none spilled)
  int32_t run[WARPS];        // the warp's run (warp_run_of), -1: idle
};
// one per CTA of k_compress (file scope: its address is a constant, so no register holds it)
__shared__ EfStage g_es;
// this warp's slab [lo, hi) of the count and selection phases (empty for an idle warp)
__device__ __forceinline__ void warp_slab(const SearchParams& sp, int warp, uint64_t& lo, uint64_t& hi) {
  const int32_t j = g_es.run[warp];
  lo = j < 0 ? sp.n : min(sp.n, (uint64_t)j * sp.S);
  hi = j < 0 ? sp.n : min(sp.n, lo + sp.S);
}

// A warp's compacted entries, wherever they are (ascending index order): generic pointers into the
// warp's shared-memory staging buffer or its global region.  Plain (generic) loads are safe for the
// global case too: a warp only ever reads entries it wrote itself earlier in the same launch (same
// SM, whose L1 never holds a stale copy of its own stores).
struct Entries {
  const uint32_t* idx;
  const uint32_t* bits;
  uint32_t n;
  __device__ __forceinline__ uint32_t b(uint32_t j) const { return bits[j]; }
  __device__ __forceinline__ uint32_t i(uint32_t j) const { return idx[j]; }
  __device__ __forceinline__ uint4 b4(uint32_t j) const { return make_uint4(bits[j], bits[j + 1], bits[j + 2], bits[j + 3]); }
  __device__ __forceinline__ uint4 i4(uint32_t j) const { return make_uint4(idx[j], idx[j + 1], idx[j + 2], idx[j + 3]); }
};
__device__ __forceinline__ Entries warp_entries(const Compact& cp, uint32_t cmp_bottom, uint32_t gw, int warp) {
  const EfStage& es = g_es;
  Entries e;
  if (cmp_bottom && es.in_smem[warp]) {
    e.idx = es.si[warp];
    e.bits = es.sb[warp];
    e.n = es.n[warp];
  } else {
    e.n = min(__ldcg(cp.cnt + gw), cp.C);
    const uint32_t off = entry_off(cp, e.n, cmp_bottom);
    e.idx = cp.idx + (size_t)gw * cp.C + off;
    e.bits = cp.bits + (size_t)gw * cp.C + off;
  }
  return e;
}

__device__ __forceinline__ double lane_quad_sum(float4 v) {
  return __dadd_rn(__dadd_rn((double)fabsf(v.x), (double)fabsf(v.y)), __dadd_rn((double)fabsf(v.z), (double)fabsf(v.w)));
}
__device__ __forceinline__ uint32_t quad_max_bits(float4 v) {
  const uint32_t a = __float_as_uint(v.x) & 0x7FFFFFFFu, b = __float_as_uint(v.y) & 0x7FFFFFFFu;
  const uint32_t c = __float_as_uint(v.z) & 0x7FFFFFFFu, d = __float_as_uint(v.w) & 0x7FFFFFFFu;
  return max(max(a, b), max(c, d));
}

// A1 + A2 (+ H1 when NP > 0): acc = (sum of the NP sources, or g) (+ r with EF), stored to accw
// when not already in memory (EF: accw = r, in place; the HiTopKComm peer sum without EF: a
// segment scratch), the canonical fp64 pairwise tree of |acc| (Q3) - lane: 4 leaves, xor-shuffle:
// 128-leaf chunks, unit: 512, warp: aligned power-of-two run of units (binary-counter stack) - and
// max |acc|.
// Optional compaction (ckey > 0, a key predicted by the previous call): every element with
// bits(|acc|) >= ckey is appended, in index order, to the warp's entries (EfStage; spilled to the
// BOTTOM of the warp's global region [0, cnt) if they outgrow it); the warp's units are exactly its
// count-pass slab.  Per-CTA entry totals go to cta_ent; a warp holding more than the global
// capacity writes this launch's sequence number to *overflow (a flag that is never cleared, so no
// CTA can wipe another's report).
template <bool EF, int NP>
__device__ __forceinline__ void ef_phase(const float* __restrict__ g, const Peers& pr, const float* r,
                                         float* accw, const SearchParams& sp, uint32_t units_per_warp,
                                         double* __restrict__ run_sum, uint32_t* __restrict__ cta_max,
                                         uint32_t ckey, const Compact cp, uint32_t* overflow, uint32_t seq,
                                         uint32_t* __restrict__ cta_ent) {
  EfStage& es = g_es;
  constexpr bool STORE = EF || NP > 0;
  __shared__ uint32_t s_wm[WARPS];
  __shared__ double s_ws[WARPS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t n = sp.n;
  const uint32_t gw = blockIdx.x * WARPS + warp;
  const int32_t run = es.run[warp];
  const uint64_t u0 = run < 0 ? 0 : (uint64_t)run * units_per_warp;
  const uint32_t nunits = run < 0 ? 0u : units_per_warp;
  const bool cmp_on = ckey > 0u;
  const int32_t ckm1 = (int32_t)ckey - 1;
  uint32_t staged = 0, flushed = 0;  // warp-uniform: entries in the staging buffer / spilled
  uint32_t* oi = cp.idx + (size_t)gw * cp.C;
  uint32_t* ob = cp.bits + (size_t)gw * cp.C;
  uint32_t* si = es.si[warp];
  uint32_t* sb = es.sb[warp];
  auto spill = [&]() {
    __syncwarp();
    for (uint32_t j = lane; j < staged; j += 32)
      if (flushed + j < cp.C) {
        oi[flushed + j] = si[j];
        ob[flushed + j] = sb[j];
      }
    flushed += staged;
    staged = 0;
    __syncwarp();
  };
  double stk[24];
  stk[0] = 0.0;
  uint32_t mx = 0;
  for (uint32_t i = 0; i < nunits; ++i) {
    const uint64_t u = u0 + i;
    const uint64_t base = u * ROUND + 4 * lane;
    float4 acc[4];
    if ((u + 1) * ROUND <= n) {
      load_g<NP>(g, pr, base, acc);
      if (EF) {
        float4 rv[4];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) rv[ch] = __ldcs(reinterpret_cast<const float4*>(r + base + ch * 128));
#pragma unroll
        for (int ch = 0; ch < 4; ++ch)
          acc[ch] = make_float4(__fadd_rn(acc[ch].x, rv[ch].x), __fadd_rn(acc[ch].y, rv[ch].y),
                                __fadd_rn(acc[ch].z, rv[ch].z), __fadd_rn(acc[ch].w, rv[ch].w));
      }
      if (STORE) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) __stcs(reinterpret_cast<float4*>(accw + base + ch * 128), acc[ch]);
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
            if (EF) x = __fadd_rn(x, r[idx]);
            if (STORE) accw[idx] = x;
          }
          v[e] = x;
        }
        acc[ch] = make_float4(v[0], v[1], v[2], v[3]);
      }
    }
    if (cmp_on) {
      // element (ch, lane, e) has index u*512 + ch*128 + 4*lane + e: chunk-major, then lane, then
      // e is index order; one packed scan (a byte per chunk) places every hit of the unit
      uint32_t m = 0;
#pragma unroll
      for (int ch = 0; ch < 4; ++ch) {
        const uint32_t w4[4] = {__float_as_uint(acc[ch].x), __float_as_uint(acc[ch].y), __float_as_uint(acc[ch].z),
                                __float_as_uint(acc[ch].w)};
#pragma unroll
        for (int e = 0; e < 4; ++e) m |= ((uint32_t)(ckm1 - (int32_t)(w4[e] & 0x7FFFFFFFu)) >> 31) << (4 * ch + e);
      }
      if (__any_sync(0xffffffffu, m != 0u)) {
        const uint32_t packed = __popc(m & 0xFu) | (__popc((m >> 4) & 0xFu) << 8) | (__popc((m >> 8) & 0xFu) << 16) |
                                (__popc(m >> 12) << 24);
        uint32_t incl = packed;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl += o;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        const uint32_t excl = incl - packed;
        const uint32_t tu = (tot & 0xFFu) + ((tot >> 8) & 0xFFu) + ((tot >> 16) & 0xFFu) + (tot >> 24);
        if (staged + tu > SCAP) spill();
        // the unit's hits go to the warp's staging buffer (or, if more than it holds, straight to
        // the global entries); only this lane's hits are visited (usually none or one): chunk
        // ch's run starts at b0 + hits of the earlier chunks, then the earlier lanes' hits of
        // chunk ch, then this lane's earlier hits in the chunk
        const bool direct = tu > SCAP;
        const uint32_t b0 = direct ? flushed : staged;
        const uint32_t t0 = tot & 0xFFu, t1 = (tot >> 8) & 0xFFu, t2 = (tot >> 16) & 0xFFu;
        for (uint32_t mm = m; mm; mm &= mm - 1u) {
          const int j = __ffs(mm) - 1;
          const int ch = j >> 2, e = j & 3;
          const uint32_t cbase = b0 + (ch > 0 ? t0 : 0u) + (ch > 1 ? t1 : 0u) + (ch > 2 ? t2 : 0u);
          const uint32_t pos = cbase + ((excl >> (8 * ch)) & 0xFFu) + __popc(m & ((1u << j) - 1u) & (0xFu << (4 * ch)));
          const float4 a4 = ch == 0 ? acc[0] : (ch == 1 ? acc[1] : (ch == 2 ? acc[2] : acc[3]));
          const float av = e == 0 ? a4.x : (e == 1 ? a4.y : (e == 2 ? a4.z : a4.w));
          const uint32_t ii = (uint32_t)(u * ROUND + ch * 128 + 4 * lane + e);
          if (direct) {
            if (pos < cp.C) { oi[pos] = ii; ob[pos] = __float_as_uint(av); }
          } else {
            si[pos] = ii;
            sb[pos] = __float_as_uint(av);
          }
        }
        if (direct) flushed += tu; else staged += tu;
        __syncwarp();
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
  // entries that never left shared memory stay there; otherwise the rest follows the spilled ones
  const bool in_smem = cmp_on && flushed == 0;
  if (cmp_on && !in_smem) spill();
  const uint32_t ncomp = flushed + staged;
  int top = 0;
  while ((1u << top) < units_per_warp) ++top;
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) {
    // this run's aligned subtree of the canonical tree: to run_sum (balanced map) or, folded with
    // the CTA's other 7 runs, to run_sum[blockIdx.x] (identity map)
    if (!sp.fold && run >= 0) run_sum[run] = stk[top];
    s_ws[warp] = run >= 0 ? stk[top] : 0.0;
    s_wm[warp] = mx;
    es.n[warp] = cmp_on ? ncomp : 0u;
    es.in_smem[warp] = in_smem ? 1u : 0u;
    if (cmp_on) {
      cp.cnt[gw] = ncomp;
      if (ncomp > cp.C) atomicExch(overflow, seq);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t te = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) te += es.n[w];
    cta_ent[blockIdx.x] = te;
    if (sp.fold)
      run_sum[blockIdx.x] = __dadd_rn(__dadd_rn(__dadd_rn(s_ws[0], s_ws[1]), __dadd_rn(s_ws[2], s_ws[3])),
                                      __dadd_rn(__dadd_rn(s_ws[4], s_ws[5]), __dadd_rn(s_ws[6], s_ws[7])));
    uint32_t m = s_wm[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) m = max(m, s_wm[w]);
    cta_max[blockIdx.x] = m;
  }
}

// Root of the canonical tree: the CTA partials (identity map) or the run subtrees (balanced map)
// zero-padded to Lp = 2^j >= THREADS leaves (extra zero leaves never change a pairwise sum of
// non-negatives, Q3), then a-bar, u and the first pass's candidates.  stats_fold reads the
// partials and returns (S, u bits, entries) in thread 0.
__device__ __forceinline__ void stats_fold(const double* __restrict__ run_sum, const uint32_t* __restrict__ cta_max,
                                           const uint32_t* __restrict__ cta_ent, const SearchParams& sp, double& S_out,
                                           uint32_t& m_out, uint32_t& t_out) {
  // Leaves: the G CTA partials (identity map, sp.fold) or the R run subtrees (balanced map),
  // zero-padded to Lp = 2^j >= 256 leaves (extra zero leaves never change a pairwise sum of
  // non-negatives, Q3); <= 4096 of them (plan_launches).  Folded in the canonical pairs:
  //   fold: lane l of warp w holds its Lp/256 consecutive leaves (levels 1..), then xor shuffles;
  //   runs: row q of 32 consecutive leaves per warp, loaded coalesced (lane l: leaf q*32 + l),
  //         reduced by xor shuffles (levels 1-5), then the rows pairwise;
  // then thread 0 folds the 8 warps.
  __shared__ double s_v[WARPS];
  __shared__ uint32_t s_m[WARPS], s_n[WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nl = sp.fold ? gridDim.x : sp.R;
  uint32_t Lp = THREADS;
  while (Lp < nl) Lp <<= 1;
  const uint32_t G = Lp / THREADS;  // 1..16, a power of two
  uint32_t m2 = 0, ne = 0;
#pragma unroll 2  // (grid <= 512 CTAs: both rounds' loads in flight together)
  for (uint32_t b = tid; b < gridDim.x; b += THREADS) {
    m2 = max(m2, __ldcg(cta_max + b));
    ne += __ldcg(cta_ent + b);
  }
  double lv[16];
  if (sp.fold) {
    const uint32_t l0 = (uint32_t)tid * G;
#pragma unroll
    for (uint32_t q = 0; q < 16; ++q) lv[q] = (q < G && l0 + q < nl) ? __ldcg(run_sum + l0 + q) : 0.0;
#pragma unroll
    for (uint32_t w = 1; w < 16; w <<= 1)
#pragma unroll
      for (uint32_t q = 0; q < 16; q += 2 * w)
        if (w < G) lv[q] = __dadd_rn(lv[q], lv[q + w]);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) lv[0] = __dadd_rn(lv[0], __shfl_xor_sync(0xffffffffu, lv[0], off));
  } else {
#pragma unroll
    for (uint32_t q = 0; q < 16; ++q) {
      const uint32_t li = warp * (Lp / WARPS) + q * 32 + lane;
      lv[q] = (q < G && li < nl) ? __ldcg(run_sum + li) : 0.0;
    }
#pragma unroll
    for (uint32_t q = 0; q < 16; ++q)
      if (q < G) {
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) lv[q] = __dadd_rn(lv[q], __shfl_xor_sync(0xffffffffu, lv[q], off));
      }
#pragma unroll
    for (uint32_t w = 1; w < 16; w <<= 1)
#pragma unroll
      for (uint32_t q = 0; q < 16; q += 2 * w)
        if (w < G) lv[q] = __dadd_rn(lv[q], lv[q + w]);
  }
  const double v = lv[0];
  m2 = __reduce_max_sync(0xffffffffu, m2);
  ne = __reduce_add_sync(0xffffffffu, ne);
  if (lane == 0) { s_v[warp] = v; s_m[warp] = m2; s_n[warp] = ne; }
  __syncthreads();
  if (tid == 0) {
    static_assert(WARPS == 8, "the CTA-level fold below is written for 8 warps");
    const double S = __dadd_rn(__dadd_rn(__dadd_rn(s_v[0], s_v[1]), __dadd_rn(s_v[2], s_v[3])),
                               __dadd_rn(__dadd_rn(s_v[4], s_v[5]), __dadd_rn(s_v[6], s_v[7])));
    uint32_t m = s_m[0], t = s_n[0];
    for (int w = 1; w < WARPS; ++w) { m = max(m, s_m[w]); t += s_n[w]; }
    S_out = S;
    m_out = m;
    t_out = t;
  }
}

// Root after the grid barrier: every CTA folds the partials itself and finalises its own control
// block.  (Measured alternative: the CTA that arrives last folds and publishes the root through a
// flag - 0.3 us slower at C2, the flag round trip costs more than the shared L2 reads it saves.)
template <int SEL>
__device__ __forceinline__ void stats_root(const double* __restrict__ run_sum, const uint32_t* __restrict__ cta_max,
                                           const uint32_t* __restrict__ cta_ent, const SearchParams& sp, Ctrl* sc,
                                           uint64_t step) {
  __shared__ double s_S;
  __shared__ uint32_t s_mt[2];
  stats_fold(run_sum, cta_max, cta_ent, sp, s_S, s_mt[0], s_mt[1]);
  TK_TRACE(10);
  if (threadIdx.x == 0) {
    stats_finalize<SEL>(sc, sp, s_S, s_mt[0], step);
    sc->n_compacted = s_mt[1];  // entries the ef phase kept (statistics)
  }
  TK_TRACE(11);
  __syncthreads();
}

// ------------------------------------------------------------------------------------------
// Count passes (Alg. 1 l.10): one read of the data resolves LEV bisection levels at once - the
// T = 2^LEV - 1 candidate thresholds of those levels are counted together (integer keys, Q4) and
// Alg. 1 l.11-23 is replayed on the exact totals.  Three modes:
//   COUNT_FIRST   whole vector, LEV <= 2; also appends, per warp and in index order, every element
//                 at or above the compaction key (one of the candidate keys) to the warp's entries
//   COUNT_CAP     the warp's compacted entries only (exact when the bracket lies above the key), LEV <= 4
//   COUNT_FULL    whole vector, LEV <= 2 (the general path when the compacted one is not exact)
// Each element costs one compare-and-add per key.  Per-warp-slab counts are stored (wcnt) for the
// selection's prefix sums; per-CTA sums go to the pass's global totals.
// HBM/L2: 4 B/elem (FIRST, FULL), 4 B/entry (CAP); FIRST also writes 8 B per compacted entry.
enum { COUNT_FIRST = 0, COUNT_CAP = 1, COUNT_FULL = 2 };

template <int NK, int MODE>
__device__ __forceinline__ void count_phase(const float* __restrict__ acc, const Ctrl* sc, const SearchParams sp,
                                            uint32_t* __restrict__ wcnt, const Compact cp, uint32_t* totals,
                                            uint32_t* overflow, uint32_t seq, int pass) {
  constexpr int T = NK;  // keys counted in this pass
  __shared__ uint32_t s_cnt[WARPS][16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t km1[T];  // key - 1: a >= key  <=>  (key - 1 - a) < 0 (no overflow for 0 <= a, key < 2^31)
#pragma unroll
  for (int s = 0; s < T; ++s) km1[s] = (int32_t)sc->cand_key[s] - 1;
  const int32_t kcmp1 = (int32_t)sc->cmp_key - 1;
  const uint32_t gw = blockIdx.x * WARPS + warp;
  uint64_t lo, hi;
  warp_slab(sp, warp, lo, hi);
  const uint32_t* a32 = reinterpret_cast<const uint32_t*>(acc);
  uint32_t cnt[T];
#pragma unroll
  for (int s = 0; s < T; ++s) cnt[s] = 0;
  auto count1 = [&](uint32_t bits) {
    const int32_t a = (int32_t)(bits & 0x7FFFFFFFu);
#pragma unroll
    for (int s = 0; s < T; ++s) cnt[s] += (uint32_t)(km1[s] - a) >> 31;
  };
  if (MODE == COUNT_CAP) {
    const Entries e = warp_entries(cp, sc->cmp_bottom, gw, warp);
#pragma unroll 1
    for (uint32_t j = lane; j < e.n; j += 32) count1(e.b(j));
  } else {
    // Whole slab.  Lane l owns the 16 consecutive elements [16l, 16l + 16) of each 512-element
    // round (four 128-bit loads; a warp instruction touches every other 16 B, its neighbour
    // instruction the rest, through L1), so (lane, j) order is index order and the compaction
    // needs one warp scan per round.
    // The slab is walked from its END to its start: the slabs coincide with the ef phase's warp
    // runs, so the most recently written (still L2-resident) part of acc is read first.  The
    // compacted entries are therefore filled from the top of the warp's region downward and end
    // up in ascending index order in [C - count, C).
    uint32_t ncomp = 0;  // FIRST: entries kept by this warp so far
    // two rounds' entries with one warp scan (16-bit packed per-lane counts); round A holds the
    // higher indices so its block goes above round B's (entries descend from the region's top)
    auto append2 = [&](uint32_t ma, uint64_t ra, uint32_t mb, uint64_t rb) {
      if (!__any_sync(0xffffffffu, (ma | mb) != 0u)) return;
      const uint32_t ca = __popc(ma), cb = __popc(mb);
      const uint32_t packed = ca | (cb << 16);
      uint32_t incl = packed;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += o;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t excl = incl - packed;
      const uint32_t ta = tot & 0xFFFFu, tb = tot >> 16;
      uint32_t* oi = cp.idx + (size_t)gw * cp.C;
      uint32_t* ob = cp.bits + (size_t)gw * cp.C;
      int64_t pa = (int64_t)cp.C - (int64_t)ncomp - (int64_t)ta + (int64_t)(excl & 0xFFFFu);
      int64_t pb = (int64_t)cp.C - (int64_t)ncomp - (int64_t)ta - (int64_t)tb + (int64_t)(excl >> 16);
      const uint32_t ia = (uint32_t)(ra + 16 * lane), ib = (uint32_t)(rb + 16 * lane);
#pragma unroll 1
      for (uint32_t mm = ma; mm; mm &= mm - 1u) {
        const uint32_t j = __ffs(mm) - 1;
        if (pa >= 0) { oi[pa] = ia + j; ob[pa] = __ldg(a32 + ia + j); }
        ++pa;
      }
#pragma unroll 1
      for (uint32_t mm = mb; mm; mm &= mm - 1u) {
        const uint32_t j = __ffs(mm) - 1;
        if (pb >= 0) { oi[pb] = ib + j; ob[pb] = __ldg(a32 + ib + j); }
        ++pb;
      }
      ncomp += ta + tb;
    };
    auto round16 = [&](uint4 q0, uint4 q1, uint4 q2, uint4 q3) -> uint32_t {
      const uint32_t w[16] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w,
                              q2.x, q2.y, q2.z, q2.w, q3.x, q3.y, q3.z, q3.w};
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int32_t a = (int32_t)(w[j] & 0x7FFFFFFFu);
        const bool p0 = a > km1[0];  // key 0 (= the compaction key in the first pass)
        cnt[0] += p0 ? 1u : 0u;
        if (MODE == COUNT_FIRST && p0) m |= 1u << j;
#pragma unroll
        for (int s = 1; s < T; ++s) cnt[s] += (uint32_t)(km1[s] - a) >> 31;
      }
      return m;
    };
    const uint4* p4 = reinterpret_cast<const uint4*>(a32 + lo) + 4 * lane;
    const uint64_t nfull = (hi - lo) / ROUND;  // full rounds of this slab
    const uint64_t tbase = lo + nfull * ROUND;
    if (tbase < hi) {  // ragged tail round (end of the vector only): first, in reverse order
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint64_t i = tbase + 16 * lane + j;
        if (i < hi) {
          const int32_t a = (int32_t)(a32[i] & 0x7FFFFFFFu);
#pragma unroll
          for (int s = 0; s < T; ++s) cnt[s] += (uint32_t)(km1[s] - a) >> 31;
          if (MODE == COUNT_FIRST) m |= ((uint32_t)(kcmp1 - a) >> 31) << j;
        }
      }
      if (MODE == COUNT_FIRST) append2(m, tbase, 0u, 0u);
    }
    // two rounds of 128-bit loads in flight per lane while a round is counted (last round first)
    uint4 a0 = make_uint4(0u, 0u, 0u, 0u), a1 = a0, a2 = a0, a3 = a0, b0 = a0, b1 = a0, b2 = a0, b3 = a0;
#define TK_LOAD(q0, q1, q2, q3, r)   \
  do {                               \
    const uint4* p_ = p4 + (r) * 128; \
    q0 = p_[0];                      \
    q1 = p_[1];                      \
    q2 = p_[2];                      \
    q3 = p_[3];                      \
  } while (0)
    if (nfull > 0) TK_LOAD(a0, a1, a2, a3, nfull - 1);
    if (nfull > 1) TK_LOAD(b0, b1, b2, b3, nfull - 2);
    for (uint64_t i = 0; i < nfull; i += 2) {
      const uint32_t ma = round16(a0, a1, a2, a3);
      if (i + 2 < nfull) TK_LOAD(a0, a1, a2, a3, nfull - 3 - i);
      uint32_t mb = 0;
      if (i + 1 < nfull) {
        mb = round16(b0, b1, b2, b3);
        if (i + 3 < nfull) TK_LOAD(b0, b1, b2, b3, nfull - 4 - i);
      }
      // one append for the pair: round A (higher indices) above round B in the region
      if (MODE == COUNT_FIRST) append2(ma, lo + (nfull - 1 - i) * ROUND, mb, lo + (nfull - 2 - i) * ROUND);
    }
#undef TK_LOAD
    if (MODE == COUNT_FIRST && lane == 0) {
      cp.cnt[gw] = ncomp;
      if (ncomp > cp.C) atomicExch(overflow, seq);
    }
  }
  // warp totals -> per-slab counts and the CTA's contribution to the pass totals
#pragma unroll
  for (int s = 0; s < T; ++s) {
    const uint32_t t = __reduce_add_sync(0xffffffffu, cnt[s]);
    if (lane == 0) {
      wcnt[(size_t)(pass * TMAX + s) * sp.W + gw] = t;
      s_cnt[warp][s] = t;
    }
  }
  __syncthreads();
  if (threadIdx.x < T) {
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) tot += s_cnt[w][threadIdx.x];
    atomicAdd(&totals[(blockIdx.x & (HREP - 1)) * TOT_STRIDE + threadIdx.x], tot);
  }
  __syncthreads();
}

// COUNT_HIST (compacted entries, up to HIST_LEV levels in ONE pass): the T = 2^LEV - 1 sorted
// candidate keys sit in shared memory; each entry finds its bucket b = #{s : key_s <= a} by a
// LEV-step binary search and bumps a per-warp shared-memory histogram; the CTA histogram is added
// to the pass's global histogram; after the barrier nnz_s = sum_{b > s} hist[b] (exact).
struct HistSmem {
  uint32_t h[HIST_BINS];  // the CTA's histogram (shared-memory atomics; entries spread over the bins)
};

// suf (optional): this CTA's suffix sums S[b] = sum_{b' >= b} h[b'] of its own histogram, so that
// after the replay each CTA can read the class counts of the CTAs before it without another
// grid barrier (#entries of CTA c at or above candidate s = S_c[s + 1]).
__device__ __forceinline__ void hist_phase(const Ctrl* sc, const Compact cp, uint32_t* ghist, HistSmem& hs, int LEV,
                                           uint32_t* suf = nullptr) {
  // LEV is a runtime value: one copy of this once-per-launch code instead of ten (code size and
  // register pressure of the whole kernel)
  const int NB = 1 << LEV;
  const int32_t* s_key = reinterpret_cast<const int32_t*>(sc->cand_key);  // sorted, in shared memory
  uint32_t* s_h = hs.h;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TK_TRACE(20);
  for (int i = threadIdx.x; i < NB; i += THREADS) s_h[i] = 0u;
  __syncthreads();
  TK_TRACE(21);
  const uint32_t gw = blockIdx.x * WARPS + warp;
  const Entries e = warp_entries(cp, sc->cmp_bottom, gw, warp);
  const uint32_t ne = e.n;
  auto add = [&](uint32_t bits) {
    const int32_t a = (int32_t)(bits & 0x7FFFFFFFu);
    uint32_t b = 0;
#pragma unroll 1
    for (int l = LEV - 1; l >= 0; --l) b += (a >= s_key[b + (1u << l) - 1]) ? (1u << l) : 0u;
    // warp-aggregated: the entries crowd into the few bins just above the compaction key
    const uint32_t peers = __match_any_sync(__activemask(), b);
    if ((__ffs(peers) - 1) == (threadIdx.x & 31)) atomicAdd(&s_h[b], (uint32_t)__popc(peers));
  };
  // a warp holds few entries in the EF-pass regime (~15 at C2): one per lane per iteration keeps
  // this once-per-launch code small (its instructions are fetched cold every launch)
#pragma unroll 1
  for (uint32_t j = lane; j < ne; j += 32) add(e.b(j));
  __syncthreads();
  TK_TRACE(22);
  for (int b = threadIdx.x; b < NB; b += THREADS) {
    const uint32_t t = s_h[b];
    if (b > 0 && t) atomicAdd(ghist + (blockIdx.x & (HREP - 1)) * TOT_STRIDE + b, t);  // bucket 0 is never needed
  }
  TK_TRACE(23);
  if (suf) {
    __shared__ uint32_t s_sw[WARPS];
    uint32_t v[4], sum = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int b = NB - 1 - (4 * (int)threadIdx.x + q);
      v[q] = b >= 0 ? s_h[b] : 0u;
      sum += v[q];
    }
    uint32_t total;
    uint32_t acc = block_excl_scan(sum, s_sw, total);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int b = NB - 1 - (4 * (int)threadIdx.x + q);
      acc += v[q];
      if (b >= 0) suf[b] = acc;
    }
  }
  __syncthreads();
}

// the first nk pass totals (summed over the HREP copies) into shared memory
__device__ __forceinline__ void load_totals(const uint32_t* tot_p, int nk, uint32_t* s_tot) {
  if ((int)threadIdx.x < nk) {
    uint32_t v = 0u;
    for (int c = 0; c < HREP; ++c) v += __ldcg(tot_p + c * TOT_STRIDE + threadIdx.x);
    s_tot[threadIdx.x] = v;
  }
  __syncthreads();
}

// nnz of every candidate from the global histogram: nnz_s = sum_{b >= s+1} hist[b].  Thread t
// owns the reversed positions 4t..4t+3 (bins NB-1-4t .. NB-4-4t); a block scan of the thread
// sums gives the suffix sums.
__device__ __forceinline__ void hist_to_counts(const uint32_t* ghist, int lev, uint32_t* s_tot) {
  __shared__ uint32_t s_w[WARPS];
  const int NB = 1 << lev;
  uint32_t x[4][HREP];  // every load issued before any is used
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int b = NB - 1 - (4 * (int)threadIdx.x + q);
#pragma unroll
    for (int c = 0; c < HREP; ++c) x[q][c] = b >= 1 ? __ldcg(ghist + c * TOT_STRIDE + b) : 0u;
  }
  uint32_t v[4], sum = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q] = 0u;
#pragma unroll
    for (int c = 0; c < HREP; ++c) v[q] += x[q][c];
    sum += v[q];
  }
  TK_TRACE(14);
  uint32_t total;
  uint32_t acc = block_excl_scan(sum, s_w, total);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int b = NB - 1 - (4 * (int)threadIdx.x + q);
    acc += v[q];
    if (b >= 1) s_tot[b - 1] = acc;  // sum over bins b..NB-1 = nnz of candidate b-1
  }
  __syncthreads();
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
// Where a selected pair goes (A7) and what stays in the residual (A8).  FP16 wire values (F3,
// reading Q31): the value sent is v16 = fp16_RN(clamp(v, +-65504)); the residual keeps
// fl32(v - v16) instead of +0.
struct SelOut {
  uint32_t* idx;
  float* val;       // fp32 value sent (optional)
  uint16_t* val16;  // binary16 value sent (optional; FP16 wire)
  float* r;         // residual write-back (EF; nullptr without)
  float* out;       // P = 1: the dense aggregate (Alg. 2 l.15-20 with one chunk: out[i] = +0 + sent)
  uint32_t w16;
};

__device__ __forceinline__ void put_sel(const SelOut& o, uint32_t pos, uint32_t i, float v) {
  o.idx[pos] = i;
  float sent = v;
  if (o.w16) {
    const __half h = __float2half_rn(fminf(fmaxf(v, -65504.0f), 65504.0f));
    sent = __half2float(h);
    if (o.val16) o.val16[pos] = __half_as_ushort(h);
  }
  if (o.val) o.val[pos] = sent;
  if (o.r) o.r[i] = o.w16 ? __fsub_rn(v, sent) : 0.0f;
  if (o.out) o.out[i] = __fadd_rn(0.0f, sent);
}

__device__ __forceinline__ void select_phase(const float* __restrict__ acc, const Ctrl* c, const SearchParams sp,
                                          uint32_t c1, uint32_t c2, uint32_t b1, uint32_t b2, const SelOut& so,
                                          const Compact cp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gw = blockIdx.x * WARPS + warp;
  uint64_t lo, hi;
  warp_slab(sp, warp, lo, hi);
  TK_TRACE(12);
  if (lo >= hi) return;
  const int32_t p1 = c->prov1, p2 = c->prov2;
  const int32_t key1 = (p1 >= 0) ? (int32_t)c->key1 : (int32_t)INF_BITS;
  const int32_t key2 = (p2 >= 0) ? (int32_t)c->key2 : 0;
  const uint32_t rnd = (uint32_t)c->rand, need = c->need;
  if (c1 == 0 && (c2 == 0 || b2 >= rnd + need || b2 + c2 <= rnd)) return;  // nothing kept here
  if (c->cap_ok) {
    // ---- compacted entries of this warp (ascending index order): 128 per iteration, lane l
    // holds entries 4l..4l+3 of the group, so (lane, e) order is index order ----
    const Entries en = warp_entries(cp, c->cmp_bottom, gw, warp);
    const uint32_t ne = en.n;
    for (uint32_t j0 = 0; j0 < ne; j0 += 128) {
      const uint32_t j = j0 + 4 * lane;
      uint32_t bb[4] = {0u, 0u, 0u, 0u}, ii[4] = {0u, 0u, 0u, 0u};
      if (j + 4 <= ne) {
        const uint4 q = en.b4(j);
        const uint4 x = en.i4(j);
        bb[0] = q.x; bb[1] = q.y; bb[2] = q.z; bb[3] = q.w;
        ii[0] = x.x; ii[1] = x.y; ii[2] = x.z; ii[3] = x.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (j + e < ne) { bb[e] = en.b(j + e); ii[e] = en.i(j + e); }
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
      // one put_sel per element (this once-per-launch code is fetched cold: keep it small)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t x1 = (fc1 >> e) & 1u, x2 = (fc2 >> e) & 1u;
        uint32_t pos = 0xFFFFFFFFu;
        if (x1) pos = q1 + ((q2 > rnd) ? min(q2 - rnd, need) : 0u);
        else if (x2 && q2 >= rnd && q2 < rnd + need) pos = q1 + (q2 - rnd);
        q1 += x1;
        q2 += x2;
        if (pos != 0xFFFFFFFFu) {
          TK_DCHECK(pos < sp.k && ii[e] < sp.n, "sel-cap", pos, ii[e]);
          put_sel(so, pos, ii[e], __uint_as_float(bb[e]));
        }
      }
      b1 += tot & 0xFFFFu;
      b2 += tot >> 16;
    }
    TK_TRACE(13);
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
          TK_DCHECK(pos < sp.k && i < sp.n, "sel-full1", pos, i);
          put_sel(so, pos, i, __uint_as_float(__ldg(a32 + i)));
          ++q1;
        } else {
          if (q2 >= rnd && q2 < rnd + need) {
            const uint32_t pos = q1 + (q2 - rnd);
            TK_DCHECK(pos < sp.k && i < sp.n, "sel-full2", pos, i);
            put_sel(so, pos, i, __uint_as_float(__ldg(a32 + i)));
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
// The whole compression (A1-A8) as ONE persistent cooperative kernel: the phases above, separated
// by grid barriers.  After each barrier every CTA runs the scalar control of Alg. 1 itself, on
// its own shared-memory copy of the control block, from the same global totals - so every CTA
// takes the same decisions and no serial tail, ticket or extra launch is needed.

struct Fused {
  SearchParams sp;
  PushOut push;              // np == 0: no fused all-gather
  const float* g;            // gradient (flat) - unused when the peers supply it
  Peers pr;                  // HiTopKComm ordered reduce-scatter sources
  float* r;                  // residual in, acc / r' out (EF); nullptr without EF
  float* accw;               // where the ef phase stores acc: r (EF), a scratch segment (peer sum
                             // without EF), nullptr (acc = g)
  const float* acc;          // the vector MSTopK reads: accw or g
  uint32_t units_per_warp;   // ef phase: aligned power-of-two run of 512-element units per warp
  double* cta_sum;           // [R] ef partials: one aligned canonical-tree subtree per run
  uint32_t* cta_max;         // [grid]
  uint32_t* wcnt;            // [npass * TMAX][W] per-warp-slab trial counts
  uint32_t* totals;          // [npass][16] global trial counts
  uint32_t* cta_cls;         // [2][grid] per-CTA class-1 / class-2 counts
  uint64_t* bar;             // grid barrier: monotonic arrival counter
  uint32_t* flags;           // overflow flags [0] first pass, [1] exact retry, [2] ef phase: each holds
                             // the sequence number of the last launch that overflowed (never cleared)
  uint32_t seq;              // this launch's sequence number (never 0)
  uint32_t exact_counts;     // count every trial exactly (an extra whole-vector pass when the fast
                             // search skipped the counts of trials below the ef-phase key)
  Compact cp;
  uint32_t* idx_out;
  float* val_out;
  Ctrl* c;                   // the control block (stats / next call's bracket prediction)
  uint64_t step;
  uint32_t n_iters;          // N
  int lev0;                  // levels of the first (whole-vector) pass: min(2, N, cap_levels)
  int cap_levels;            // max levels per later pass on compacted entries (whole-vector: <= 2)
  int max_pass;              // passes for which totals / wcnt are allocated
  uint32_t ef_compact;       // 1: compact in the ef phase at the key the previous call predicted
  uint16_t* val16_out;       // FP16 wire: binary16 values of the selection (nullptr: none)
  uint32_t* cta_suffix;      // [grid][HIST_BINS] per-CTA histogram suffix sums (barrier-free prefix)
  uint32_t wire16;           // FP16 wire values (F3): round the values sent, keep the error in r
  float* out_dense;          // P = 1 tk_step without the fused update: the dense aggregate, which this
                             // kernel writes whole (zeros after its last grid barrier, then the k values)
  uint32_t out_values;       // 1: the selection writes the values into out_dense (P = 1; no decompression)
};

// Grid-wide barrier (the launch is cooperative: every CTA is resident) on a monotonic 64-bit
// arrival counter that is never reset: barrier number e of the context completes when the counter
// reaches e * gridDim.x.  Thread 0 of each CTA arrives with a release reduction (cumulative over
// the CTA's writes, which __syncthreads orders before it) and polls with acquire loads; the
// following __syncthreads extends the acquire to the CTA.  No fence, exchange or generation word:
// 1.6 us per barrier on 444 CTAs vs 2.7 us for a reset-counter barrier with full fences
// (tools/barrier_bench2.cu).  target (thread 0 only) holds e * gridDim.x.
__device__ __forceinline__ void grid_sync(uint64_t* ctr, uint64_t& target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += gridDim.x;
#ifdef TK_BARRIER_FENCED  // experiment: full fences and a volatile poll (the round-1 barrier's ordering)
    __threadfence();
    atomicAdd(reinterpret_cast<unsigned long long*>(ctr), 1ull);
    while (*reinterpret_cast<volatile uint64_t*>(ctr) < target) __nanosleep(32);
    __threadfence();
#else
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
    // poll with relaxed loads (an acquire load invalidates the SM's whole L1 - the other CTAs'
    // cached lines and spilled registers - on every iteration), then one acquire fence
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    while (v < target) {
      __nanosleep(20);
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
#endif
  }
  __syncthreads();
}
// barriers completed before this launch: the counter lies in [B*G, B*G + G) until every CTA has
// arrived at this launch's first barrier, and each CTA reads it before its own first arrival
__device__ __forceinline__ uint64_t grid_sync_base(const uint64_t* ctr) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
  return v / gridDim.x * gridDim.x;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int NK, int MODE>
__device__ __forceinline__ void run_count(const Fused& f, Ctrl* sc, int pass) {
  count_phase<NK, MODE>(f.acc, sc, f.sp, f.wcnt, f.cp, f.totals + HIST_BINS * HREP * pass, f.flags, f.seq, pass);
}

// ------------------------------------------------------------------------------------------
// Exact selector (TK_SELECT_EXACT; Eq. 2, ties -> lower index, Q6): the k-th
// largest magnitude key T is found by narrowing an integer bracket [xlo, xhi) over the 31-bit key
// space with the same count / compaction / histogram passes: T = the largest key with
// #{a >= key} >= k.  Then class 1 = {a > T} (all kept), class 2 = {a == T} with the window at 0
// (the lowest indices), i.e. key1 = T + 1, key2 = T, rand = 0 in the MSTopK selection.

// bracket update from counted keys (one thread)
__device__ __forceinline__ void exact_update(Ctrl* c, const uint32_t* keys, const uint32_t* cnt, int nk, uint64_t k) {
  for (int s = 0; s < nk; ++s) {
    const uint32_t key = keys[s], n = cnt[s];
    if ((uint64_t)n >= k) {
      if (key > c->xlo) { c->xlo = key; c->xcnt_lo = n; }
    } else if (key < c->xhi) {
      c->xhi = key; c->xcnt_hi = n;
    }
  }
}

// nk keys splitting (xlo, xhi] evenly: xlo + ceil(j * w / (nk + 1)), j = 1..nk (ascending; with
// w <= nk + 1 they cover every key of the bracket, so a pass always narrows it)
__device__ __forceinline__ uint32_t exact_split(const Ctrl* c, uint32_t j, uint32_t parts) {
  // the first histogram pass after the EF-pass compaction spans only the predicted neighbourhood
  // [xlo, xguess] of T (keys above it count < k or not, either way the bracket narrows)
  const uint32_t hi = (c->xguess > c->xlo && c->xguess < c->xhi) ? c->xguess : c->xhi;
  const uint64_t w = (uint64_t)hi - c->xlo;
  return c->xlo + (uint32_t)((j * w + parts - 1) / parts);
}

#ifndef TK_MIN_BLOCKS
#define TK_MIN_BLOCKS 3
#endif

template <bool EF, int NP, int SEL>
__global__ void __launch_bounds__(THREADS, TK_MIN_BLOCKS) k_compress(Fused f) {
  static_assert(SEL == SEL_MSTOPK || SEL == SEL_EXACT || SEL == SEL_PROSE, "selector");
  __shared__ Ctrl sc;
  __shared__ uint32_t s_tot[HIST_BINS];
  __shared__ HistSmem s_hist;
  __shared__ uint32_t s_w[2][WARPS];
  __shared__ uint32_t s_base[2];
  __shared__ uint32_t s_ne[WARPS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // programmatic dependent launch: this grid may have been launched while the previous kernel on
  // the stream was finishing; nothing it wrote (nor anything before it) is read before this wait
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __shared__ uint64_t bar_t;  // thread 0: target of the next grid barrier (shared: keeps it out of registers)
  __shared__ uint64_t s_H;    // Alg. 1 l.27's random source for this call (window_hash)
  __shared__ int s_fast;      // the fast search's single pass took the selection's inputs from fast_walk
  __shared__ int s_zeroed;    // the dense aggregate's zeros were issued (flat tk_step)
  if (tid == 0) {
    s_fast = 0;
    s_zeroed = 0;
    bar_t = grid_sync_base(f.bar);
    s_H = window_hash(f.sp.seed, f.step, f.sp.rank);
  }
  if (lane == 0) g_es.run[warp] = warp_run_of(f.sp, blockIdx.x * WARPS + warp);
#ifdef TK_PHASE_TRACE
  if (tid == 0 && blockIdx.x < 2048) {
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_trace[1][30][blockIdx.x] = smid;
  }
#endif
  ctrl_to_smem(&sc, f.c);  // previous call's final state (bracket prediction)  (syncs the CTA)
  // Flat tk_step without the fused update: the dense aggregate (Alg. 2 l.15-20: +0 everywhere, then
  // the rank-ordered sums of the pairs) gets its zeros from this kernel, after its LAST grid barrier
  // (a barrier's release would wait for them) while HBM would otherwise idle through the rest of the
  // search and the selection.  Each warp zeroes its own slab, where its selection writes the values
  // afterwards (same warp: program order, __syncwarp and the CTA barriers in between order them).
  auto zero_out = [&]() {
    uint64_t zlo, zhi;
    warp_slab(f.sp, warp, zlo, zhi);
    float* o = f.out_dense;
    const uint64_t a4 = min(zhi, (uint64_t)((zlo + 3) & ~(uint64_t)3)), b4 = max(a4, (uint64_t)(zhi & ~(uint64_t)3));
    for (uint64_t i = zlo + lane; i < a4; i += 32) o[i] = 0.0f;
#pragma unroll 4
    for (uint64_t i = a4 + 4 * lane; i < b4; i += 128) __stcs(reinterpret_cast<float4*>(o + i), make_float4(0.f, 0.f, 0.f, 0.f));
    for (uint64_t i = b4 + lane; i < zhi; i += 32) o[i] = 0.0f;
    __syncwarp();
  };
  int nph = 0;
  auto gsync = [&]() __attribute__((always_inline)) {
#ifdef TK_PHASE_TRACE
    if (tid == 0 && nph < 32 && blockIdx.x < 2048) g_trace[1][nph][blockIdx.x] = globaltimer();
#endif
    grid_sync(f.bar, bar_t);
  };
  auto stamp = [&]() {
#ifdef TK_PHASE_TRACE
    if (tid == 0 && nph < 32 && blockIdx.x < 2048) g_trace[0][nph][blockIdx.x] = globaltimer();
#endif
    if (tid == 0 && nph < 12) sc.phase_ns[nph] = globaltimer();
    ++nph;
    sc.n_phase = (uint32_t)min(nph, 12);
  };
  stamp();
  for (int i = blockIdx.x * THREADS + tid; i < HIST_BINS * HREP * f.max_pass; i += gridDim.x * THREADS)
    f.totals[i] = 0u;
  if (blockIdx.x == 0 && tid == 0) {
    if (f.val16_out && (f.sp.k & 1u)) f.val16_out[f.sp.k] = 0u;  // FP16 wire: the chunk's padding half
  }
  // ---- A1-A2: error feedback, |acc| pairwise tree and max; compaction at the key the previous
  // call predicted (its entries replace the whole-vector first count pass when they are exact) ----
  const uint32_t efk = f.ef_compact ? sc.ef_key : 0u;
  uint32_t* cta_ent = f.cta_cls + 3 * gridDim.x;
  ef_phase<EF, NP>(f.g, f.pr, f.r, f.accw, f.sp, f.units_per_warp, f.cta_sum, f.cta_max, efk, f.cp, f.flags + 2,
                   f.seq, cta_ent);
  gsync();
  stamp();
  const uint32_t of2 = __ldcg(f.flags + 2);
  stats_root<SEL>(f.cta_sum, f.cta_max, cta_ent, f.sp, &sc, f.step);
  stamp();
  const bool ef_ok = efk > 0u && of2 != f.seq;  // entries = {a >= efk}, none dropped
  bool nobar = false;  // the cross-CTA prefix comes from the published histogram suffixes (no barrier)
  if (tid == 0) { sc.cmp_bottom = 0u; sc.cap_ok = 0u; sc.ef_used = 0u; sc.nnz_lb = 0ull; }
  __syncthreads();
  if constexpr (SEL == SEL_EXACT) {
    const uint64_t k = f.sp.k;
    __shared__ uint32_t s_e;
    if (ef_ok) {  // E = #{a >= efk}
      uint32_t e = 0;
      for (uint32_t b = tid; b < gridDim.x; b += THREADS) e += __ldcg(cta_ent + b);
      e = __reduce_add_sync(0xffffffffu, e);
      if (lane == 0) s_w[0][warp] = e;
      __syncthreads();
      if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < WARPS; ++w) t += s_w[0][w];
        s_e = t;
      }
      __syncthreads();
    }
    int p = 0;
    if (tid == 0) {
      sc.xlo = 0u; sc.xcnt_lo = (uint32_t)f.sp.n;
      sc.xhi = min(sc.umax_bits, 0x7FFFFFFFu) + 1u; sc.xcnt_hi = 0u;
      sc.xretry = 0u;
      sc.xguess = 0u;
      sc.it = 0u;
      if (ef_ok && (uint64_t)s_e >= k && efk < sc.xhi) {
        // T >= efk: the ef-phase entries hold every element the narrowing and the selection need
        sc.xlo = efk; sc.xcnt_lo = s_e;
        // T is expected near the previous T moved once more by its last move (error feedback
        // keeps it rising): the first histogram pass spans [efk, P + 2 * move + margin]
        const uint32_t P = sc.prev_T;
        const uint32_t mv = min(sc.prev_dT, 1u << 22);
        sc.xguess = (P > efk) ? P + 2u * mv + (1u << 12) : 0u;
        sc.cap_ok = 1u; sc.cmp_bottom = 1u; sc.ef_used = 1u;
      }
    }
    __syncthreads();
    if (!sc.ef_used) {
      // pass 0 (whole vector, compacting at key 0).  With a previous T: keys P - delta (the
      // compaction key), P - 8 delta (a fallback lower bound) and P + delta, delta = twice the last
      // move of T plus a margin; else u/4 (compaction key), u/2, u/8.  Any choice is exact: the
      // compaction is used only if its key turns out to lie at or below T and no warp overflowed.
      if (tid == 0) {
        const uint32_t P = sc.prev_T, u = sc.umax_bits;
        auto sub = [](uint32_t a, uint32_t b) { return a > b ? a - b : 0u; };
        if (P > 0u && P < sc.xhi) {
          const uint32_t delta = min(1u << 22, 2u * min(sc.prev_dT, 1u << 22) + (1u << 10));
          sc.cand_key[0] = sub(P, delta);
          sc.cand_key[1] = sub(P, 8u * delta);
          sc.cand_key[2] = min(P + delta, sc.xhi);
        } else {
          sc.cand_key[0] = sub(u, 2u << 23);
          sc.cand_key[1] = sub(u, 1u << 23);
          sc.cand_key[2] = sub(u, 3u << 23);
        }
        sc.cmp_key = sc.cand_key[0];
        sc.ncand = 3u;
      }
      __syncthreads();
      run_count<3, COUNT_FIRST>(f, &sc, 0);
      gsync();
      stamp();
      load_totals(f.totals, 3, s_tot);
      if (tid == 0) {
        exact_update(&sc, sc.cand_key, s_tot, 3, k);
        sc.cap_ok = ((uint64_t)s_tot[0] >= k && __ldcg(f.flags) != f.seq) ? 1u : 0u;
        sc.it = 1u;
      }
      __syncthreads();
      p = 1;
    }
    __shared__ int s_mode;
    while (sc.xhi > sc.xlo + 1u && p + 1 < f.max_pass) {
      uint32_t* tot_p = f.totals + HIST_BINS * HREP * p;
      if (tid == 0) {
        if (sc.cap_ok) {
          s_mode = 0;  // histogram of the compacted entries over 1023 keys splitting the bracket
        } else if (!sc.xretry && (uint64_t)sc.xcnt_lo * 8u <= f.sp.n) {
          s_mode = 1;  // compact again at xlo (<= T, so exact unless a warp overflows)
          sc.xretry = 1u;
        } else {
          s_mode = 2;  // whole-vector count of 3 keys
        }
      }
      __syncthreads();
      const int mode = s_mode;
      if (mode == 0) {
        for (int j = tid; j < HIST_BINS - 1; j += THREADS) sc.cand_key[j] = exact_split(&sc, j + 1, HIST_BINS);
        __syncthreads();
        hist_phase(&sc, f.cp, tot_p, s_hist, HIST_LEV);
      } else {
        if (tid == 0) {
          if (mode == 1) {
            sc.cand_key[0] = sc.xlo;
            sc.cand_key[1] = exact_split(&sc, 1, 3);
            sc.cand_key[2] = exact_split(&sc, 2, 3);
            sc.cmp_key = sc.xlo;
          } else {
            for (int j = 0; j < 3; ++j) sc.cand_key[j] = exact_split(&sc, j + 1, 4);
          }
        }
        __syncthreads();
        if (mode == 1)
          count_phase<3, COUNT_FIRST>(f.acc, &sc, f.sp, f.wcnt, f.cp, tot_p, f.flags + 1, f.seq, p);
        else
          run_count<3, COUNT_FULL>(f, &sc, p);
      }
      gsync();
      stamp();
      if (mode == 0) hist_to_counts(tot_p, HIST_LEV, s_tot);
      else load_totals(tot_p, 3, s_tot);
      if (tid == 0) {
        if (mode == 0) {
          // counts are non-increasing in the key: binary search for the last key with >= k
          int lo = -1, hi = HIST_BINS - 1;  // s_tot[lo] >= k (lo = -1: none), s_tot[hi] < k (hi = 1023: none)
          while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if ((uint64_t)s_tot[mid] >= k) lo = mid; else hi = mid;
          }
          if (lo >= 0) { sc.xlo = sc.cand_key[lo]; sc.xcnt_lo = s_tot[lo]; }
          if (hi < HIST_BINS - 1) { sc.xhi = sc.cand_key[hi]; sc.xcnt_hi = s_tot[hi]; }
          sc.xguess = 0u;
        } else {
          exact_update(&sc, sc.cand_key, s_tot, 3, k);
          if (mode == 1) sc.cap_ok = (__ldcg(f.flags + 1) != f.seq) ? 1u : 0u;
        }
        sc.it += 1u;
      }
      __syncthreads();
      ++p;
    }
    // T = xlo: #{a > T} = xcnt_hi, #{a >= T} = xcnt_lo
    if (!sc.cap_ok) {
      // per-warp counts of a > T and a >= T for the selection's prefix sums (whole vector)
      if (tid == 0) {
        sc.cand_key[0] = sc.xlo + 1u;
        sc.cand_key[1] = sc.xlo;
      }
      __syncthreads();
      run_count<2, COUNT_FULL>(f, &sc, p);
      gsync();
      stamp();
    }
    if (tid == 0) {
      const uint32_t T = sc.xlo;
      sc.k1 = sc.xcnt_hi;
      sc.k2 = sc.xcnt_lo;
      sc.key1 = T + 1u;
      sc.key2 = T;
      sc.thres1 = (double)__uint_as_float(T + 1u);
      sc.thres2 = (double)__uint_as_float(T);
      sc.prov1 = sc.cap_ok ? 0 : p * TMAX + 0;
      sc.prov2 = sc.cap_ok ? 0 : p * TMAX + 1;
      sc.need = (uint32_t)(k - sc.k1);
      sc.len2 = (uint64_t)sc.k2 - sc.k1;
      sc.rand = 0u;
      const uint32_t P = sc.prev_T;
      sc.prev_dT = (P > 0u) ? (T > P ? T - P : P - T) : (1u << 21);
      sc.prev_T = T;
      // next call's ef-phase compaction key: below T by half its last move if T rose (error
      // feedback grows the residual), else twice it, plus a margin
      // as for MSTopK's key2 below: twice the decaying maximum fall of T plus an eighth of its rise
      const uint32_t fall = (P > 0u) ? (T < P ? P - T : 0u) : (1u << 21);
      const uint32_t rise = (P > 0u && T > P) ? T - P : 0u;
      const uint32_t est = max(min(fall, 1u << 22), sc.mv_est - sc.mv_est / 4u);
      sc.mv_est = est;
      const uint32_t delta = min(1u << 22, 2u * est + (1u << 14) + rise / 8u);
      sc.ef_key = T > delta ? T - delta : 0u;
    }
    __syncthreads();
  } else {
  // ---- A3-A5: count passes.  A search runs passes from slot p0 until N levels are resolved.
  // fast: every pass is a histogram pass (up to HIST_LEV levels at once) over the ef-phase
  // entries {a >= efk}.  A count is exact for a key >= efk and a lower bound below it, so a
  // trial below efk can only err toward "nnz <= k" (hi := ratio), after which every later trial
  // and the final l lie below that key.  Hence the search is exact (same decisions, k1, k2,
  // thresholds, window and selection) iff thres2 ends up set with key2 >= efk - checked after
  // the search, with a full restart on failure.  The logged nnz of a trial below efk is then a
  // lower bound (> k); those trials are flagged in nnz_lb.  Otherwise the first
  // pass counts lev0 levels on the whole vector and compacts; when those entries are exact for
  // the rest, each further pass is a histogram pass on them, else it resolves up to 2 levels on
  // the whole vector.  The bits do not depend on this schedule. ----
  const int N = (int)f.n_iters;
  const bool single = N <= min(HIST_LEV, f.cap_levels);  // the fast search resolves all N levels in one pass
  __shared__ int s_got;
  // the search (always inlined: a call would spill the whole kernel's live state)
  auto search = [&](int p0, bool fast) __attribute__((always_inline)) -> int {
    int done = 0;
    int p = p0;
    if (fast) {
      make_candidates_par<SEL>(&sc, min(min(HIST_LEV, f.cap_levels), N));
      __syncthreads();
#ifdef TK_ICACHE_EXPERIMENT  // trace builds: the same (idempotent) work again, now with warm caches
      TK_TRACE(24);
      make_candidates_par<SEL>(&sc, min(min(HIST_LEV, f.cap_levels), N));
      __syncthreads();
      TK_TRACE(25);
#endif
    }
    for (; done < N; ++p) {
      int lev;
      bool hist = false;
      uint32_t* tot_p = f.totals + HIST_BINS * HREP * p;
      const bool first = (p == p0) && !fast;
      // the fast search's single pass also publishes this CTA's histogram suffix sums
      uint32_t* suf = (fast && single) ? f.cta_suffix + (size_t)blockIdx.x * HIST_BINS : nullptr;
      if (first) {
        lev = f.lev0;  // keys along the predicted path
        if (lev == 1) run_count<1, COUNT_FIRST>(f, &sc, p);
        else if (lev == 2) run_count<2, COUNT_FIRST>(f, &sc, p);
        else run_count<3, COUNT_FIRST>(f, &sc, p);
      } else if (sc.cap_ok) {
        hist = true;
        lev = min(min(HIST_LEV, f.cap_levels), N - done);
        hist_phase(&sc, f.cp, tot_p, s_hist, lev, suf);
      } else {
        lev = min(min(2, f.cap_levels), N - done);
        if (lev == 1) run_count<1, COUNT_FULL>(f, &sc, p); else run_count<3, COUNT_FULL>(f, &sc, p);
      }
      gsync();
      stamp();
      // the fast single pass's barrier is the last one when its decision holds (nearly always)
      if (f.out_dense && fast && single && SEL == SEL_MSTOPK && !f.exact_counts) {
        zero_out();
        if (tid == 0) s_zeroed = 1;  // read before the prefix, after several CTA barriers
      }
      if (hist) hist_to_counts(tot_p, lev, s_tot);
      else load_totals(tot_p, 16, s_tot);
      if (fast) stamp();
      if (SEL == SEL_MSTOPK && fast && single && !f.exact_counts) {
        // the single pass resolved all N levels: the selection's inputs come from fast_walk (every
        // thread, no serial replay on the critical path); block 0 replays the log after selecting
        const FastDecision fd = fast_walk(&sc, s_tot, lev, f.sp, efk, s_H);
        if (tid == 0 && fd.ok) {
          sc.k1 = fd.k1; sc.k2 = fd.k2; sc.key1 = fd.key1; sc.key2 = fd.key2;
          sc.prov1 = fd.s1 >= 0 ? p * TMAX + fd.s1 : -1;
          sc.prov2 = p * TMAX + fd.s2;
          sc.len2 = fd.w.len2; sc.need = (uint32_t)fd.w.need; sc.rand = fd.w.rand;
        }
        if (fd.ok) {
          s_fast = 1;  // (uniform: every thread took the same decision)
          stamp();
          return p + 1;
        }
      }
      if (tid == 0) {
        const double cmp_ratio = sc.cmp_ratio;
        s_got = replay_levels<SEL>(&sc, s_tot, min(lev, N - done), p, f.sp.k);
        if (first) {
          // compacted mode is exact iff every later threshold (and thres2) lies above the compaction
          // key: the bracket's lower end must have reached its coordinate, and nothing overflowed
          sc.cap_ok = (bracket_low_at_least<SEL>(&sc, cmp_ratio) && __ldcg(f.flags) != f.seq) ? 1u : 0u;
        }
        if (done + s_got == N) finish_window(&sc, f.sp, s_H);
      }
      __syncthreads();
      if (fast) stamp();
      done += s_got;
      if (done < N) {
        const int next = sc.cap_ok ? min(min(HIST_LEV, f.cap_levels), N - done) : min(min(2, f.cap_levels), N - done);
        make_candidates_par<SEL>(&sc, next);
        __syncthreads();
      }
    }
    return p;
  };
  int pnext = 0;
  bool ok = false;
  if (ef_ok) {
    if (tid == 0) { sc.cap_ok = 1u; sc.cmp_bottom = 1u; }
    __syncthreads();
    pnext = search(0, true);
    if (s_fast) {
      ok = true;
    } else {
    if (tid == 0) {
      s_got = (sc.prov2 >= 0 && sc.key2 >= efk) ? 1 : 0;  // the search was exact (see above)
      uint64_t lb = 0;
      for (uint32_t i = 0; i < sc.it && i < (uint32_t)NMAX; ++i)
        if (sc.key_log[i] < efk) lb |= 1ull << i;
      sc.nnz_lb = s_got ? lb : 0ull;
    }
    __syncthreads();
    ok = s_got != 0;
    }
  }
  if (!ok) {
    if (tid == 0) {
      search_reset<SEL>(&sc, f.sp.n);
      sc.nnz_lb = 0ull;
      sc.cap_ok = 0u;
      sc.cmp_bottom = 0u;
      first_pass_candidates<SEL>(&sc, f.lev0);
    }
    __syncthreads();
    pnext = search(pnext, false);
  }
  nobar = ok && single;
#ifndef TK_NO_EXACT_COUNTS
  if (f.exact_counts) {
    // exact_trial_counts: the trials the fast search only knows as "nnz > k" (key below the
    // ef-phase key) are counted exactly, up to 8 per whole-vector pass, before the selection
    // touches acc (Alg. 1 l.10 for every trial; the decisions were already exact)
    __shared__ int s_tr[8];
    __shared__ int s_nk;
    while (sc.nnz_lb != 0ull) {
      __syncthreads();
      if (tid == 0) {
        int nk = 0;
        for (uint32_t i = 0; i < sc.it && i < (uint32_t)NMAX && nk < 8; ++i)
          if (sc.nnz_lb >> i & 1ull) { s_tr[nk] = (int)i; sc.cand_key[nk] = sc.key_log[i]; ++nk; }
        for (int q = nk; q < 8; ++q) sc.cand_key[q] = INF_BITS;  // counts nothing (finite input)
        s_nk = nk;
      }
      __syncthreads();
      run_count<8, COUNT_FULL>(f, &sc, pnext);
      gsync();
      stamp();
      load_totals(f.totals + HIST_BINS * HREP * pnext, 8, s_tot);
      if (tid == 0) {
        for (int q = 0; q < s_nk; ++q) {
          sc.nnz_log[s_tr[q]] = s_tot[q];
          sc.nnz_lb &= ~(1ull << s_tr[q]);
        }
      }
      __syncthreads();
      ++pnext;
    }
  }
#endif
  if (tid == 0) {
    sc.ef_used = ok ? 1u : 0u;
    // next call's ef-phase compaction key: below this key2 by twice its last move plus a margin
    const uint32_t K = sc.key2;
    if (sc.prov2 >= 0) {
      const uint32_t P = sc.prev_key2;
      // The margin below key2 covers twice the largest recent FALL of key2 (a decaying maximum,
      // x3/4 per call) plus an eighth of this call's rise: a fall beyond it costs a whole-vector
      // restart (~100-200 us at C2), a margin too generous costs entries (the histogram, prefix and
      // selection work on them).  Measured: i.i.d. inputs without EF move key2 both ways by
      // ~20-60K ulps per call; with EF it keeps rising (by up to ~1M ulps per call for heavy tails).
      const uint32_t fall = (P > 0u) ? (K < P ? P - K : 0u) : (1u << 21);
      const uint32_t rise = (P > 0u && K > P) ? K - P : 0u;
      const uint32_t est = max(min(fall, 1u << 22), sc.mv_est - sc.mv_est / 4u);
      sc.mv_est = est;
      const uint32_t margin = min(1u << 22, 2u * est + (1u << 14) + rise / 8u);
      sc.ef_key = K > margin ? K - margin : 0u;
      sc.prev_key2 = K;
    } else {
      sc.ef_key = 0u;
      sc.prev_key2 = 0u;
    }
  }
  __syncthreads();
  }  // SEL_MSTOPK
  stamp();
  // ---- A7 prefix: class-1 / class-2 counts of each warp slab, then of the CTAs before it ----
  const uint32_t gw = blockIdx.x * WARPS + warp;
  const uint32_t W = f.sp.W;
  uint64_t slo, shi;
  warp_slab(f.sp, warp, slo, shi);
  if (f.out_dense && !s_zeroed) zero_out();  // (s_zeroed is uniform here: set before a CTA barrier, never after)
  uint32_t c1 = 0, call = 0;
  if (lane == 0) s_ne[warp] = 0u;
  if (sc.cap_ok) {
    // count the warp's compacted entries at key1 / key2 directly (exact: both keys lie at or
    // above every element excluded from the entries)
    const int32_t k1m1 = sc.prov1 >= 0 ? (int32_t)sc.key1 - 1 : 0x7FFFFFFF;
    const int32_t k2m1 = (int32_t)sc.key2 - 1;
    const Entries e = warp_entries(f.cp, sc.cmp_bottom, gw, warp);
    const uint32_t ne = e.n;
    if (lane == 0) s_ne[warp] = ne;
#pragma unroll 4
    for (uint32_t j = lane; j < ne; j += 32) {
      const int32_t a = (int32_t)(e.b(j) & 0x7FFFFFFFu);
      c1 += (uint32_t)(k1m1 - a) >> 31;
      call += (uint32_t)(k2m1 - a) >> 31;
    }
    c1 = __reduce_add_sync(0xffffffffu, c1);
    call = __reduce_add_sync(0xffffffffu, call);
  } else {
    c1 = sc.prov1 >= 0 ? __ldcg(f.wcnt + (size_t)sc.prov1 * W + gw) : 0u;
    call = sc.prov2 >= 0 ? __ldcg(f.wcnt + (size_t)sc.prov2 * W + gw) : (uint32_t)(shi - slo);
  }
  const uint32_t c2 = call - c1;
  if (lane == 0) {
    s_w[0][warp] = c1;
    s_w[1][warp] = c2;
  }
  __syncthreads();
  if (!nobar) {
    if (tid == 0) {
      uint32_t t1 = 0, t2 = 0, tn = 0;
      for (int w = 0; w < WARPS; ++w) { t1 += s_w[0][w]; t2 += s_w[1][w]; tn += s_ne[w]; }
      f.cta_cls[blockIdx.x] = t1;
      f.cta_cls[gridDim.x + blockIdx.x] = t2;
      f.cta_cls[2 * gridDim.x + blockIdx.x] = tn;  // compacted entries (statistics)
    }
    gsync();
  }
  stamp();
  {
    uint32_t a1 = 0, a2 = 0;
    if (nobar) {
      // class counts of the CTAs before this one, from their published histogram suffixes: key1 /
      // key2 are candidates s1 / s2 of the single pass (prov = pass 0 * TMAX + s)
      const int s1 = sc.prov1, s2 = sc.prov2;
#pragma unroll 2  // (grid <= 512 CTAs: both rounds' loads in flight together)
      for (uint32_t b = tid; b < blockIdx.x; b += THREADS) {
        const uint32_t* S = f.cta_suffix + (size_t)b * HIST_BINS;
        const uint32_t x1 = s1 >= 0 ? __ldcg(S + s1 + 1) : 0u;
        const uint32_t xa = __ldcg(S + s2 + 1);
        a1 += x1;
        a2 += xa - x1;
      }
    } else {
      for (uint32_t b = tid; b < blockIdx.x; b += THREADS) {
        a1 += __ldcg(f.cta_cls + b);
        a2 += __ldcg(f.cta_cls + gridDim.x + b);
      }
    }
    a1 = __reduce_add_sync(0xffffffffu, a1);
    a2 = __reduce_add_sync(0xffffffffu, a2);
    __shared__ uint32_t s_red[2][WARPS];
    if (lane == 0) { s_red[0][warp] = a1; s_red[1][warp] = a2; }
    __syncthreads();
    if (tid == 0) {
      uint32_t b1 = 0, b2 = 0;
      for (int w = 0; w < WARPS; ++w) { b1 += s_red[0][w]; b2 += s_red[1][w]; }
      s_base[0] = b1;
      s_base[1] = b2;
    }
    __syncthreads();
  }
  uint32_t b1 = s_base[0], b2 = s_base[1];
  for (int w = 0; w < warp; ++w) { b1 += s_w[0][w]; b2 += s_w[1][w]; }
  // the next kernel on the stream (the decompression) may start launching: its CTAs wait for this
  // grid's completion (griddepcontrol.wait) before reading anything
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- A7-A8: selection, compaction, residual write-back ----
  {
    SelOut so;
    so.idx = f.idx_out;
    so.val = f.val_out;
    so.val16 = f.val16_out;
    so.r = EF ? f.r : nullptr;
    so.out = f.out_values ? f.out_dense : nullptr;
    so.w16 = f.wire16;
    select_phase(f.acc, &sc, f.sp, c1, c2, b1, b2, so, f.cp);
  }
  stamp();
  if (f.push.np > 0) {
    // Fused all-gather.  The kept elements of this CTA occupy ONE contiguous run of output
    // positions: pos = #class1 before + clamp(#class2 before - rand, 0, need) is monotone and
    // steps by one per kept element.  Copy the run (written locally above) as tagged packets to
    // this rank's chunk on every GPU (peers over NVLink, coalesced 16-byte stores).
    uint32_t t1 = 0, t2 = 0;
    for (int w = 0; w < WARPS; ++w) { t1 += s_w[0][w]; t2 += s_w[1][w]; }
    const uint32_t rnd = sc.rand, need = sc.need;
    auto kept2 = [&](uint32_t q2) { return q2 > rnd ? min(q2 - rnd, need) : 0u; };
    const uint32_t p0 = s_base[0] + kept2(s_base[1]);
    const uint32_t p1 = s_base[0] + t1 + kept2(s_base[1] + t2);
    __syncthreads();
    for (uint32_t pos = p0 + tid; pos < p1; pos += THREADS) {
      const uint32_t i = __ldcg(f.idx_out + pos);
      const uint32_t v = f.val16_out ? __float_as_uint(__half2float(__ushort_as_half(__ldcg(f.val16_out + pos))))
                                     : __ldcg(reinterpret_cast<const uint32_t*>(f.val_out) + pos);
      for (uint32_t q = 0; q < f.push.np; ++q) st_ll(f.push.slot[q] + pos, i, v, f.push.tag);
    }
  }
  if (blockIdx.x == 0) {
    // entries the selection ran on (statistics): the ef phase's (summed in stats_root) or, on the
    // whole-vector path, the first count pass's (per CTA, from the prefix phase)
    if (!sc.ef_used) {
      uint32_t tn = 0;
      if (sc.cap_ok)
        for (uint32_t b = tid; b < gridDim.x; b += THREADS) tn += __ldcg(f.cta_cls + 2 * gridDim.x + b);
      tn = __reduce_add_sync(0xffffffffu, tn);
      if (lane == 0) s_w[0][warp] = tn;
      __syncthreads();
      if (tid == 0) {
        uint32_t t = 0;
        for (int w = 0; w < WARPS; ++w) t += s_w[0][w];
        sc.n_compacted = t;
      }
    }
    if constexpr (SEL == SEL_MSTOPK) {
      if (s_fast && tid == 0) {
        // the fast path selected from fast_walk's decisions: Alg. 1's trial log, thresholds and
        // bracket for the control block, by the same replay (identical decisions and results)
        search_reset<SEL>(&sc, f.sp.n);
        replay_levels<SEL>(&sc, s_tot, (int)f.n_iters, 0, f.sp.k);
        finish_window(&sc, f.sp, s_H);
        uint64_t lb = 0;
        for (uint32_t i = 0; i < sc.it && i < (uint32_t)NMAX; ++i)
          if (sc.key_log[i] < efk) lb |= 1ull << i;
        sc.nnz_lb = lb;
      }
    }
    ctrl_to_global(f.c, &sc);
  }
#ifdef TK_PHASE_TRACE
  __syncthreads();
  if (tid == 0 && blockIdx.x < 2048) g_trace[0][31][blockIdx.x] = globaltimer();  // end of this CTA
#endif
}

// ------------------------------------------------------------------------------------------
// Decompression (Alg. 2 l.15-20): out = +0; for p in rank order: out[idx_p] += val_p (fp32 RN).
// Tile-owner design: a persistent CTA owns a contiguous run of 4096-element output tiles; per
// tile it zero-fills shared memory, applies the ranks' pairs falling in the tile in rank order
// (one barrier per rank; indices within one rank are distinct so its adds never collide), and
// writes the tile once with streaming 128-bit stores.  Each rank's cursor only moves forward
// (chunks are ascending), found once per CTA by a warp-cooperative 32-ary search.  No global
// atomics, no read-modify-write of out.  HBM: 4 B/elem write + 8 B per gathered pair.

// first j in [0, n) with src.idx(p, j) >= target (n if none); all lanes of the warp participate
template <class Src>
__device__ uint32_t warp_lower_bound(const Src& src, uint32_t p, uint32_t n, uint32_t target) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = n;
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t pos = lo + lane * step;
    const uint32_t v = pos < hi ? src.idx(p, pos) : 0xFFFFFFFFu;
    const uint32_t m = __ballot_sync(0xffffffffu, v >= target);
    const uint32_t f = m ? (uint32_t)(__ffs(m) - 1) : 32u;
    if (f == 0) return lo;
    const uint32_t nlo = lo + (f - 1) * step + 1;
    const uint32_t nhi = (f < 32) ? min(hi, lo + f * step) : hi;
    lo = nlo;
    hi = nhi;
  }
  const uint32_t pos = lo + lane;
  const uint32_t v = pos < hi ? src.idx(p, pos) : 0xFFFFFFFFu;
  const uint32_t m = __ballot_sync(0xffffffffu, pos < hi && v >= target);
  return m ? lo + (uint32_t)(__ffs(m) - 1) : hi;
}

// Replicas of the decompressed output: every tile is also written to p[0..n) (e.g. the row peers'
// copies of this segment over NVLink: HiTopKComm's dense step 4 fused into step 3's accumulation,
// Alg. 2 l.15-23 - each GPU writes its aggregated segment straight into every node peer's output)
struct OutReplicas {
  float* p[8];
  uint32_t n;
};

// plain_out (optional): the consumed pairs re-emitted in the plain [nchunks][idx k | val k]
// layout (each pair lies in exactly one tile, so each is written exactly once)
// w (optional): the SGD update of Eq. 1 fused into the tile write-back,
// w_i := fl32(w_i - fl32(lr * out_i)) for every i (two RN operations, no FMA; reading Q29);
// out (optional when w is given) still receives the aggregate.
template <class Src>
__global__ void __launch_bounds__(THREADS) k_decompress(const Src src, uint32_t nchunks, uint64_t k, uint64_t n,
                                                        uint32_t ntiles, uint32_t tiles_per_cta,
                                                        float* __restrict__ out, uint32_t* __restrict__ plain_out,
                                                        float* __restrict__ w, float lr, uint64_t cw, uint32_t w16,
                                                        const OutReplicas rep) {
  __shared__ __align__(16) float s_tile[TILE];
  extern __shared__ uint32_t s_cur[];  // [nchunks] per-rank cursors
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // programmatic dependent launch (see k_compress): wait for the previous grid, then let the next
  // one start launching
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t t0 = blockIdx.x * tiles_per_cta;
  const uint32_t t1 = min(ntiles, t0 + tiles_per_cta);
  if (t0 >= t1) return;
  auto emit = [&](uint32_t p, uint32_t j, uint32_t i, float v) {
    if (plain_out) {
      plain_out[(size_t)p * cw + j] = i;
      if (w16) {
        uint16_t* h = reinterpret_cast<uint16_t*>(plain_out + (size_t)p * cw + k);
        h[j] = __half_as_ushort(__float2half_rn(v));
        if ((k & 1u) && j == k - 1) h[k] = 0u;  // the chunk's padding half
      }
      else
        plain_out[(size_t)p * cw + k + j] = __float_as_uint(v);
    }
  };
  for (uint32_t p = warp; p < nchunks; p += WARPS) {
    const uint32_t j = warp_lower_bound(src, p, (uint32_t)k, t0 * TILE);
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
      cur = s_cur[warp];
      const uint32_t j = cur + lane;
      if (j < k) src.get(warp, j, pi, pv);
      cnt = __popc(__ballot_sync(0xffffffffu, pi < thi));
    }
    for (int q = threadIdx.x; q < TILE / 4; q += THREADS) s4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncthreads();
    for (uint32_t p = 0; p < nchunks; ++p) {
      if ((uint32_t)warp == (p & (WARPS - 1))) {
        uint32_t c0;
        if (p < WARPS) {
          if (pi < thi && pi >= tlo) {  // (pi < tlo only for a packet that timed out: memory safety)
            s_tile[pi - tlo] = __fadd_rn(s_tile[pi - tlo], pv);
            emit(p, cur + lane, pi, pv);
          }
          c0 = cur + cnt;
        } else {
          c0 = s_cur[p];
        }
        if (p >= WARPS || cnt == 32) {  // more pairs of this rank in this tile
          for (;;) {
            const uint32_t j = c0 + lane;
            uint32_t i = NO_INDEX;
            float v = 0.0f;
            if (j < k) src.get(p, j, i, v);
            const bool in = i < thi;
            if (in && i >= tlo) {
              s_tile[i - tlo] = __fadd_rn(s_tile[i - tlo], v);
              emit(p, j, i, v);
            }
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
      if (out) {
        float4* o4 = reinterpret_cast<float4*>(out + tlo);
        for (int q = threadIdx.x; q < TILE / 4; q += THREADS) __stcs(o4 + q, s4[q]);
      }
#pragma unroll
      for (uint32_t r = 0; r < 8; ++r) {  // replicas (peer memory): 128-bit coalesced stores
        if (r < rep.n) {                   // (constant indices: rep stays in parameter space)
          float4* o4 = reinterpret_cast<float4*>(rep.p[r] + tlo);
          for (int q = threadIdx.x; q < TILE / 4; q += THREADS) __stcs(o4 + q, s4[q]);
        }
      }
      if (w) {
        float4* w4 = reinterpret_cast<float4*>(w + tlo);
        for (int q = threadIdx.x; q < TILE / 4; q += THREADS) {
          const float4 v = s4[q];
          float4 x = __ldcs(w4 + q);
          x.x = __fsub_rn(x.x, __fmul_rn(lr, v.x));
          x.y = __fsub_rn(x.y, __fmul_rn(lr, v.y));
          x.z = __fsub_rn(x.z, __fmul_rn(lr, v.z));
          x.w = __fsub_rn(x.w, __fmul_rn(lr, v.w));
          __stcs(w4 + q, x);
        }
      }
    } else {
      for (int q = threadIdx.x; q < TILE; q += THREADS)
        if ((uint64_t)tlo + q < n) {
          if (out) out[tlo + q] = s_tile[q];
#pragma unroll
          for (uint32_t r = 0; r < 8; ++r)
            if (r < rep.n) rep.p[r][tlo + q] = s_tile[q];
          if (w) w[tlo + q] = __fsub_rn(w[tlo + q], __fmul_rn(lr, s_tile[q]));
        }
    }
    __syncthreads();  // s_tile is rewritten by the next tile
  }
}

// The SGD update of Eq. 1 on a dense aggregate (HiTopKComm dense step 4, where the aggregate is
// only complete after the row all-gather): w_i := fl32(w_i - fl32(lr * out_i)).
__global__ void __launch_bounds__(THREADS) k_sgd_update(float* __restrict__ w, const float* __restrict__ out,
                                                        uint64_t n, float lr) {
  const uint64_t n4 = n / 4;
  const uint64_t stride = (uint64_t)gridDim.x * THREADS;
  for (uint64_t q = (uint64_t)blockIdx.x * THREADS + threadIdx.x; q < n4; q += stride) {
    const float4 v = __ldcs(reinterpret_cast<const float4*>(out) + q);
    float4 x = __ldcs(reinterpret_cast<const float4*>(w) + q);
    x.x = __fsub_rn(x.x, __fmul_rn(lr, v.x));
    x.y = __fsub_rn(x.y, __fmul_rn(lr, v.y));
    x.z = __fsub_rn(x.z, __fmul_rn(lr, v.z));
    x.w = __fsub_rn(x.w, __fmul_rn(lr, v.w));
    __stcs(reinterpret_cast<float4*>(w) + q, x);
  }
  for (uint64_t i = n4 * 4 + (uint64_t)blockIdx.x * THREADS + threadIdx.x; i < n; i += stride)
    w[i] = __fsub_rn(w[i], __fmul_rn(lr, out[i]));
}

// FP16 wire (F3): pack a selection into [idx k | binary16 val k (padded)] (values already fp16-exact)
__global__ void k_pack16(const uint32_t* __restrict__ idx, const float* __restrict__ val, uint32_t* __restrict__ out,
                         uint64_t k) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < k) {
    out[j] = idx[j];
    reinterpret_cast<uint16_t*>(out + k)[j] = __half_as_ushort(__float2half_rn(val[j]));
  }
  if (j == 0 && (k & 1)) reinterpret_cast<uint16_t*>(out + k)[k] = 0;  // padding half
}

// Debug (TK_CHECK=1): a selection / gathered chunk must hold strictly ascending indices < n.
__global__ void k_check_sel(const uint32_t* idx, uint64_t k, uint64_t n, uint32_t rank, uint32_t step, uint32_t where) {
  for (uint64_t j = threadIdx.x; j < k; j += blockDim.x) {
    const uint32_t i = idx[j];
    const bool bad = i >= n || (j > 0 && idx[j - 1] >= i);
    if (bad) {
      printf("TK_CHECK rank %u step %u where %u: j=%llu idx=%u prev=%u n=%llu k=%llu\n", rank, step, where,
             (unsigned long long)j, i, j > 0 ? idx[j - 1] : 0u, (unsigned long long)n, (unsigned long long)k);
      __trap();
    }
  }
}

}  // namespace tk
