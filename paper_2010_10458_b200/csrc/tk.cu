// tk.cu — libtk runtime: the C ABI declared in include/tk.h.
//
// Owns the per-context scratch (tile partials, per-tile trial counts, prefix sums, control
// block, packed send/receive buffers), the NCCL communicators (world; for HiTopKComm also the
// row comm of the n GPUs of a virtual node and the column comm of the m GPUs with the same
// position), and the launch sequence of one iteration.  Everything is enqueued on the caller's
// stream with no host synchronisation inside an iteration, so a whole tk_step is capturable in
// a CUDA graph by the caller (except with the push all-gather: its per-step packet tag is a
// kernel argument).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <type_traits>
#include <vector>

#include "tk.h"
#include "tk_kernels.cuh"

using namespace tk;

struct tk_ctx {
  tk_config cfg;
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t P = 1, m = 1, n = 1, rank = 0;
  uint32_t row_pos = 0, col_pos = 0;  // j = rank % n (position in the node), i = rank / n (node)
  uint64_t d = 0, L = 0, k = 0;       // L = d / n (segment length); k = k (flat) or k~ (HiTopK)
  uint64_t cw = 0;                    // u32 words per packed chunk: 2k (fp32 values) or k + ceil(k/2) (FP16 wire)
  uint32_t sms = 148;
  uint32_t grid = 0;                  // CTAs of the cooperative compression kernel
  uint32_t W = 0;                     // warp slabs
  uint64_t S = 0;                     // slab length
  uint32_t R = 0;                     // runs of S elements (<= W; warp_run spreads them over the warps)
  uint32_t occ_dec = 1;               // resident decompression CTAs per SM
  uint32_t levels = 4, npass = 0;
  uint32_t debug_check = 0;           // cfg.check_selection: verify every selection on the device
  uint32_t ef_compact = 1;            // compaction in the ef phase (cfg.disable_ef_compaction; bits unchanged)
  uint32_t seq = 0;                   // k_compress launch sequence number (overflow flags, never 0)
  uint32_t* dev_err = nullptr;        // device word: the fused all-gather's wait timed out (sticky)
  uint32_t timeout_sticky = 0;
  uint64_t timeout_ns = 0;
#ifdef TK_NO_PDL  // experiment builds
  bool pdl = false;
#else
  bool pdl = true;                    // programmatic dependent launch (falls back when refused)
#endif
  int lev_sched[NMAX];
  uint32_t units_per_warp = 1;        // ef phase: aligned power-of-two run of 512-element units per warp
  uint32_t* cta_cls = nullptr;        // [4][grid] per-CTA class counts, entries
  uint32_t* cta_suffix = nullptr;     // [grid][HIST_BINS] per-CTA histogram suffix sums
  uint32_t* totals = nullptr;         // [npass][HREP][256] pass totals / histograms
  uint64_t* bar = nullptr;            // grid barrier: monotonic arrival counter (never reset)
  uint32_t* flags = nullptr;          // overflow flags [4] (launch sequence numbers)
  double* cta_sum = nullptr;          // K1 per-CTA partial sums / maxima
  uint32_t* cta_max = nullptr;
  uint32_t* wcnt = nullptr;           // per-warp-slab counts [npass*TMAX][W]
  Compact cp;                         // compacted entries of the first count pass
  Ctrl* ctrl = nullptr;
  uint32_t* send = nullptr;      // [2k]
  uint32_t* recv = nullptr;      // flat: [P][2k]; HiTopK: [m][2k~]
  uint32_t* recv_row = nullptr;  // HiTopK sparse step 4: [n][m][2k~]
  float* seg = nullptr;          // HiTopK step-1 output [L]
  float* h_g = nullptr;          // tk_step_host device staging
  float* h_r = nullptr;
  float* h_out = nullptr;
  ncclComm_t world = nullptr, row = nullptr, col = nullptr;
  float* sym_g = nullptr;             // HiTopKComm ordered RS: this GPU's peer-visible gradient [d]
  float* peer_g[8] = {nullptr};       // row peers' sym_g (IPC-opened; [row_pos] = sym_g)
  struct Sym {                        // symmetric buffers (tk_alloc_symmetric): every row peer holds one
    char* base;                       // of the same size, allocated in the same collective order
    size_t bytes;
    char* peer[8];                    // [q] = row peer q's copy, IPC-opened ([row_pos] = base)
  };
  std::vector<Sym> syms;
  int32_t* sync_buf = nullptr;        // 4-byte buffer of the row barrier all-reduce
  ulonglong2* pg = nullptr;           // TK_AG_PUSH: [2][P][k] tagged packets (double-buffered)
  ulonglong2* peer_pg[8] = {nullptr}; // every rank's pg (IPC-opened; [rank] = pg)
  uint32_t push_seq = 0;              // completed pushed steps (the packets' tag is push_seq + 1)
  uint64_t step = 0;
  uint64_t launches = 0;
  uint32_t nonfinite_sticky = 0;
  // stage profiling (tk_profile_begin / tk_profile_end): events at stage boundaries
  cudaEvent_t* prof_ev = nullptr;
  uint8_t* prof_kind = nullptr;
  uint32_t prof_cap = 0, prof_n = 0;
  bool prof_on = false;
  uint32_t prof_launch[TK_NSTAGES] = {0};
  char err[512] = {0};
};

namespace {

tk_status fail(tk_ctx* c, tk_status s, const char* fmt, ...) {
  if (c) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(c->err, sizeof(c->err), fmt, ap);
    va_end(ap);
  }
  return s;
}

#define TK_CUDA(ctx, expr)                                                                     \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) return fail((ctx), TK_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

#define TK_NCCL(ctx, expr)                                                                     \
  do {                                                                                         \
    ncclResult_t r_ = (expr);                                                                  \
    if (r_ != ncclSuccess) return fail((ctx), TK_ERR_NCCL, "%s: %s", #expr, ncclGetErrorString(r_)); \
  } while (0)

#define TK_TRY(expr)               \
  do {                             \
    tk_status s_ = (expr);         \
    if (s_ != TK_OK) return s_;    \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

tk_status check_launch(tk_ctx* c, const char* what) {
  c->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(c, TK_ERR_CUDA, "launch %s: %s", what, cudaGetErrorString(e));
  return TK_OK;
}

// Launch one of libtk's kernels on the context stream with programmatic dependent launch (the grid
// may be scheduled while the previous kernel drains; every kernel opens with griddepcontrol.wait),
// cooperatively for k_compress.  A driver that refuses the attribute gets a plain launch.
tk_status launch(tk_ctx* c, const void* kern, dim3 grid, size_t smem, void** args, bool cooperative) {
  if (c->pdl) {
    cudaLaunchAttribute at[2];
    unsigned na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (cooperative) {
      at[na].id = cudaLaunchAttributeCooperative;
      at[na].val.cooperative = 1;
      ++na;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.gridDim = grid;
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cfg.attrs = at;
    cfg.numAttrs = na;
    if (cudaLaunchKernelExC(&cfg, kern, args) == cudaSuccess) return TK_OK;
    (void)cudaGetLastError();
    c->pdl = false;  // not supported here: plain launches from now on
  }
  if (cooperative) {
    TK_CUDA(c, cudaLaunchCooperativeKernel(kern, grid, dim3(THREADS), args, smem, c->stream));
  } else {
    TK_CUDA(c, cudaLaunchKernel(kern, grid, dim3(THREADS), args, smem, c->stream));
  }
  return TK_OK;
}

// Record a stage boundary: the interval since the previous mark is attributed to `kind`.
void mark(tk_ctx* c, int kind) {
  if (!c->prof_on || c->prof_n >= c->prof_cap) return;
  cudaEventRecord(c->prof_ev[c->prof_n], c->stream);
  c->prof_kind[c->prof_n] = (uint8_t)kind;
  c->prof_n++;
  if (kind > 0 && kind < TK_NSTAGES) c->prof_launch[kind]++;
}

SearchParams search_params(const tk_ctx* c) {
  SearchParams sp;
  sp.n = c->L;
  sp.k = c->k;
  sp.W = c->W;
  sp.S = c->S;
  sp.R = c->R;
  sp.fold = (uint64_t)c->R * 8 >= (uint64_t)c->W * 7 ? 1u : 0u;
  sp.rank = c->rank;
  sp.rand_mode = c->cfg.rand_mode;
  sp.seed = c->cfg.seed;
  return sp;
}

template <int SEL>
const void* compress_kernel_sel(bool ef, int np) {
  // NP: the number of gradient sources summed in the ef phase (0 = one plain vector)
#ifdef TK_ANALYZE  // register / spill analysis of one instantiation only (never a product build)
  return (ef && np == 0 && SEL == SEL_MSTOPK) ? reinterpret_cast<const void*>(&k_compress<true, 0, SEL_MSTOPK>) : nullptr;
#endif
  switch ((ef ? 100 : 0) + np) {
    case 100: return reinterpret_cast<const void*>(&k_compress<true, 0, SEL>);
    case 102: return reinterpret_cast<const void*>(&k_compress<true, 2, SEL>);
    case 104: return reinterpret_cast<const void*>(&k_compress<true, 4, SEL>);
    case 108: return reinterpret_cast<const void*>(&k_compress<true, 8, SEL>);
    case 0: return reinterpret_cast<const void*>(&k_compress<false, 0, SEL>);
    case 2: return reinterpret_cast<const void*>(&k_compress<false, 2, SEL>);
    case 4: return reinterpret_cast<const void*>(&k_compress<false, 4, SEL>);
    case 8: return reinterpret_cast<const void*>(&k_compress<false, 8, SEL>);
  }
  return nullptr;
}

const void* compress_kernel(bool ef, int np, uint32_t sel) {
  if (sel == TK_SELECT_EXACT) return compress_kernel_sel<SEL_EXACT>(ef, np);
  if (sel == TK_SELECT_PROSE) return compress_kernel_sel<SEL_PROSE>(ef, np);
  return compress_kernel_sel<SEL_MSTOPK>(ef, np);
}


// MSTopK on a vector of length L (= c->L) with error feedback: g (+ r) -> idx/val, as ONE
// cooperative launch of k_compress.  With peers != nullptr the gradient is the ordered sum of the
// np peer segments (HiTopKComm step 1).
tk_status compress_impl(tk_ctx* c, const float* g, float* r, uint32_t* idx, float* val, const Peers* peers = nullptr,
                        int np = 0, const PushOut* push = nullptr, uint16_t* val16 = nullptr,
                        float* out_dense = nullptr, bool out_values = false) {
  const bool ef = c->cfg.error_feedback != 0;
  Fused f;
  memset(&f, 0, sizeof(f));
  f.sp = search_params(c);
  f.g = g;
  if (peers) f.pr = *peers;
  f.r = ef ? r : nullptr;
  // acc lives in r (EF, in place), in the segment scratch (peer sum without EF) or is g itself
  f.accw = ef ? r : (np > 0 ? c->seg : nullptr);
  if (np > 0 && !ef && !c->seg) return fail(c, TK_ERR_STATE, "no scratch segment for the peer sum");
  f.acc = f.accw ? f.accw : g;
  if (++c->seq == 0) c->seq = 1;  // overflow flags hold the launch that raised them (0 = never)
  f.seq = c->seq;
  f.exact_counts = c->cfg.exact_trial_counts ? 1u : 0u;
  f.units_per_warp = c->units_per_warp;
  f.cta_sum = c->cta_sum;
  f.cta_max = c->cta_max;
  f.wcnt = c->wcnt;
  f.totals = c->totals;
  f.cta_cls = c->cta_cls;
  f.cta_suffix = c->cta_suffix;
  f.bar = c->bar;
  f.flags = c->flags;
  f.cp = c->cp;
  f.idx_out = idx;
  f.val_out = val;
  f.val16_out = val16;
  f.wire16 = c->cfg.wire == TK_WIRE_F16 ? 1u : 0u;
  if (push) f.push = *push;
  f.out_dense = out_dense;
  f.out_values = out_values ? 1u : 0u;
  f.c = c->ctrl;
  f.step = c->step;
  f.n_iters = c->cfg.n_iters;
  f.lev0 = c->lev_sched[0];
  f.cap_levels = (int)c->levels;
  f.max_pass = (int)c->npass;
  f.ef_compact = c->ef_compact;
  const void* kern = compress_kernel(ef, np, c->cfg.select);
  if (!kern) return fail(c, TK_ERR_CONFIG, "unsupported peer count %d", np);
  void* args[] = {&f};
  TK_TRY(launch(c, kern, dim3(c->grid), 0, args, true));
  if (c->debug_check) {
    k_check_sel<<<1, 1024, 0, c->stream>>>(idx, c->k, c->L, (uint32_t)c->rank, (uint32_t)c->step, 0u);
    TK_TRY(check_launch(c, "k_check_sel"));
  }
  TK_TRY(check_launch(c, "k_compress"));
  mark(c, TK_STAGE_COMPRESS);
  return TK_OK;
}

// Rank-ordered decompression of nchunks chunks of kk pairs into out[0, len), from plain chunks or
// (fused all-gather) from tagged packets, optionally re-emitting the pairs in the plain layout.
template <class Src>
tk_status decompress_impl(tk_ctx* c, const Src& src, uint32_t nchunks, uint64_t kk, uint64_t len, float* out,
                          uint32_t* plain_out = nullptr, float* w = nullptr, float lr = 0.0f,
                          const OutReplicas* reps = nullptr) {
  OutReplicas rp;
  memset(&rp, 0, sizeof(rp));
  if (reps) rp = *reps;
  const uint32_t nt = (uint32_t)((len + TILE - 1) / TILE);
  const uint32_t max_cta = c->sms * c->occ_dec;
  const uint32_t per = (nt + max_cta - 1) / max_cta;
  const uint32_t grid = (nt + per - 1) / per;
  if (c->debug_check) {
    if constexpr (std::is_same<Src, PlainChunks>::value || std::is_same<Src, PlainChunks16>::value)
      for (uint32_t p = 0; p < nchunks; ++p)
        k_check_sel<<<1, 1024, 0, c->stream>>>(src.g + (size_t)p * c->cw, kk, len, (uint32_t)c->rank, (uint32_t)c->step,
                                               1u + p);
  }
  const uint32_t w16 = c->cfg.wire == TK_WIRE_F16 ? 1u : 0u;
  const uint64_t cw = c->cw;
  void* args[] = {const_cast<Src*>(&src), &nchunks, &kk, &len, const_cast<uint32_t*>(&nt), const_cast<uint32_t*>(&per),
                  &out, &plain_out, &w, &lr, const_cast<uint64_t*>(&cw), const_cast<uint32_t*>(&w16), &rp};
  TK_TRY(launch(c, reinterpret_cast<const void*>(&k_decompress<Src>), dim3(grid), sizeof(uint32_t) * nchunks, args,
                false));
  TK_TRY(check_launch(c, "k_decompress"));
  mark(c, TK_STAGE_DECOMPRESS);
  return TK_OK;
}

// decompression of packed chunks in the context's wire format
tk_status decompress_plain(tk_ctx* c, const uint32_t* base, uint32_t nchunks, uint64_t len, float* out,
                           float* w = nullptr, float lr = 0.0f, const OutReplicas* reps = nullptr) {
  if (c->cfg.wire == TK_WIRE_F16)
    return decompress_impl(c, PlainChunks16{base, c->k, c->cw}, nchunks, c->k, len, out, nullptr, w, lr, reps);
  return decompress_impl(c, PlainChunks{base, c->k}, nchunks, c->k, len, out, nullptr, w, lr, reps);
}

// where the selection writes its values inside a packed chunk
struct ChunkOut {
  float* val;
  uint16_t* val16;
};
ChunkOut chunk_out(const tk_ctx* c, uint32_t* chunk) {
  if (c->cfg.wire == TK_WIRE_F16) return {nullptr, reinterpret_cast<uint16_t*>(chunk + c->k)};
  return {reinterpret_cast<float*>(chunk + c->k), nullptr};
}

template <typename T>
tk_status dev_alloc(tk_ctx* c, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * count);
  if (e != cudaSuccess) return fail(c, TK_ERR_NOMEM, "cudaMalloc(%zu B): %s", sizeof(T) * count, cudaGetErrorString(e));
  return TK_OK;
}

// Grid of the cooperative compression kernel (#SMs x resident CTAs), the warp-slab partition of
// the count and selection phases, the ef phase's units per warp, and the scratch they use.
tk_status plan_launches(tk_ctx* c) {
  int v = 0;
  TK_CUDA(c, cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, c->device));
  c->sms = (uint32_t)v;
  int occ = 1 << 30, o7 = 0;
  for (int np : {0, 2, 4, 8}) {  // every source count tk_compress_segment may launch
    const void* kern = compress_kernel(c->cfg.error_feedback != 0, np, c->cfg.select);
    if (!kern) return fail(c, TK_ERR_CONFIG, "unsupported peer count");
    int o = 0;
    TK_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, THREADS, 0));
    occ = std::min(occ, o);
  }
  TK_CUDA(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o7, k_decompress<PlainChunks>, THREADS, 64 * sizeof(uint32_t)));
  if (occ < 1) return fail(c, TK_ERR_CUDA, "k_compress cannot be resident");
  c->occ_dec = (uint32_t)std::max(1, o7);
  const uint64_t L = c->L;
  const uint64_t rounds = (L + ROUND - 1) / ROUND;
  // persistent cooperative grid: every CTA resident; no more CTAs than warp rounds of work
  // units per warp >= TK_MIN_UNITS_PER_WARP.  Measured at d = 1M / 4M (tools/c1_probe.py): 4 or 8
  // units per warp (61 / 31 CTAs at 1M) make the ef phase 2-3x slower than they save in the
  // barrier-bound tail, so every warp gets >= 1 unit and the grid stays as wide as the SMs allow
#ifndef TK_MIN_UNITS_PER_WARP
#define TK_MIN_UNITS_PER_WARP 1
#endif
  const uint64_t per_cta = (uint64_t)WARPS * TK_MIN_UNITS_PER_WARP;
  c->grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)c->sms * occ, (rounds + per_cta - 1) / per_cta));
  c->grid = std::min<uint32_t>(c->grid, 4096 / WARPS);  // stats_root folds <= 4096 run sums (R <= W)
  c->W = c->grid * WARPS;
  uint64_t upw = 1;  // ef phase: aligned power-of-two run of units per warp covering the vector
  while ((uint64_t)c->W * upw < rounds) upw <<= 1;
  c->units_per_warp = (uint32_t)upw;
  c->S = upw * ROUND;  // count / select slabs = the ef phase's warp runs (acc is re-read from L2)
  c->R = (uint32_t)((rounds + upw - 1) / upw);
  TK_TRY(dev_alloc(c, &c->cta_sum, c->W));  // one partial sum per run (R <= W)
  TK_TRY(dev_alloc(c, &c->cta_max, c->grid));
  TK_TRY(dev_alloc(c, &c->cta_cls, 4 * (size_t)c->grid));
  TK_TRY(dev_alloc(c, &c->cta_suffix, (size_t)c->grid * HIST_BINS));
  TK_TRY(dev_alloc(c, &c->totals, (size_t)HIST_BINS * HREP * c->npass));
  TK_TRY(dev_alloc(c, &c->bar, 1));
  TK_CUDA(c, cudaMemset(c->bar, 0, sizeof(uint64_t)));
  TK_TRY(dev_alloc(c, &c->flags, 4));
  TK_CUDA(c, cudaMemset(c->flags, 0, 4 * sizeof(uint32_t)));
  // compacted entries: capacity S/4 per warp slab (the whole-vector path covers an overflow)
  c->cp.C = (uint32_t)std::max<uint64_t>(4, (c->S / 4 + 3) / 4 * 4);
  TK_TRY(dev_alloc(c, &c->cp.idx, (size_t)c->W * c->cp.C));
  TK_TRY(dev_alloc(c, &c->cp.bits, (size_t)c->W * c->cp.C));
  TK_TRY(dev_alloc(c, &c->cp.cnt, c->W));
  return TK_OK;
}

// Map `mine` (a cudaMalloc'd buffer) of every rank of `comm` into this process through CUDA IPC:
// the 64-byte handles are exchanged with an NCCL all-gather; peers[me] = mine.
tk_status exchange_ipc(tk_ctx* c, ncclComm_t comm, uint32_t nr, uint32_t me, void* mine_ptr, void** peers) {
  cudaIpcMemHandle_t mine;
  TK_CUDA(c, cudaIpcGetMemHandle(&mine, mine_ptr));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  char* dev = nullptr;
  TK_TRY(dev_alloc(c, &dev, 64 * (size_t)(nr + 1)));
  TK_CUDA(c, cudaMemcpy(dev, &mine, 64, cudaMemcpyHostToDevice));
  ncclResult_t r = ncclAllGather(dev, dev + 64, 64, ncclChar, comm, c->stream);
  if (r != ncclSuccess) {
    cudaFree(dev);
    return fail(c, TK_ERR_NCCL, "handle all-gather: %s", ncclGetErrorString(r));
  }
  std::vector<cudaIpcMemHandle_t> all(nr);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaMemcpy(all.data(), dev + 64, 64 * (size_t)nr, cudaMemcpyDeviceToHost);
  cudaFree(dev);
  if (e != cudaSuccess) return fail(c, TK_ERR_CUDA, "handle exchange: %s", cudaGetErrorString(e));
  for (uint32_t q = 0; q < nr; ++q) {
    if (q == me) {
      peers[q] = mine_ptr;
      continue;
    }
    TK_CUDA(c, cudaIpcOpenMemHandle(&peers[q], all[q], cudaIpcMemLazyEnablePeerAccess));
  }
  return TK_OK;
}

// HiTopKComm ordered reduce-scatter: every GPU exposes a gradient buffer to its row peers.
tk_status open_row_peers(tk_ctx* c) {
  TK_TRY(dev_alloc(c, &c->sym_g, c->d));
  TK_TRY(dev_alloc(c, &c->sync_buf, 1));
  TK_CUDA(c, cudaMemset(c->sync_buf, 0, sizeof(int32_t)));
  void* peers[8] = {nullptr};
  TK_TRY(exchange_ipc(c, c->row, c->n, c->row_pos, c->sym_g, peers));
  for (uint32_t q = 0; q < c->n; ++q) c->peer_g[q] = static_cast<float*>(peers[q]);
  tk_ctx::Sym y;
  memset(&y, 0, sizeof(y));
  y.base = reinterpret_cast<char*>(c->sym_g);
  y.bytes = sizeof(float) * c->d;
  for (uint32_t q = 0; q < c->n; ++q) y.peer[q] = reinterpret_cast<char*>(peers[q]);
  c->syms.push_back(y);
  return TK_OK;
}

// Flat fused all-gather (TK_AG_PUSH): every rank exposes a double-buffered buffer of tagged
// packets [2][P][k] (16 B per pair, zeroed: tag 0 is never a step's tag); the compression writes
// its pairs straight into its chunk on every peer over NVLink (see PushOut).
tk_status open_push_peers(tk_ctx* c) {
  const size_t n = 2 * (size_t)c->P * c->k;
  TK_TRY(dev_alloc(c, &c->pg, n));
  TK_CUDA(c, cudaMemset(c->pg, 0, sizeof(ulonglong2) * n));
  void* peers[8] = {nullptr};
  TK_TRY(exchange_ipc(c, c->world, c->P, c->rank, c->pg, peers));
  for (uint32_t q = 0; q < c->P; ++q) c->peer_pg[q] = static_cast<ulonglong2*>(peers[q]);
  return TK_OK;
}

void free_all(tk_ctx* c) {
  void* ptrs[] = {c->cp.idx, c->cp.bits, c->cp.cnt, c->cta_sum, c->cta_max, c->cta_cls, c->cta_suffix, c->totals,
                  c->bar, c->flags, c->wcnt,
                  c->ctrl, c->send, c->recv,
                  c->recv_row, c->seg, c->h_g, c->h_r, c->h_out, c->dev_err};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (c->prof_ev) {
    for (uint32_t i = 0; i < c->prof_cap; ++i) cudaEventDestroy(c->prof_ev[i]);
    delete[] c->prof_ev;
    delete[] c->prof_kind;
  }
  for (auto& y : c->syms) {
    for (uint32_t q = 0; q < 8; ++q)
      if (y.peer[q] && y.peer[q] != y.base) cudaIpcCloseMemHandle(y.peer[q]);
    cudaFree(y.base);
  }
  c->syms.clear();
  for (uint32_t q = 0; q < 8; ++q)
    if (c->peer_pg[q] && c->peer_pg[q] != c->pg) cudaIpcCloseMemHandle(c->peer_pg[q]);
  if (c->pg) cudaFree(c->pg);
  if (c->sync_buf) cudaFree(c->sync_buf);
  if (c->row) ncclCommDestroy(c->row);
  if (c->col) ncclCommDestroy(c->col);
  if (c->world) ncclCommDestroy(c->world);
}

// the symmetric buffer holding [p, p + bytes), and p's offset in it (nullptr: none)
const tk_ctx::Sym* find_sym(const tk_ctx* c, const void* p, size_t bytes, size_t* off) {
  const char* q = static_cast<const char*>(p);
  for (const auto& y : c->syms)
    if (q >= y.base && q + bytes <= y.base + y.bytes) {
      *off = (size_t)(q - y.base);
      return &y;
    }
  return nullptr;
}

}  // namespace

extern "C" {

uint64_t tk_k(uint64_t d, double rho) {
  if (d == 0 || !(rho > 0.0) || rho > 1.0) return 0;
  const double prod = rho * (double)d;  // fl64(rho * d)
  const uint64_t k = (uint64_t)std::floor(prod);
  return k < 1 ? 1 : k;
}

tk_status tk_get_unique_id(uint8_t uid[128]) {
  if (!uid) return TK_ERR_INVALID_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return TK_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  memcpy(uid, &id, 128);
  return TK_OK;
}

tk_status tk_init(const tk_config* cfg, const uint8_t* uid, tk_stream_t stream, tk_ctx** out) {
  if (!cfg || !out) return TK_ERR_INVALID_ARG;
  *out = nullptr;
  const tk_config& k = *cfg;
  if (k.d == 0 || k.d >= (1ull << 32)) return TK_ERR_INVALID_ARG;
  if (k.k == 0 && (!(k.rho > 0.0) || k.rho > 1.0)) return TK_ERR_INVALID_ARG;
  if (k.n_iters < 1 || k.n_iters > (uint32_t)NMAX) return TK_ERR_INVALID_ARG;
  if (k.nranks < 1 || k.rank >= k.nranks) return TK_ERR_INVALID_ARG;
  if (k.rand_mode > 1 || k.step4 > 1 || k.levels_per_pass > 10 || k.rs_mode > 1 ||
      k.ag_mode > 1 || k.select > 2 || k.wire > 1 || k.exact_trial_counts > 1 || k.disable_ef_compaction > 1 ||
      k.first_pass_keys > 3 || k.check_selection > 1 || k.loopback > 1)
    return TK_ERR_INVALID_ARG;
  const uint32_t n = k.group_size == 0 ? 1 : k.group_size;
  if (k.nranks % n != 0) return TK_ERR_CONFIG;
  if (k.d % n != 0) return TK_ERR_CONFIG;
  if (n > 1 && (k.d / n) % 4 != 0) return TK_ERR_CONFIG;  // segments start 16-byte aligned (128-bit access)
  if (k.nranks > 1 && !uid && !k.loopback) return TK_ERR_CONFIG;
  if (n > 1 && k.rs_mode == TK_RS_ORDERED && n != 2 && n != 4 && n != 8) return TK_ERR_CONFIG;
  if (n == 1 && k.ag_mode == TK_AG_PUSH && k.nranks > 8) return TK_ERR_CONFIG;
  const uint64_t L = k.d / n;
  uint64_t kk = k.k;
  if (kk == 0) kk = tk_k(L, k.rho);
  if (kk < 1 || kk > L) return TK_ERR_RANGE;

  tk_ctx* c = new (std::nothrow) tk_ctx();
  if (!c) return TK_ERR_NOMEM;
  c->cfg = k;
  c->cfg.group_size = n;
  c->P = k.nranks;
  c->n = n;
  c->m = k.nranks / n;
  c->rank = k.rank;
  c->row_pos = k.rank % n;
  c->col_pos = k.rank / n;
  c->d = k.d;
  c->L = L;
  c->k = kk;
  c->stream = reinterpret_cast<cudaStream_t>(stream);
  c->levels = k.levels_per_pass == 0 ? 10 : k.levels_per_pass;
  // pass schedule (decided on the device): the first pass resolves min(2, levels) levels on the
  // whole vector; later passes take up to `levels` levels on the compacted entries, or up to 2 on
  // the whole vector.  Scratch is sized for the worst case (all passes on the whole vector).
  {
    // first pass: up to 3 keys along the predicted path (at least one level resolved)
    const uint32_t keys = k.first_pass_keys == 0 ? 3u : k.first_pass_keys;  // results do not depend on it
    const uint32_t first = std::min<uint32_t>(std::min<uint32_t>(keys, c->levels), k.n_iters);
    c->lev_sched[0] = (int)first;
    const uint32_t per = std::min<uint32_t>(2u, c->levels);
    c->npass = 1 + (k.n_iters - 1 + per - 1) / per;  // worst case: the first pass resolves one level
    // exact selector: <= 2 compacting passes + <= 16 whole-vector passes (2 bits each over the
    // 31-bit key space) + <= 4 histogram passes (8 bits each) + the final per-warp count
    if (k.select == TK_SELECT_EXACT) c->npass = 24;
    // an ef-phase search (>= 1 level per pass) may precede a restart; exact_trial_counts adds up
    // to ceil(NMAX / 8) whole-vector count passes
    else c->npass += k.n_iters + (NMAX + 7) / 8;
    c->ef_compact = k.disable_ef_compaction ? 0u : 1u;
    c->debug_check = k.check_selection;
    c->timeout_ns = (uint64_t)(k.push_timeout_ms == 0 ? 300000u : k.push_timeout_ms) * 1000000ull;
  }
  auto bail = [&](tk_status s) {
    free_all(c);
    // keep no context on failure; report through the return code only
    delete c;
    return s;
  };
  if (k.device >= 0) {
    if (cudaSetDevice(k.device) != cudaSuccess) return bail(TK_ERR_CUDA);
  }
  cudaGetDevice(&c->device);
  tk_status s;
  if ((s = plan_launches(c)) != TK_OK) return bail(s);
  if ((s = dev_alloc(c, &c->wcnt, (size_t)c->npass * TMAX * c->W)) != TK_OK) return bail(s);
  if ((s = dev_alloc(c, &c->ctrl, 1)) != TK_OK) return bail(s);
  if ((s = dev_alloc(c, &c->dev_err, 1)) != TK_OK) return bail(s);
  if (cudaMemset(c->dev_err, 0, sizeof(uint32_t)) != cudaSuccess) return bail(TK_ERR_CUDA);
  c->cw = (k.wire == TK_WIRE_F16) ? kk + (kk + 1) / 2 : 2 * kk;
  if ((s = dev_alloc(c, &c->send, c->cw)) != TK_OK) return bail(s);
  const uint32_t chunks_recv = (n == 1) ? c->P : c->m;
  if ((s = dev_alloc(c, &c->recv, (size_t)chunks_recv * c->cw)) != TK_OK) return bail(s);
  // scratch segment: the NCCL reduce-scatter's output, or where the peer-sum kernel stores acc
  // without error feedback (tk_compress_segment allocates it on first use in flat mode)
  if (n > 1 && (k.rs_mode == TK_RS_NCCL || !k.error_feedback))
    if ((s = dev_alloc(c, &c->seg, L)) != TK_OK) return bail(s);
  if (n > 1) {
    if (k.step4 == TK_STEP4_SPARSE)
      if ((s = dev_alloc(c, &c->recv_row, (size_t)n * c->m * c->cw)) != TK_OK) return bail(s);
  }
  if (cudaMemset(c->ctrl, 0, sizeof(Ctrl)) != cudaSuccess) return bail(TK_ERR_CUDA);
  if (c->P > 1 && !k.loopback) {
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    if (ncclCommInitRank(&c->world, (int)c->P, id, (int)c->rank) != ncclSuccess) return bail(TK_ERR_NCCL);
    if (n > 1) {
      if (ncclCommSplit(c->world, (int)(c->rank / n), (int)c->rank, &c->row, nullptr) != ncclSuccess)
        return bail(TK_ERR_NCCL);
      if (c->m > 1 &&
          ncclCommSplit(c->world, (int)(c->rank % n), (int)c->rank, &c->col, nullptr) != ncclSuccess)
        return bail(TK_ERR_NCCL);
      if (k.rs_mode == TK_RS_ORDERED && (s = open_row_peers(c)) != TK_OK) return bail(s);
    } else if (k.ag_mode == TK_AG_PUSH) {
      if ((s = open_push_peers(c)) != TK_OK) return bail(s);
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(TK_ERR_CUDA);
  *out = c;
  return TK_OK;
}

tk_status tk_compress(tk_ctx* c, const float* g, float* r, uint32_t* idx, float* val) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (c->n != 1) return fail(c, TK_ERR_STATE, "tk_compress is the flat-mode entry point (group_size == 1)");
  const bool ef = c->cfg.error_feedback != 0;
  if (!g || !idx || !val || (ef && !r)) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(g) || (ef && !aligned16(r))) return fail(c, TK_ERR_INVALID_ARG, "g/r must be 16-byte aligned");
  if ((const void*)g == (const void*)r) return fail(c, TK_ERR_INVALID_ARG, "g aliases r");
  TK_TRY(compress_impl(c, g, ef ? r : nullptr, idx, val));
  return TK_OK;
}

tk_status tk_compress_segment(tk_ctx* c, const float* const* src, uint32_t nsrc, float* r, uint32_t* idx,
                              float* val) {
  if (!c) return TK_ERR_INVALID_ARG;
  const bool ef = c->cfg.error_feedback != 0;
  if (!src || !idx || !val || (ef && !r)) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  if (nsrc != 1 && nsrc != 2 && nsrc != 4 && nsrc != 8) return fail(c, TK_ERR_INVALID_ARG, "nsrc must be 1, 2, 4 or 8");
  if (ef && !aligned16(r)) return fail(c, TK_ERR_INVALID_ARG, "r must be 16-byte aligned");
  Peers pr;
  memset(&pr, 0, sizeof(pr));
  for (uint32_t q = 0; q < nsrc; ++q) {
    if (!src[q]) return fail(c, TK_ERR_INVALID_ARG, "null source pointer");
    if (!aligned16(src[q])) return fail(c, TK_ERR_INVALID_ARG, "source %u must be 16-byte aligned", q);
    if (ef && (const void*)src[q] == (const void*)r) return fail(c, TK_ERR_INVALID_ARG, "a source aliases r");
    pr.p[q] = src[q];
  }
  if (nsrc == 1) return compress_impl(c, src[0], ef ? r : nullptr, idx, val);
  if (!ef && !c->seg) TK_TRY(dev_alloc(c, &c->seg, c->L));  // where the peer sum is stored without EF
  return compress_impl(c, nullptr, ef ? r : nullptr, idx, val, &pr, (int)nsrc);
}

tk_status tk_loopback_push(tk_ctx* c, const float* g, float* r, uint32_t* chunk, void* const* slots, uint32_t nslots,
                           uint32_t tag) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!c->cfg.loopback) return fail(c, TK_ERR_STATE, "tk_loopback_push needs a loopback context");
  if (c->n != 1) return fail(c, TK_ERR_STATE, "the fused all-gather is the flat mode's");
  const bool ef = c->cfg.error_feedback != 0;
  if (!g || !chunk || !slots || (ef && !r)) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  if (nslots < 1 || nslots > 8 || tag == 0) return fail(c, TK_ERR_INVALID_ARG, "nslots in [1, 8], tag != 0");
  if (!aligned16(g) || (ef && !aligned16(r))) return fail(c, TK_ERR_INVALID_ARG, "misaligned pointer");
  PushOut po;
  memset(&po, 0, sizeof(po));
  po.np = nslots;
  po.me = c->rank;
  po.tag = tag;
  for (uint32_t q = 0; q < nslots; ++q) {
    if (!slots[q] || !aligned16(slots[q])) return fail(c, TK_ERR_INVALID_ARG, "slot %u null or misaligned", q);
    po.slot[q] = static_cast<ulonglong2*>(slots[q]);
  }
  const ChunkOut co = chunk_out(c, chunk);
  return compress_impl(c, g, ef ? r : nullptr, chunk, co.val, nullptr, 0, &po, co.val16);
}

tk_status tk_loopback_decompress(tk_ctx* c, const void* packets, uint32_t nchunks, uint32_t tag, float* out,
                                 uint32_t* plain_out) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!c->cfg.loopback) return fail(c, TK_ERR_STATE, "tk_loopback_decompress needs a loopback context");
  if (!packets || !out) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(out) || !aligned16(packets)) return fail(c, TK_ERR_INVALID_ARG, "misaligned pointer");
  if (nchunks < 1 || nchunks > 4096 || tag == 0) return fail(c, TK_ERR_INVALID_ARG, "nchunks in [1, 4096], tag != 0");
  const uint64_t len = (c->n == 1) ? c->d : c->L;
  TaggedChunks src{static_cast<const ulonglong2*>(packets), c->k, tag, c->dev_err, c->timeout_ns};
  return decompress_impl(c, src, nchunks, c->k, len, out, plain_out);
}

tk_status tk_sparse_allgather(tk_ctx* c, const uint32_t* idx, const float* val, uint32_t* gathered) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!idx || !val || !gathered) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  const size_t kb = sizeof(uint32_t) * c->k;
  const uint32_t* src = c->send;
  if (c->cfg.wire == TK_WIRE_F16) {
    // FP16 wire: pack [idx | binary16 val] (the values tk_compress returned are already fp16-exact)
    k_pack16<<<(unsigned)((c->k + THREADS - 1) / THREADS), THREADS, 0, c->stream>>>(idx, val, c->send, c->k);
    TK_TRY(check_launch(c, "k_pack16"));
  } else if ((const void*)val == (const void*)(idx + c->k)) {
    src = idx;  // caller already holds the packed [idx | val] layout
  } else {
    TK_CUDA(c, cudaMemcpyAsync(c->send, idx, kb, cudaMemcpyDeviceToDevice, c->stream));
    TK_CUDA(c, cudaMemcpyAsync(c->send + c->k, val, kb, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (c->P == 1) {
    if (src != gathered)
      TK_CUDA(c, cudaMemcpyAsync(gathered, src, sizeof(uint32_t) * c->cw, cudaMemcpyDeviceToDevice, c->stream));
    return TK_OK;
  }
  ncclComm_t comm = (c->n == 1) ? c->world : c->col;
  if (!comm) return fail(c, TK_ERR_STATE, "no communicator for the sparse all-gather");
  TK_NCCL(c, ncclAllGather(src, gathered, c->cw, ncclUint32, comm, c->stream));
  return TK_OK;
}

tk_status tk_decompress(tk_ctx* c, const uint32_t* gathered, uint32_t nchunks, float* out) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!gathered || !out) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  if (!aligned16(out)) return fail(c, TK_ERR_INVALID_ARG, "out must be 16-byte aligned");
  if (nchunks < 1 || nchunks > 4096) return fail(c, TK_ERR_INVALID_ARG, "nchunks must lie in [1, 4096]");
  const uint64_t len = (c->n == 1) ? c->d : c->L;
  return decompress_plain(c, gathered, nchunks, len, out);
}

// One iteration (tk_step / tk_step_sgd).  w != nullptr: Eq. 1's update fused into the final
// decompression (out may then be nullptr, except for HiTopKComm dense step 4, which needs it).
static tk_status step_impl(tk_ctx* c, const float* g, float* r, float* out, uint32_t* gathered, float* w, float lr) {
  const bool ef = c->cfg.error_feedback != 0;
  if (c->cfg.loopback && c->P > 1) return fail(c, TK_ERR_STATE, "a loopback context has no communicators");
  if (!g || (!out && !w) || (ef && !r)) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  if (w && !aligned16(w)) return fail(c, TK_ERR_INVALID_ARG, "misaligned w");
  if (w && ((const void*)w == (const void*)g || (const void*)w == (const void*)r || (const void*)w == (const void*)out))
    return fail(c, TK_ERR_INVALID_ARG, "w must not alias g, r or out");
  if (!aligned16(g) || (out && !aligned16(out)) || (ef && !aligned16(r)))
    return fail(c, TK_ERR_INVALID_ARG, "misaligned pointer");
  if ((const void*)g == (const void*)r || (out && ((const void*)g == (const void*)out || (const void*)r == (const void*)out)))
    return fail(c, TK_ERR_INVALID_ARG, "g, r and out must not alias");
  mark(c, TK_STAGE_NONE);
  if (c->n == 1) {
    // flat NaiveAG: compress straight into this rank's slot of the gathered buffer -> one packed
    // in-place all-gather -> rank-ordered decompress
    uint32_t* gat = gathered ? gathered : c->recv;
    uint32_t* mine = gat + (size_t)c->rank * c->cw;
    const ChunkOut co = chunk_out(c, mine);
    if (c->P > 1 && c->pg) {
      // fused all-gather (TK_AG_PUSH): the compression selects into this rank's plain slot, then
      // each CTA pushes its run of pairs as tagged packets into this rank's chunk on every GPU;
      // the decompression consumes the packets as they land (waiting per packet on its tag) and
      // re-emits the gathered pairs in the plain layout.  Double-buffered by step parity: a
      // peer writes step s+2 into a buffer only after its step s+1 decompression consumed this
      // rank's step s+1 packets, which this rank pushed after its step s decompression finished.
      const uint32_t parity = c->push_seq & 1u;
      const size_t stride = (size_t)c->P * c->k;
      PushOut po;
      memset(&po, 0, sizeof(po));
      po.np = c->P;
      po.me = c->rank;
      po.tag = c->push_seq + 1;
      for (uint32_t q = 0; q < c->P; ++q) po.slot[q] = c->peer_pg[q] + parity * stride + (size_t)c->rank * c->k;
      TK_TRY(compress_impl(c, g, ef ? r : nullptr, mine, co.val, nullptr, 0, &po, co.val16));
      c->push_seq++;
      mark(c, TK_STAGE_ALLGATHER);
      TaggedChunks src{c->pg + parity * stride, c->k, po.tag, c->dev_err, c->timeout_ns};
      TK_TRY(decompress_impl(c, src, c->P, c->k, c->d, out, gat, w, lr));
    } else {
      // P = 1 without the fused update: the aggregate of one chunk is the selection itself (Alg. 2
      // l.15-20: out = +0; out[idx] += val), so the compression writes it whole (zeros after its last
      // grid barrier, then the k values, each warp over its own slab) and no decompression runs
      const bool fuse_out = c->P == 1 && !w && out;
      TK_TRY(compress_impl(c, g, ef ? r : nullptr, mine, co.val, nullptr, 0, nullptr, co.val16,
                           fuse_out ? out : nullptr, fuse_out));
      if (c->P > 1) TK_NCCL(c, ncclAllGather(mine, gat, c->cw, ncclUint32, c->world, c->stream));
      mark(c, TK_STAGE_ALLGATHER);
      if (!fuse_out) TK_TRY(decompress_plain(c, gat, c->P, c->d, out, w, lr));
    }
  } else {
    // HiTopKComm (Alg. 2).  The compressed segment goes straight into this GPU's slot (its node
    // index i = col_pos) of the column-gathered buffer.
    uint32_t* gat = gathered ? gathered : c->recv;
    uint32_t* mine = gat + (size_t)c->col_pos * c->cw;
    const ChunkOut co = chunk_out(c, mine);
    // Step 1: intra-node reduce-scatter of g (Eq. 4) ...
    if (c->cfg.rs_mode == TK_RS_ORDERED) {
      // ... ordered, read by this GPU's EF kernel straight from the row peers' buffers: make g
      // peer-visible, then a row barrier (stream-ordered all-reduce of 4 bytes) so every peer's
      // copy is complete before anyone reads it.  The previous step's row all-gather (step 4)
      // already ordered every peer's last read of these buffers before this copy.
      // a g inside a symmetric buffer (tk_alloc_symmetric, tk_input_buffer) is read in place by
      // the peers; any other g is first copied into this GPU's input buffer
      size_t goff = 0;
      const tk_ctx::Sym* gs = find_sym(c, g, sizeof(float) * c->d, &goff);
      if (!gs) {
        TK_CUDA(c, cudaMemcpyAsync(c->sym_g, g, sizeof(float) * c->d, cudaMemcpyDeviceToDevice, c->stream));
        gs = find_sym(c, c->sym_g, sizeof(float) * c->d, &goff);
        if (!gs) return fail(c, TK_ERR_STATE, "input buffer not registered");
      }
      TK_NCCL(c, ncclAllReduce(c->sync_buf, c->sync_buf, 1, ncclInt32, ncclSum, c->row, c->stream));
      mark(c, TK_STAGE_REDUCE_SCATTER);
      Peers pr;
      memset(&pr, 0, sizeof(pr));
      for (uint32_t q = 0; q < c->n; ++q)
        pr.p[q] = reinterpret_cast<const float*>(gs->peer[q] + goff) + (size_t)c->row_pos * c->L;
      // Step 2 (fused with step 1): MSTopK on the segment with k~ (Eq. 5), EF on the segment residual.
      TK_TRY(compress_impl(c, nullptr, ef ? r : nullptr, mine, co.val, &pr, (int)c->n, nullptr, co.val16));
    } else {
      TK_NCCL(c, ncclReduceScatter(g, c->seg, c->L, ncclFloat32, ncclSum, c->row, c->stream));
      mark(c, TK_STAGE_REDUCE_SCATTER);
      // Step 2: MSTopK on the segment with k~ (Eq. 5), error feedback on the segment residual.
      TK_TRY(compress_impl(c, c->seg, ef ? r : nullptr, mine, co.val, nullptr, 0, nullptr, co.val16));
    }
    // Step 3: inter-node all-gather among the m GPUs at the same position j (Eq. 6), in place ...
    if (c->m > 1) TK_NCCL(c, ncclAllGather(mine, gat, c->cw, ncclUint32, c->col, c->stream));
    mark(c, TK_STAGE_ALLGATHER);
    if (c->cfg.step4 == TK_STEP4_DENSE && !out) {  // the dense step 4 gathers the aggregate itself
      if (!c->h_out) TK_TRY(dev_alloc(c, &c->h_out, c->d));
      out = c->h_out;
    }
    float* my_seg = out ? out + (size_t)c->row_pos * c->L : nullptr;
    if (c->cfg.step4 == TK_STEP4_DENSE) {
      // ... accumulated in group order into this GPU's segment, then step 4: dense intra-node
      // all-gather of the segments (Alg. 2 l.21-23).  When out is a symmetric buffer the
      // decompression writes the segment straight into every row peer's out as well (NVLink
      // stores, fused with step 3's accumulation), and a row barrier completes the exchange;
      // otherwise an in-place ncclAllGather follows.
      size_t ooff = 0;
      const tk_ctx::Sym* os = c->cfg.loopback ? nullptr : find_sym(c, out, sizeof(float) * c->d, &ooff);
      if (os && c->n <= 8) {
        OutReplicas rp;
        memset(&rp, 0, sizeof(rp));
        for (uint32_t q = 0; q < c->n; ++q)
          if (q != c->row_pos)
            rp.p[rp.n++] = reinterpret_cast<float*>(os->peer[q] + ooff) + (size_t)c->row_pos * c->L;
        TK_TRY(decompress_plain(c, gat, c->m, c->L, my_seg, nullptr, 0.0f, &rp));
        // every peer's segment stores into this GPU's out are complete once every peer's
        // decompression has finished: a stream-ordered 4-byte row all-reduce
        TK_NCCL(c, ncclAllReduce(c->sync_buf, c->sync_buf, 1, ncclInt32, ncclSum, c->row, c->stream));
      } else {
        TK_TRY(decompress_plain(c, gat, c->m, c->L, my_seg));
        TK_NCCL(c, ncclAllGather(my_seg, out, c->L, ncclFloat32, c->row, c->stream));
      }
      mark(c, TK_STAGE_STEP4_ALLGATHER);
      if (w) {
        k_sgd_update<<<c->sms * 4, THREADS, 0, c->stream>>>(w, out, c->d, lr);
        TK_TRY(check_launch(c, "k_sgd_update"));
      }
    } else {
      // step 4 sparse (Eq. 10): all-gather the m*k~ gathered pairs of every segment, then every
      // GPU accumulates all segments itself (same per-element order -> identical bits).
      TK_NCCL(c, ncclAllGather(gat, c->recv_row, (size_t)c->m * c->cw, ncclUint32, c->row, c->stream));
      mark(c, TK_STAGE_STEP4_ALLGATHER);
      for (uint32_t j = 0; j < c->n; ++j)
        TK_TRY(decompress_plain(c, c->recv_row + (size_t)j * c->m * c->cw, c->m, c->L,
                                out ? out + (size_t)j * c->L : nullptr, w ? w + (size_t)j * c->L : nullptr, lr));
    }
  }
  c->step++;
  return TK_OK;
}

tk_status tk_step(tk_ctx* c, const float* g, float* r, float* out, uint32_t* gathered) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!out) return fail(c, TK_ERR_INVALID_ARG, "null pointer");
  return step_impl(c, g, r, out, gathered, nullptr, 0.0f);
}

tk_status tk_step_sgd(tk_ctx* c, const float* g, float* r, float* w, float lr, float* out, uint32_t* gathered) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!w) return fail(c, TK_ERR_INVALID_ARG, "null w");
  if (!(lr == lr) || lr == INFINITY || lr == -INFINITY) return fail(c, TK_ERR_INVALID_ARG, "lr must be finite");
  return step_impl(c, g, r, out, gathered, w, lr);
}

tk_status tk_step_host(tk_ctx* c, const float* g_host, uint32_t* gathered_host, float* out_host) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!g_host) return fail(c, TK_ERR_INVALID_ARG, "null g_host");
  if (!c->h_g) {
    TK_TRY(dev_alloc(c, &c->h_g, c->d));
    TK_TRY(dev_alloc(c, &c->h_r, c->L));
    TK_TRY(dev_alloc(c, &c->h_out, c->d));
    TK_CUDA(c, cudaMemsetAsync(c->h_r, 0, sizeof(float) * c->L, c->stream));
  }
  TK_CUDA(c, cudaMemcpyAsync(c->h_g, g_host, sizeof(float) * c->d, cudaMemcpyHostToDevice, c->stream));
  TK_TRY(tk_step(c, c->h_g, c->h_r, c->h_out, nullptr));
  if (gathered_host) {
    const size_t chunks = (c->n == 1) ? c->P : c->m;
    TK_CUDA(c, cudaMemcpyAsync(gathered_host, c->recv, sizeof(uint32_t) * chunks * c->cw, cudaMemcpyDeviceToHost,
                               c->stream));
  }
  if (out_host)
    TK_CUDA(c, cudaMemcpyAsync(out_host, c->h_out, sizeof(float) * c->d, cudaMemcpyDeviceToHost, c->stream));
  TK_CUDA(c, cudaStreamSynchronize(c->stream));
  return TK_OK;
}

tk_status tk_alloc_symmetric(tk_ctx* c, size_t bytes, void** p) {
  if (!c || !p || bytes == 0) return TK_ERR_INVALID_ARG;
  *p = nullptr;
  if (c->n == 1 || c->cfg.rs_mode != TK_RS_ORDERED || !c->row)
    return fail(c, TK_ERR_STATE, "symmetric buffers belong to HiTopKComm with the ordered reduce-scatter");
  char* base = nullptr;
  TK_TRY(dev_alloc(c, &base, bytes));
  void* peers[8] = {nullptr};
  tk_status s = exchange_ipc(c, c->row, c->n, c->row_pos, base, peers);
  if (s != TK_OK) {
    cudaFree(base);
    return s;
  }
  tk_ctx::Sym y;
  memset(&y, 0, sizeof(y));
  y.base = base;
  y.bytes = bytes;
  for (uint32_t q = 0; q < c->n; ++q) y.peer[q] = static_cast<char*>(peers[q]);
  c->syms.push_back(y);
  *p = base;
  return TK_OK;
}

tk_status tk_free_symmetric(tk_ctx* c, void* p) {
  if (!c || !p) return TK_ERR_INVALID_ARG;
  for (size_t i = 1; i < c->syms.size(); ++i)  // [0] is the context's own input buffer
    if (c->syms[i].base == p) {
      TK_CUDA(c, cudaStreamSynchronize(c->stream));
      for (uint32_t q = 0; q < 8; ++q)
        if (c->syms[i].peer[q] && c->syms[i].peer[q] != c->syms[i].base) cudaIpcCloseMemHandle(c->syms[i].peer[q]);
      cudaFree(c->syms[i].base);
      c->syms.erase(c->syms.begin() + (long)i);
      return TK_OK;
    }
  return fail(c, TK_ERR_INVALID_ARG, "not a symmetric buffer of this context");
}

tk_status tk_decompress_replicated(tk_ctx* c, const uint32_t* gathered, uint32_t nchunks, float* const* outs,
                                   uint32_t nout) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (!gathered || !outs || nout < 1 || nout > 9) return fail(c, TK_ERR_INVALID_ARG, "gathered/outs, nout in [1, 9]");
  if (nchunks < 1 || nchunks > 4096) return fail(c, TK_ERR_INVALID_ARG, "nchunks must lie in [1, 4096]");
  OutReplicas rp;
  memset(&rp, 0, sizeof(rp));
  for (uint32_t q = 0; q < nout; ++q)
    if (!outs[q] || !aligned16(outs[q])) return fail(c, TK_ERR_INVALID_ARG, "output %u null or misaligned", q);
  for (uint32_t q = 1; q < nout; ++q) rp.p[rp.n++] = outs[q];
  const uint64_t len = (c->n == 1) ? c->d : c->L;
  return decompress_plain(c, gathered, nchunks, len, outs[0], nullptr, 0.0f, &rp);
}

tk_status tk_input_buffer(tk_ctx* c, float** g) {
  if (!c || !g) return TK_ERR_INVALID_ARG;
  *g = c->sym_g;
  return TK_OK;
}

tk_status tk_get_stats(tk_ctx* c, tk_stats* st) {
  if (!c || !st) return TK_ERR_INVALID_ARG;
  Ctrl h;
  TK_CUDA(c, cudaMemcpyAsync(&h, c->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, c->stream));
  TK_CUDA(c, cudaStreamSynchronize(c->stream));
  memset(st, 0, sizeof(*st));
  st->mean = h.abar;
  st->max_bits = h.umax_bits;
  st->n_trials = h.it;
  // the exact selector keeps no trial log (n_trials = its narrowing passes)
  for (uint32_t i = 0; c->cfg.select != TK_SELECT_EXACT && i < h.it && i < (uint32_t)NMAX; ++i) {
    st->ratio[i] = h.ratio_log[i];
    st->thres[i] = h.thres_log[i];
    st->key[i] = h.key_log[i];
    st->nnz[i] = h.nnz_log[i];
  }
  st->k = c->k;
  st->k1 = h.k1;
  st->k2 = h.k2;
  st->thres1 = h.thres1;
  st->thres2 = h.thres2;
  st->thres1_set = h.prov1 >= 0;
  st->thres2_set = h.prov2 >= 0;
  st->key1 = st->thres1_set ? h.key1 : INF_BITS;
  st->key2 = st->thres2_set ? h.key2 : 0u;
  st->len2 = h.len2;
  st->rand_start = h.rand;
  st->step = h.step;
  c->nonfinite_sticky |= h.nonfinite;
  st->nonfinite = c->nonfinite_sticky;
  st->compacted = h.cap_ok;
  st->n_compacted = h.n_compacted;
  st->ef_compacted = h.ef_used;
  st->nnz_not_counted = c->cfg.select == TK_SELECT_EXACT ? 0ull : h.nnz_lb;
  for (uint32_t i = 0; i < st->n_trials && i < (uint32_t)NMAX; ++i)
    if (st->nnz_not_counted >> i & 1ull) st->nnz[i] = TK_NNZ_NOT_COUNTED;  // only "nnz > k" is known
  st->n_phases = std::min<uint32_t>(12, h.n_phase);
  for (int i = 0; i < 12; ++i) st->phase_ns[i] = h.phase_ns[i];
  uint32_t terr = 0;
  TK_CUDA(c, cudaMemcpy(&terr, c->dev_err, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  c->timeout_sticky |= terr;
  if (c->timeout_sticky)
    return fail(c, TK_ERR_TIMEOUT, "a peer's packets did not arrive within push_timeout_ms (aggregate invalid)");
  if (c->nonfinite_sticky) return fail(c, TK_ERR_NONFINITE, "non-finite value in acc (precondition, Q24)");
  return TK_OK;
}

tk_status tk_set_step(tk_ctx* c, uint64_t step) {
  if (!c) return TK_ERR_INVALID_ARG;
  c->step = step;
  return TK_OK;
}

tk_status tk_query(const tk_ctx* c, uint64_t* k, uint64_t* seg_len, uint32_t* nranks, uint32_t* m, uint32_t* n) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (k) *k = c->k;
  if (seg_len) *seg_len = c->L;
  if (nranks) *nranks = c->P;
  if (m) *m = c->m;
  if (n) *n = c->n;
  return TK_OK;
}

uint64_t tk_launch_count(const tk_ctx* c) { return c ? c->launches : 0; }

tk_status tk_profile_begin(tk_ctx* c, uint32_t max_steps) {
  if (!c || max_steps == 0) return TK_ERR_INVALID_ARG;
  const uint32_t need = max_steps * 32u;
  if (need > c->prof_cap) {
    if (c->prof_ev) {
      TK_CUDA(c, cudaStreamSynchronize(c->stream));
      for (uint32_t i = 0; i < c->prof_cap; ++i) cudaEventDestroy(c->prof_ev[i]);
      delete[] c->prof_ev;
      delete[] c->prof_kind;
    }
    c->prof_ev = new (std::nothrow) cudaEvent_t[need];
    c->prof_kind = new (std::nothrow) uint8_t[need];
    if (!c->prof_ev || !c->prof_kind) return TK_ERR_NOMEM;
    for (uint32_t i = 0; i < need; ++i) TK_CUDA(c, cudaEventCreate(&c->prof_ev[i]));
    c->prof_cap = need;
  }
  c->prof_n = 0;
  memset(c->prof_launch, 0, sizeof(c->prof_launch));
  c->prof_on = true;
  return TK_OK;
}

tk_status tk_profile_end(tk_ctx* c, double ms[TK_NSTAGES], uint32_t launches[TK_NSTAGES]) {
  if (!c || !ms) return TK_ERR_INVALID_ARG;
  c->prof_on = false;
  for (int i = 0; i < TK_NSTAGES; ++i) ms[i] = 0.0;
  TK_CUDA(c, cudaStreamSynchronize(c->stream));
  for (uint32_t i = 1; i < c->prof_n; ++i) {
    const int kind = c->prof_kind[i];
    if (kind == TK_STAGE_NONE) continue;  // a step's opening mark: the gap to it is not a stage
    float t = 0.f;
    TK_CUDA(c, cudaEventElapsedTime(&t, c->prof_ev[i - 1], c->prof_ev[i]));
    ms[kind] += (double)t;
  }
  if (launches) memcpy(launches, c->prof_launch, sizeof(c->prof_launch));
  return TK_OK;
}

const char* tk_stage_name(uint32_t stage) {
  static const char* names[TK_NSTAGES] = {"none",      "k_compress", "reserved2",       "reserved3",
                                          "reserved4", "reserved5",  "reserved6",       "reserved7",
                                          "reserved8", "allgather",  "reserved10",      "k_decompress",
                                          "reduce_scatter", "step4_allgather", "reserved14", "reserved15"};
  return stage < TK_NSTAGES ? names[stage] : "invalid";
}

tk_status tk_destroy(tk_ctx* c) {
  if (!c) return TK_ERR_INVALID_ARG;
  if (c->stream) cudaStreamSynchronize(c->stream);
  free_all(c);
  delete c;
  return TK_OK;
}

const char* tk_status_string(tk_status s) {
  switch (s) {
    case TK_OK: return "ok";
    case TK_ERR_INVALID_ARG: return "invalid argument";
    case TK_ERR_RANGE: return "k out of range";
    case TK_ERR_CONFIG: return "invalid configuration";
    case TK_ERR_NONFINITE: return "non-finite input";
    case TK_ERR_CUDA: return "CUDA error";
    case TK_ERR_NCCL: return "NCCL error";
    case TK_ERR_STATE: return "invalid state";
    case TK_ERR_NOMEM: return "out of device memory";
    case TK_ERR_TIMEOUT: return "fused all-gather timed out waiting for a peer";
  }
  return "unknown status";
}

const char* tk_last_error(const tk_ctx* c) { return c ? c->err : "no context"; }

#ifdef TK_PHASE_TRACE
// experiment builds only (tools/trace_probe.py): the per-CTA phase timeline of the last k_compress
tk_status tk_debug_trace(uint64_t* out /* host [2][32][2048] */) {
  return cudaMemcpyFromSymbol(out, tk::g_trace, sizeof(tk::g_trace)) == cudaSuccess ? TK_OK : TK_ERR_CUDA;
}
#endif

}  // extern "C"
