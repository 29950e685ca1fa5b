/* tk.h — C ABI of the B200-native top-k sparsified gradient aggregation library (libtk.so).
 *
 * Implements the data-parallel hot path of "Towards Scalable Distributed Training of Deep
 * Learning on Public Cloud Clusters" (Shi et al., arXiv 2010.10458, MLSys'21), CommLib §3
 * (PAPER.md P:127-266):
 *   error feedback (acc = g + r)                     — BASELINE.json north_star (not in the paper)
 *   MSTopK approximate top-k, Algorithm 1            — P:148-188
 *   compaction into ascending (index, value) pairs   — Alg. 1 l.25-29, P:180-185 (reading Q11)
 *   sparse All-Gather of (kappa, iota)               — §3.2, Eq. 3
 *   rank-ordered index accumulation (decompress)     — Alg. 2 l.15-20
 *   residual write-back of the unsent mass           — BASELINE.json north_star
 *   HiTopKComm (m x n virtual nodes), Algorithm 2    — P:203-248
 * and the adjacent rows of SURVEY.md §8(f):
 *   exact top-k selector (TK_SELECT_EXACT)           — Eq. 2, P:131-139 (F1)
 *   MSTopK with the prose threshold search           — P:148, reading Q33 (F3, TK_SELECT_PROSE)
 *   fused all-gather pushed over NVLink (TK_AG_PUSH) — P:197 (F2)
 *   FP16 values on the wire (TK_WIRE_F16)            — Fig. 7 ran FP16, P:337 (F3)
 *   SGD update fused into decompression (tk_step_sgd)— Eq. 1, P:65-67 (F4)
 * "Q<n>" refers to the numbered readings of silent/ambiguous passages in DESIGN.md.
 *
 * Conventions (all entry points):
 *   - Pointers to vectors are DEVICE pointers (cudaMalloc / torch CUDA tensors), 16-byte aligned,
 *     unless the name ends in _host.  The caller owns every vector it passes; libtk owns only its
 *     scratch (allocated in tk_init, freed in tk_destroy).
 *   - All device work is enqueued on the stream given to tk_init, asynchronously w.r.t. the host,
 *     except tk_init, tk_get_stats, tk_step_host and tk_destroy, which synchronise that stream.
 *   - Every call returns a tk_status; no C++ exception crosses the ABI.  Arguments are validated
 *     before anything is launched.  Details of the last failure: tk_last_error(ctx).
 *   - Results are a pure function of (inputs, config, step counter, rank): independent of grid
 *     size, SM count and timing.  A context is single-stream and not thread-safe.
 *   - Gradients are fp32 (Eq. 3 bills 4-byte FP32 elements).  d < 2^32 (u32 indices).
 */
#ifndef TK_H_
#define TK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tk_ctx tk_ctx;
typedef void* tk_stream_t; /* a cudaStream_t (0 = legacy default stream) */

typedef enum tk_status {
  TK_OK = 0,
  TK_ERR_INVALID_ARG = 1, /* NULL / misaligned pointer, d == 0 or d >= 2^32, rho not in (0,1],
                             N not in [1,52], rank >= P, aliasing buffers                    */
  TK_ERR_RANGE = 2,       /* explicit k not in [1, d] (segment length for HiTopKComm)          */
  TK_ERR_CONFIG = 3,      /* P % n != 0, d % n != 0, (d/n) % 4 != 0 for n > 1 (segments must be
                             16-byte aligned), NCCL unique id missing for P > 1               */
  TK_ERR_NONFINITE = 4,   /* NaN/Inf met in acc (precondition, Q24); sticky, reported by the
                             next tk_get_stats                                                 */
  TK_ERR_CUDA = 5,        /* CUDA runtime error; text in tk_last_error                        */
  TK_ERR_NCCL = 6,        /* NCCL error; text in tk_last_error                                 */
  TK_ERR_STATE = 7,       /* wrong call order (e.g. tk_sparse_allgather with P == 1 comm absent)*/
  TK_ERR_NOMEM = 8,       /* device allocation of scratch failed                              */
  TK_ERR_TIMEOUT = 9      /* the fused all-gather waited longer than push_timeout_ms for a peer's
                             packets (a peer died or stalled): that step's aggregate is invalid;
                             sticky, reported by the next tk_get_stats                          */
} tk_status;

enum { TK_RAND_SEEDED = 0, TK_RAND_FIRST = 1 };   /* Alg. 1 l.27 window start (Q10)           */
enum { TK_STEP4_DENSE = 0, TK_STEP4_SPARSE = 1 }; /* HiTopKComm step 4: Alg. 2 l.21-23 vs Eq.10*/
enum { TK_AG_PUSH = 0, TK_AG_NCCL = 1 };          /* flat sparse all-gather (A9):
                                                     PUSH = the compression writes its pairs into
                                                     every peer's buffer over NVLink (P <= 8);
                                                     NCCL = ncclAllGather after the compression */
enum { TK_SELECT_MSTOPK = 0, TK_SELECT_EXACT = 1, TK_SELECT_PROSE = 2 };
                                                  /* selector:
                                                     MSTOPK = Alg. 1 under Q1-Q27;
                                                     EXACT = exact top-k of Eq. 2:
                                                     the k largest |acc|, ties -> lower index (Q6);
                                                     n_iters is then unused;
                                                     PROSE = MSTopK with the threshold search of
                                                     the prose of P:148 (start at a-bar, double /
                                                     halve until bracketed, then bisect the
                                                     bracket; reading Q33); selection as Alg. 1 */
enum { TK_WIRE_F32 = 0, TK_WIRE_F16 = 1 };         /* value format on the wire (Fig. 7
                                                     ran FP16; reading Q31): F16 = each
                                                     selected value v is sent as
                                                     fp16_RN(clamp(v, +-65504)) and the residual
                                                     keeps fl32(v - sent) instead of +0; a packed
                                                     chunk is then [idx k | binary16 val k] padded
                                                     to k + ceil(k/2) u32 words (6k bytes + pad)  */
enum { TK_RS_ORDERED = 0, TK_RS_NCCL = 1 };       /* HiTopKComm step 1 reduce-scatter (Q20):
                                                     ORDERED = ascending-row-rank fp32 sum read over
                                                     NVLink peer pointers inside the EF kernel
                                                     (bit-exact; n in {2,4,8});
                                                     NCCL = ncclReduceScatter (order unspecified) */

typedef struct tk_config {
  uint64_t d;              /* gradient length (the paper's d)                           */
  double rho;              /* density, 0 < rho <= 1                                    */
  uint64_t k;              /* 0: k = max(1, floor(rho*d)) (Q13); else explicit, 1 <= k <= d     */
  uint32_t n_iters;        /* MSTopK N, the number of threshold samplings (Alg. 1 input), 1..52 */
  uint32_t nranks;         /* P workers (one process per GPU)                                  */
  uint32_t rank;           /* this process's rank in [0, P)                                    */
  uint32_t group_size;     /* n: 1 = flat NaiveAG; >1 = HiTopKComm with m = P/n */
  uint64_t seed;           /* seed of the window RNG (Q10)                                     */
  uint32_t rand_mode;      /* TK_RAND_SEEDED (default) or TK_RAND_FIRST (rand = 0)             */
  uint32_t error_feedback; /* 1: acc = g + r, r' = acc with sent entries := +0.0 (Q14);
                              0: MSTopK runs on g itself and r is ignored (may be NULL)         */
  uint32_t step4;          /* HiTopKComm step 4 mode (TK_STEP4_DENSE or TK_STEP4_SPARSE)       */
  uint32_t levels_per_pass;/* bisection levels resolved per count pass (1..10; 0 = default 10): the
                              first pass over the whole vector resolves min(2, this); later passes
                              on the compacted entries resolve up to this many at once, passes
                              over the whole vector up to 2.  Result bits do not depend on it.  */
  int32_t device;          /* CUDA device ordinal to use (-1 = current)                        */
  uint32_t rs_mode;        /* HiTopKComm step-1 mode (TK_RS_ORDERED or TK_RS_NCCL)             */
  uint32_t ag_mode;        /* flat all-gather mode (TK_AG_PUSH or TK_AG_NCCL)                  */
  uint32_t select;         /* TK_SELECT_MSTOPK (default) or TK_SELECT_EXACT                    */
  uint32_t wire;           /* TK_WIRE_F32 (default) or TK_WIRE_F16 (values sent as binary16)  */
  /* --- execution options (0 = default everywhere; none changes a result bit) --------------- */
  uint32_t exact_trial_counts; /* 1: every trial's nnz in tk_stats is the exact count (Alg. 1
                              l.10).  Default 0: a trial whose threshold lies below the key
                              the previous call predicted is only known to have nnz > k (the
                              decision it needs), its nnz is reported as TK_NNZ_NOT_COUNTED;
                              1 adds a whole-vector count pass (4d bytes) when that happens */
  uint32_t disable_ef_compaction; /* 1: never compact in the error-feedback pass (the whole-vector
                              first pass runs every call).  Default 0                            */
  uint32_t first_pass_keys;  /* keys counted by a whole-vector first pass along the predicted
                              path, 1..3 (0 = 3)                                                */
  uint32_t check_selection;  /* 1: verify every selection on the device (strictly ascending,
                              in range; a violation traps); debugging only                       */
  uint32_t push_timeout_ms;  /* TK_AG_PUSH: how long a decompression waits for one peer packet
                              before it gives up and reports TK_ERR_TIMEOUT (0 = 300000, 5 min;
                              ranks may legitimately drift by seconds: checkpoints, eval)         */
  uint32_t loopback;         /* 1: emulate rank `rank` of `nranks` on this GPU without any
                              communicator (uid may be NULL): only tk_compress,
                              tk_compress_segment, tk_decompress and the tk_loopback_* calls are
                              allowed; tk_step / tk_sparse_allgather return TK_ERR_STATE.  For
                              single-GPU parity tests of the multi-GPU kernels                   */
} tk_config;

#define TK_NNZ_NOT_COUNTED 0xFFFFFFFFu

/* Snapshot of the last compression's MSTopK control block (for parity checks). */
typedef struct tk_stats {
  double mean;             /* a-bar, canonical fp64 pairwise mean of |acc| (Alg. 1 l.2, Q3)    */
  uint32_t max_bits;       /* bits of u = max |acc| (Alg. 1 l.3)                               */
  uint32_t n_trials;       /* = N (MSTopK); the narrowing passes (exact selector, no trial log) */
  double ratio[52];        /* per trial: ratio (Alg. 1 l.8)                                    */
  double thres[52];        /*            thres (l.9, fp64, Q4)                                 */
  uint32_t key[52];        /*            bits of the smallest fp32 >= thres                    */
  uint32_t nnz[52];        /*            count_nonzero(a >= thres) (l.10)                      */
  uint64_t k, k1, k2;      /* Alg. 1 l.5 state after the loop                                  */
  double thres1, thres2;   /* l.6 state after the loop (0 when never set)                      */
  uint32_t key1, key2;     /* integer keys of thres1 / thres2 (0x7F800000 / 0 when unset)      */
  uint32_t thres1_set, thres2_set;
  uint64_t len2;           /* len(iota2) (l.26)                                                */
  uint64_t rand_start;     /* rand (l.27)                                                      */
  uint64_t step;           /* step counter used for this compression's RNG draw               */
  uint32_t nonfinite;      /* 1 if a NaN/Inf was seen (sticky)                                 */
  uint32_t compacted;      /* 1 if later passes and the selection ran on compacted entries
                              (an exact shortcut)                               */
  uint32_t n_compacted;    /* entries kept (when compacted)                                     */
  uint32_t n_phases;       /* phase boundaries recorded in phase_ns                             */
  uint64_t phase_ns[12];   /* device %globaltimer (ns) at k_compress's phase boundaries (CTA 0,
                              after each grid barrier): start, stats, each count pass, prefix,
                              end of selection                                                 */
  uint32_t ef_compacted;   /* 1 if the entries were compacted inside the EF pass at the key the
                              previous call predicted (no whole-vector count pass ran)         */
  uint64_t nnz_not_counted;/* bit i set: trial i's threshold lay below that compaction key; its
                              count is only known to exceed k (the decision it needs; every
                              result is exact) and nnz[i] = TK_NNZ_NOT_COUNTED.
                              Always 0 with exact_trial_counts = 1                             */
} tk_stats;

/* k = max(1, floor(rho * d)) in fp64 (Q13).  Host-only, pure.  0 on invalid input. */
uint64_t tk_k(uint64_t d, double rho);

/* Rank 0 creates the 128-byte NCCL unique id that every rank passes to tk_init (P > 1). */
tk_status tk_get_unique_id(uint8_t uid[128]);

/* Collective over all P ranks when P > 1 (NCCL communicator bootstrap from uid; HiTopKComm also
 * splits row (size n) and column (size m) communicators).  uid may be NULL iff P == 1.
 * On success *out owns all scratch; release with tk_destroy. */
tk_status tk_init(const tk_config* cfg, const uint8_t* uid, tk_stream_t stream, tk_ctx** out);

/* MSTopK compression of one rank (Alg. 1 + error feedback), flat mode only.
 *   g   [d]  in     gradient (never written)
 *   r   [d]  in/out residual r -> r' (error_feedback = 1); ignored when error_feedback = 0
 *   idx [k]  out    selected indices iota, strictly ascending (Q11)
 *   val [k]  out    kappa = acc[iota], bit-copied (Q12); TK_WIRE_F16: the fp16-rounded values sent
 * g must not alias r, idx or val. */
tk_status tk_compress(tk_ctx* ctx, const float* g, float* r, uint32_t* idx, float* val);

/* Segment compression, HiTopKComm steps 1-2 for one GPU (Eq. 4-5; Alg. 2 l.2-8):
 * MSTopK (or the configured selector) of acc = (sum_{q=0..nsrc-1} src[q]) (+ r with error
 * feedback), the sum taken in ascending q, left to right, fp32 round-to-nearest (reading Q20).
 *   src  host array of nsrc DEVICE pointers, each to L = seg_len floats (tk_query), 16-byte
 *        aligned, readable from this GPU (local buffers or CUDA-IPC-mapped peer memory)
 *   nsrc 1, 2, 4 or 8 (nsrc = 1: acc = src[0] (+ r), i.e. tk_compress on a length-L vector)
 *   r    [L] in/out residual (error feedback; ignored otherwise); idx/val [k~] out as tk_compress
 * Valid in every mode: in HiTopKComm mode it is the step-1+2 kernel tk_step runs (there with the
 * row peers' buffers), in flat mode L = d.  Does not advance the step counter. */
tk_status tk_compress_segment(tk_ctx* ctx, const float* const* src, uint32_t nsrc, float* r, uint32_t* idx,
                              float* val);

/* Sparse All-Gather: gathered [P][cw] u32, rank-major, each rank's chunk laid out as
 * [idx k | bits(val) k] (Q15, cw = 2k) or, with TK_WIRE_F16, [idx k | binary16 val k] padded to
 * cw = k + ceil(k/2) words.  idx/val are this rank's tk_compress outputs (with TK_WIRE_F16 the
 * values are already the fp16-rounded ones).  Collective. */
tk_status tk_sparse_allgather(tk_ctx* ctx, const uint32_t* idx, const float* val, uint32_t* gathered);

/* Rank-ordered index accumulation (Alg. 2 l.15-20): out = +0^d; for p = 0..nchunks-1 in order:
 * out[idx_p] += val_p in fp32 round-to-nearest (Q16).  gathered is [nchunks][cw] as above, each
 * chunk's indices strictly ascending and < d (violations: memory-safe, result unspecified).
 * nchunks in [1, 4096]; out has d elements (flat) or d/n (HiTopKComm segment).  A larger
 * nchunks than any previous call grows an internal table (synchronises the stream). */
tk_status tk_decompress(tk_ctx* ctx, const uint32_t* gathered, uint32_t nchunks, float* out);

/* One whole iteration (flat: compress -> all-gather -> decompress; HiTopKComm: Alg. 2 steps 1-4).
 *   g   [d]            in      local gradient
 *   r   [d] or [d/n]   in/out  residual (flat: d; HiTopKComm: the segment length d/n, Q22)
 *   out [d]            out     aggregated sparse gradient, bitwise identical on every rank
 *   gathered           out     optional (NULL = internal): flat [P][cw]; HiTopKComm [m][cw~]
 * Increments the step counter after enqueueing. */
tk_status tk_step(tk_ctx* ctx, const float* g, float* r, float* out, uint32_t* gathered);

/* tk_step followed by the SGD update of Eq. 1, w_{t+1} = w_t - lr * (aggregated sparse
 * gradient), fused into the decompression's tile write-back: for every i,
 * w[i] := fl32(w[i] - fl32(lr * out[i])) (two round-to-nearest fp32 operations, no FMA; Q29).
 *   w   [d]   in/out  parameters (device, 16-byte aligned, replicated: identical on every rank)
 *   lr          in     learning rate (finite)
 *   out [d]   out     optional (NULL: the aggregate is not stored - flat and sparse-step-4
 *                      HiTopKComm never write it; dense step 4 uses an internal buffer and applies
 *                      the update after the row all-gather)
 *   g, r, gathered as for tk_step.  w must not alias g, r or out.  TK_ERR_INVALID_ARG on a NULL or
 *   misaligned w or a non-finite lr. */
tk_status tk_step_sgd(tk_ctx* ctx, const float* g, float* r, float* w, float lr, float* out, uint32_t* gathered);

/* tk_step with HOST buffers (end-to-end path): copies g_host (pinned or pageable) to the device,
 * runs tk_step with a context-owned device residual (state carried across calls; zero at init),
 * and copies the P*2k gathered pairs (flat) back to gathered_host and, if out_host != NULL, the
 * dense aggregate back to out_host.  Synchronises the context stream. */
tk_status tk_step_host(tk_ctx* ctx, const float* g_host, uint32_t* gathered_host, float* out_host);

/* HiTopKComm with TK_RS_ORDERED: the context's own symmetric gradient buffer ([d] fp32, device).
 * A caller that writes its gradient here (or into a tk_alloc_symmetric buffer) and passes that
 * pointer as g to tk_step avoids the copy-in (tk_step copies any other g into this buffer first).
 * Same usage contract as the symmetric buffers below.  NULL for flat mode. */
tk_status tk_input_buffer(tk_ctx* ctx, float** g);

/* --- loopback (cfg.loopback = 1): single-GPU emulation of the fused all-gather ----
 * TEST INFRASTRUCTURE for the multi-GPU kernels on one GPU.  A tagged packet is 16 bytes: {u64
 * idx | tag << 32, u64 bits(val) | tag << 32}; a rank's chunk is k packets.
 * tk_loopback_push: tk_compress of this rank, which also writes its k pairs as packets tagged
 *   `tag` (!= 0) to slots[q] for q < nslots (host array of device pointers to k-packet slots,
 *   e.g. this rank's chunk in every emulated rank's packet buffer) - the same kernel and stores
 *   tk_step uses with TK_AG_PUSH, there with CUDA-IPC peer pointers.  chunk [cw] receives the
 *   plain packed pairs.
 * tk_loopback_decompress: the rank-ordered decompression of nchunks k-packet chunks (packets
 *   [nchunks][k]) that waits, per packet, for `tag` (up to push_timeout_ms, then TK_ERR_TIMEOUT
 *   at the next tk_get_stats); out [d] (flat) or [d/n] receives the aggregate and plain_out
 *   (optional, [nchunks][cw]) the consumed pairs in the plain layout. */
tk_status tk_loopback_push(tk_ctx* ctx, const float* g, float* r, uint32_t* chunk, void* const* slots,
                           uint32_t nslots, uint32_t tag);
tk_status tk_loopback_decompress(tk_ctx* ctx, const void* packets, uint32_t nchunks, uint32_t tag, float* out,
                                 uint32_t* plain_out);

/* Symmetric buffers (HiTopKComm with TK_RS_ORDERED; collective over the n GPUs of a virtual node):
 * every row peer allocates one of the same size in the same order; each GPU's copy is mapped into
 * its peers (CUDA IPC over NVLink).  A gradient g passed to tk_step from inside a symmetric buffer
 * is read in place by the ordered reduce-scatter (no copy into the input buffer); an out inside one
 * (all d floats) makes the dense step 4 part of the decompression: each GPU writes its aggregated
 * segment straight into every row peer's out (NVLink stores), and a 4-byte row all-reduce
 * completes the exchange instead of an ncclAllGather.  Usage contract: every peer passes g (and
 * out) at the same offset of corresponding buffers; a buffer passed as g to step s must not be
 * rewritten by anyone before step s's call has completed on the context stream (the step's row
 * all-gather / barrier orders every peer's reads before that).  Freeing synchronises the stream;
 * free only when no peer can still read the buffer. */
tk_status tk_alloc_symmetric(tk_ctx* ctx, size_t bytes, void** p);
tk_status tk_free_symmetric(tk_ctx* ctx, void* p);

/* Rank-ordered decompression (as tk_decompress) written to nout outputs at once: outs[0] and the
 * replicas outs[1..nout) (e.g. the node peers' copies of a segment; nout in [1, 9]).  tk_step
 * uses it for HiTopKComm's fused dense step 4. */
tk_status tk_decompress_replicated(tk_ctx* ctx, const uint32_t* gathered, uint32_t nchunks, float* const* outs,
                                   uint32_t nout);

/* Copy the control block of the last compression to *st (synchronises the stream). */
tk_status tk_get_stats(tk_ctx* ctx, tk_stats* st);

/* Set the step counter used by the next compression's window draw (resume; Q10). */
tk_status tk_set_step(tk_ctx* ctx, uint64_t step);

/* Sizes derived at init: k (flat) or k~ (HiTopKComm), segment length, P, m, n. */
tk_status tk_query(const tk_ctx* ctx, uint64_t* k, uint64_t* seg_len, uint32_t* nranks, uint32_t* m,
                   uint32_t* n);

/* Number of kernel launches libtk enqueued on the context stream since init (evidence counter). */
uint64_t tk_launch_count(const tk_ctx* ctx);

/* Stage profiling with CUDA events on the context stream.  Between tk_profile_begin and
 * tk_profile_end every tk_step records an event at each stage boundary (capacity max_steps
 * steps).  tk_profile_end synchronises and returns, per stage, the summed device time in ms and
 * the number of launches (ms / launches = mean duration of one launch of that stage).  Stages:
 * k_compress (A1-A8 in one cooperative kernel), allgather (NCCL or the P = 1 copy),
 * k_decompress, reduce_scatter (HiTopKComm step-1 barrier or NCCL RS), step4_allgather. */
enum {
  TK_STAGE_NONE = 0, TK_STAGE_COMPRESS = 1, TK_STAGE_ALLGATHER = 9, TK_STAGE_DECOMPRESS = 11,
  TK_STAGE_REDUCE_SCATTER = 12, TK_STAGE_STEP4_ALLGATHER = 13, TK_NSTAGES = 16
};
tk_status tk_profile_begin(tk_ctx* ctx, uint32_t max_steps);
tk_status tk_profile_end(tk_ctx* ctx, double ms[TK_NSTAGES], uint32_t launches[TK_NSTAGES]);
const char* tk_stage_name(uint32_t stage);

tk_status tk_destroy(tk_ctx* ctx);
const char* tk_status_string(tk_status s);
const char* tk_last_error(const tk_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* TK_H_ */
