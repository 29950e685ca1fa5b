"""paper_2010_10458_b200 — B200-native top-k sparsified gradient aggregation (arXiv 2010.10458).

Thin Python binding over the C ABI of ``libtk.so`` (include/tk.h): argument marshalling only.
Every step of the hot path — error feedback, MSTopK (Alg. 1), compaction, the sparse
All-Gather (NCCL, issued inside libtk), rank-ordered decompression and HiTopKComm (Alg. 2) —
runs in libtk's sm_100a kernels.  There is no CPU fallback: importing this package without a
built ``libtk.so`` raises, and every call fails loudly on a non-CUDA tensor.

PyTorch supplies device memory, the CUDA stream and the ``torch.distributed`` bootstrap of the
NCCL unique id (plumbing only).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch  # loads the venv's libnccl.so.2 first; libtk links the same soname

__all__ = ["Context", "Bucket", "bucket_layout", "TkError", "k_from_density", "unique_id", "broadcast_unique_id", "lib_path", "STATUS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libtk.so")

STATUS = {0: "TK_OK", 1: "TK_ERR_INVALID_ARG", 2: "TK_ERR_RANGE", 3: "TK_ERR_CONFIG", 4: "TK_ERR_NONFINITE",
          5: "TK_ERR_CUDA", 6: "TK_ERR_NCCL", 7: "TK_ERR_STATE", 8: "TK_ERR_NOMEM", 9: "TK_ERR_TIMEOUT"}
NNZ_NOT_COUNTED = 0xFFFFFFFF  # tk_stats.nnz of a trial whose count was not taken (only "nnz > k" is known)
NMAX = 52


class TkError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class _Config(ctypes.Structure):
    _fields_ = [("d", ctypes.c_uint64), ("rho", ctypes.c_double), ("k", ctypes.c_uint64),
                ("n_iters", ctypes.c_uint32), ("nranks", ctypes.c_uint32), ("rank", ctypes.c_uint32),
                ("group_size", ctypes.c_uint32), ("seed", ctypes.c_uint64), ("rand_mode", ctypes.c_uint32),
                ("error_feedback", ctypes.c_uint32), ("step4", ctypes.c_uint32),
                ("levels_per_pass", ctypes.c_uint32), ("device", ctypes.c_int32), ("rs_mode", ctypes.c_uint32),
                ("ag_mode", ctypes.c_uint32), ("select", ctypes.c_uint32), ("wire", ctypes.c_uint32),
                ("exact_trial_counts", ctypes.c_uint32), ("disable_ef_compaction", ctypes.c_uint32),
                ("first_pass_keys", ctypes.c_uint32), ("check_selection", ctypes.c_uint32),
                ("push_timeout_ms", ctypes.c_uint32), ("loopback", ctypes.c_uint32)]


class _Stats(ctypes.Structure):
    _fields_ = [("mean", ctypes.c_double), ("max_bits", ctypes.c_uint32), ("n_trials", ctypes.c_uint32),
                ("ratio", ctypes.c_double * NMAX), ("thres", ctypes.c_double * NMAX),
                ("key", ctypes.c_uint32 * NMAX), ("nnz", ctypes.c_uint32 * NMAX),
                ("k", ctypes.c_uint64), ("k1", ctypes.c_uint64), ("k2", ctypes.c_uint64),
                ("thres1", ctypes.c_double), ("thres2", ctypes.c_double),
                ("key1", ctypes.c_uint32), ("key2", ctypes.c_uint32),
                ("thres1_set", ctypes.c_uint32), ("thres2_set", ctypes.c_uint32),
                ("len2", ctypes.c_uint64), ("rand_start", ctypes.c_uint64), ("step", ctypes.c_uint64),
                ("nonfinite", ctypes.c_uint32), ("compacted", ctypes.c_uint32), ("n_compacted", ctypes.c_uint32),
                ("n_phases", ctypes.c_uint32),
                ("phase_ns", ctypes.c_uint64 * 12), ("ef_compacted", ctypes.c_uint32),
                ("nnz_not_counted", ctypes.c_uint64)]


# Every symbol include/tk.h declares (checked by tests/test_abi.py).
EXPORTS = ["tk_k", "tk_get_unique_id", "tk_init", "tk_compress", "tk_sparse_allgather", "tk_decompress",
           "tk_step", "tk_step_host", "tk_get_stats", "tk_set_step", "tk_query", "tk_launch_count",
           "tk_destroy", "tk_status_string", "tk_last_error", "tk_profile_begin", "tk_profile_end",
           "tk_stage_name", "tk_input_buffer", "tk_step_sgd", "tk_compress_segment", "tk_loopback_push",
           "tk_loopback_decompress", "tk_alloc_symmetric", "tk_free_symmetric", "tk_decompress_replicated"]
NSTAGES = 16


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"libtk.so not built at {_LIB_PATH}: run `python paper_2010_10458_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    P, U32, U64, I32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    sig = {
        "tk_k": (U64, [U64, ctypes.c_double]),
        "tk_get_unique_id": (I32, [ctypes.c_char_p]),
        "tk_init": (I32, [ctypes.POINTER(_Config), ctypes.c_char_p, P, ctypes.POINTER(P)]),
        "tk_compress": (I32, [P, P, P, P, P]),
        "tk_sparse_allgather": (I32, [P, P, P, P]),
        "tk_decompress": (I32, [P, P, U32, P]),
        "tk_step": (I32, [P, P, P, P, P]),
        "tk_step_sgd": (I32, [P, P, P, P, ctypes.c_float, P, P]),
        "tk_step_host": (I32, [P, P, P, P]),
        "tk_get_stats": (I32, [P, ctypes.POINTER(_Stats)]),
        "tk_set_step": (I32, [P, U64]),
        "tk_query": (I32, [P, ctypes.POINTER(U64), ctypes.POINTER(U64), ctypes.POINTER(U32),
                           ctypes.POINTER(U32), ctypes.POINTER(U32)]),
        "tk_launch_count": (U64, [P]),
        "tk_destroy": (I32, [P]),
        "tk_status_string": (ctypes.c_char_p, [I32]),
        "tk_last_error": (ctypes.c_char_p, [P]),
        "tk_profile_begin": (I32, [P, U32]),
        "tk_profile_end": (I32, [P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(U32)]),
        "tk_stage_name": (ctypes.c_char_p, [U32]),
        "tk_input_buffer": (I32, [P, ctypes.POINTER(P)]),
        "tk_compress_segment": (I32, [P, ctypes.POINTER(P), U32, P, P, P]),
        "tk_loopback_push": (I32, [P, P, P, P, ctypes.POINTER(P), U32, U32]),
        "tk_loopback_decompress": (I32, [P, P, U32, U32, P, P]),
        "tk_alloc_symmetric": (I32, [P, ctypes.c_size_t, ctypes.POINTER(P)]),
        "tk_free_symmetric": (I32, [P, P]),
        "tk_decompress_replicated": (I32, [P, P, U32, ctypes.POINTER(P), U32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()


def lib_path() -> str:
    return _LIB_PATH


def k_from_density(d: int, rho: float) -> int:
    """k = max(1, floor(rho*d)) (reading Q13), computed by libtk."""
    k = int(_lib.tk_k(int(d), float(rho)))
    if k == 0:
        raise ValueError("invalid d / rho")
    return k


def unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = _lib.tk_get_unique_id(buf)
    if st != 0:
        raise TkError(st, "ncclGetUniqueId failed")
    return buf.raw


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL unique id; torch.distributed broadcasts the 128 bytes."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    t = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        t.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
    if dist.get_backend(group) == "nccl":
        tc = t.cuda()
        dist.broadcast(tc, src=0, group=group)
        t = tc.cpu()
    else:
        dist.broadcast(t, src=0, group=group)
    return bytes(t.tolist())


def _ptr(t, name, dtype, numel=None, device=None):
    """Device pointer of a tensor, after checking what the C ABI cannot (it takes no lengths):
    type, device (the context's GPU), contiguity and - when given - at least `numel` elements."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (libtk has no CPU path)")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, the context on {device}")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} has {t.numel()} elements, needs {numel}")
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class Stats:
    mean: float
    max_bits: int
    trials: list  # (ratio, thres, key, nnz)
    k: int
    k1: int
    k2: int
    thres1: float
    thres2: float
    thres1_set: bool
    thres2_set: bool
    key1: int
    key2: int
    len2: int
    rand: int
    step: int
    nonfinite: bool
    compacted: bool
    n_compacted: int
    phase_us: list  # k_compress phase durations (device globaltimer, CTA 0)
    ef_compacted: bool  # the entries came from the EF pass (predicted key), no whole-vector count pass
    nnz_not_counted: int  # bit i: trials[i]'s count was not taken (its threshold lay below that key;
                          # only nnz > k is known) and trials[i][3] == NNZ_NOT_COUNTED


class _DeviceView:
    """A float32 torch tensor aliasing libtk-owned device memory (via __cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, device):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False), "version": 3,
                                         "strides": None}
        self.device = device

    def tensor(self):
        with torch.cuda.device(self.device):
            return torch.as_tensor(self, device=self.device)


class Context:
    """One rank's libtk context (tk_init).  ``d, rho, n_iters`` follow the paper's statement of
    the problem (x in R^d, k = rho*d, N samplings, P workers, m x n for HiTopKComm).
    ``select="exact"`` replaces MSTopK by the exact top-k of Eq. 2 (ties -> lower index),
    ``select="prose"`` runs MSTopK with the prose's halve/double threshold search (Q33);
    ``wire="f16"`` sends the values as binary16 (Fig. 7's FP16, reading Q31).
    Execution options (none changes a result bit): ``exact_trial_counts`` (count every trial
    exactly, for parity logs), ``ef_compaction``, ``first_pass_keys``, ``check_selection``,
    ``push_timeout_ms``; ``loopback=True`` emulates rank ``rank`` of ``nranks`` on this GPU
    without communicators (single-GPU tests of the multi-GPU kernels)."""

    def __init__(self, d: int, rho: float = 0.001, n_iters: int = 10, *, k: int = 0, nranks: int = 1, rank: int = 0,
                 group_size: int = 1, seed: int = 0, rand_mode: str = "seeded", error_feedback: bool = True,
                 step4: str = "dense", levels_per_pass: int = 0, device: int | None = None, uid: bytes | None = None,
                 stream: torch.cuda.Stream | None = None, rs_mode: str = "ordered", ag_mode: str = "push",
                 select: str = "mstopk", wire: str = "f32", exact_trial_counts: bool = False,
                 ef_compaction: bool = True, first_pass_keys: int = 0, check_selection: bool = False,
                 push_timeout_ms: int = 0, loopback: bool = False):
        if not torch.cuda.is_available():
            raise RuntimeError("libtk needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        dev = torch.cuda.current_device() if device is None else int(device)
        self.device = torch.device("cuda", dev)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        cfg = _Config(d=int(d), rho=float(rho), k=int(k), n_iters=int(n_iters), nranks=int(nranks), rank=int(rank),
                      group_size=int(group_size), seed=int(seed) & ((1 << 64) - 1),
                      rand_mode={"seeded": 0, "first": 1}[rand_mode], error_feedback=1 if error_feedback else 0,
                      step4={"dense": 0, "sparse": 1}[step4], levels_per_pass=int(levels_per_pass), device=dev,
                      rs_mode={"ordered": 0, "nccl": 1}[rs_mode], ag_mode={"push": 0, "nccl": 1}[ag_mode],
                      select={"mstopk": 0, "exact": 1, "prose": 2}[select], wire={"f32": 0, "f16": 1}[wire],
                      exact_trial_counts=1 if exact_trial_counts else 0,
                      disable_ef_compaction=0 if ef_compaction else 1, first_pass_keys=int(first_pass_keys),
                      check_selection=1 if check_selection else 0, push_timeout_ms=int(push_timeout_ms),
                      loopback=1 if loopback else 0)
        self._ctx = ctypes.c_void_p()
        if nranks > 1 and uid is None and not loopback:
            raise ValueError("nranks > 1 needs the NCCL unique id (broadcast_unique_id())")
        st = _lib.tk_init(ctypes.byref(cfg), uid, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(self._ctx))
        if st != 0:
            raise TkError(st, "tk_init failed (" + _lib.tk_status_string(st).decode() + ")")
        k_, L, P, m, n = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32()
        self._check(_lib.tk_query(self._ctx, ctypes.byref(k_), ctypes.byref(L), ctypes.byref(P), ctypes.byref(m),
                                  ctypes.byref(n)))
        self.d, self.k, self.seg_len = int(d), k_.value, L.value
        self.nranks, self.m, self.n, self.rank = P.value, m.value, n.value, int(rank)
        self.error_feedback = bool(error_feedback)
        self.wire = wire
        self.select = select
        # u32 words of one packed chunk: [idx k | fp32 val k] or [idx k | binary16 val k (padded)]
        self.chunk_words = 2 * self.k if wire == "f32" else self.k + (self.k + 1) // 2

    # -------------------------------------------------------------------------------------
    def _check(self, st):
        if st != 0:
            raise TkError(st, _lib.tk_last_error(self._ctx).decode(errors="replace"))

    def _empty(self, n, dtype):
        return torch.empty(n, dtype=dtype, device=self.device)

    def _p(self, t, name, dtype, numel=None):
        return _ptr(t, name, dtype, numel, self.device)

    @property
    def chunks(self) -> int:
        return self.nranks if self.n == 1 else self.m

    @property
    def out_len(self) -> int:
        """Length of a decompression output: d (flat) or the segment d/n (HiTopKComm)."""
        return self.d if self.n == 1 else self.seg_len

    def compress(self, g, r=None, idx=None, val=None):
        """tk_compress: returns (idx uint32-as-int32 tensor, val float32 tensor)."""
        idx = self._empty(self.k, torch.int32) if idx is None else idx
        val = self._empty(self.k, torch.float32) if val is None else val
        self._check(_lib.tk_compress(self._ctx, self._p(g, "g", torch.float32, self.d),
                                     self._p(r, "r", torch.float32, self.d) if self.error_feedback else None,
                                     self._p(idx, "idx", torch.int32, self.k), self._p(val, "val", torch.float32, self.k)))
        return idx, val

    def compress_segment(self, srcs, r=None, idx=None, val=None):
        """tk_compress_segment: MSTopK of the ordered sum of the source segments (HiTopKComm steps
        1-2, Eq. 4-5) (+ r with error feedback); srcs = 1, 2, 4 or 8 CUDA tensors of seg_len
        floats (local, or views of peer memory).  Returns (idx, val) of k~ pairs."""
        srcs = list(srcs)
        idx = self._empty(self.k, torch.int32) if idx is None else idx
        val = self._empty(self.k, torch.float32) if val is None else val
        arr = (ctypes.c_void_p * len(srcs))(*[self._p(t, f"src[{i}]", torch.float32, self.seg_len).value
                                               for i, t in enumerate(srcs)])
        self._check(_lib.tk_compress_segment(self._ctx, arr, len(srcs),
                                             self._p(r, "r", torch.float32, self.seg_len) if self.error_feedback else None,
                                             self._p(idx, "idx", torch.int32, self.k),
                                             self._p(val, "val", torch.float32, self.k)))
        return idx, val

    def sparse_allgather(self, idx, val, gathered=None):
        gathered = self._empty(self.chunks * self.chunk_words, torch.int32) if gathered is None else gathered
        self._check(_lib.tk_sparse_allgather(self._ctx, self._p(idx, "idx", torch.int32, self.k),
                                             self._p(val, "val", torch.float32, self.k),
                                             self._p(gathered, "gathered", torch.int32, self.chunks * self.chunk_words)))
        return gathered

    def decompress(self, gathered, nchunks=None, out=None):
        out = self._empty(self.out_len, torch.float32) if out is None else out
        nch = self.chunks if nchunks is None else int(nchunks)
        self._check(_lib.tk_decompress(self._ctx, self._p(gathered, "gathered", torch.int32, nch * self.chunk_words),
                                       nch, self._p(out, "out", torch.float32, self.out_len)))
        return out

    def step(self, g, r=None, out=None, gathered=None):
        """tk_step: one whole iteration; returns the dense aggregated gradient."""
        out = self._empty(self.d, torch.float32) if out is None else out
        self._check(_lib.tk_step(self._ctx, self._p(g, "g", torch.float32, self.d),
                                 self._p(r, "r", torch.float32, self.seg_len) if self.error_feedback else None,
                                 self._p(out, "out", torch.float32, self.d),
                                 self._p(gathered, "gathered", torch.int32, self.chunks * self.chunk_words)
                                 if gathered is not None else None))
        return out

    def step_sgd(self, g, r, w, lr: float, out=None, gathered=None):
        """tk_step_sgd: one iteration plus Eq. 1's update w -= lr * aggregate, fused into the
        decompression; w is updated in place (out optional)."""
        self._check(_lib.tk_step_sgd(self._ctx, self._p(g, "g", torch.float32, self.d),
                                     self._p(r, "r", torch.float32, self.seg_len) if self.error_feedback else None,
                                     self._p(w, "w", torch.float32, self.d), ctypes.c_float(lr),
                                     self._p(out, "out", torch.float32, self.d) if out is not None else None,
                                     self._p(gathered, "gathered", torch.int32, self.chunks * self.chunk_words)
                                     if gathered is not None else None))
        return w

    # loopback (single-GPU emulation of the fused all-gather, tk_loopback_*): a k-packet chunk is
    # k x 16 bytes, held here as int64 tensors of 2k words
    def loopback_push(self, g, r, chunk, slots, tag: int):
        """tk_loopback_push: compress (into the plain packed `chunk`) and write this rank's pairs as
        packets tagged `tag` to every slot (int64 tensors of >= 2k elements)."""
        slots = list(slots)
        arr = (ctypes.c_void_p * len(slots))(*[self._p(t, f"slot[{i}]", torch.int64, 2 * self.k).value
                                               for i, t in enumerate(slots)])
        self._check(_lib.tk_loopback_push(self._ctx, self._p(g, "g", torch.float32, self.d),
                                          self._p(r, "r", torch.float32, self.d) if self.error_feedback else None,
                                          self._p(chunk, "chunk", torch.int32, self.chunk_words), arr, len(slots),
                                          int(tag)))

    def loopback_decompress(self, packets, nchunks: int, tag: int, out=None, plain_out=None):
        """tk_loopback_decompress: rank-ordered decompression of nchunks packet chunks that waits for
        `tag` in every packet; returns out (and fills plain_out, [nchunks][chunk_words], if given)."""
        out = self._empty(self.out_len, torch.float32) if out is None else out
        self._check(_lib.tk_loopback_decompress(
            self._ctx, self._p(packets, "packets", torch.int64, 2 * self.k * nchunks), int(nchunks), int(tag),
            self._p(out, "out", torch.float32, self.out_len),
            self._p(plain_out, "plain_out", torch.int32, nchunks * self.chunk_words) if plain_out is not None else None))
        return out

    def step_host(self, g_host, gathered_host=None, out_host=None):
        """tk_step_host: HOST buffers in/out (numpy or pinned CPU tensors); synchronous."""
        def hp(a, n, name):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                if a.is_cuda or not a.is_contiguous():
                    raise ValueError(f"{name} must be a contiguous host tensor")
                if a.numel() * a.element_size() < 4 * n:
                    raise ValueError(f"{name} holds fewer than {n} 4-byte words")
                return ctypes.c_void_p(a.data_ptr())
            if not a.flags["C_CONTIGUOUS"] or a.nbytes < 4 * n:
                raise ValueError(f"{name} must be contiguous with >= {n} 4-byte words")
            return ctypes.c_void_p(a.ctypes.data)
        self._check(_lib.tk_step_host(self._ctx, hp(g_host, self.d, "g_host"),
                                      hp(gathered_host, self.chunks * self.chunk_words, "gathered_host"),
                                      hp(out_host, self.d, "out_host")))
        return gathered_host, out_host

    def stats(self) -> Stats:
        s = _Stats()
        st = _lib.tk_get_stats(self._ctx, ctypes.byref(s))
        if st not in (0, 4):
            self._check(st)
        trials = [(s.ratio[i], s.thres[i], s.key[i], s.nnz[i]) for i in range(s.n_trials)]
        return Stats(mean=s.mean, max_bits=s.max_bits, trials=trials, k=s.k, k1=s.k1, k2=s.k2, thres1=s.thres1,
                     thres2=s.thres2, thres1_set=bool(s.thres1_set), thres2_set=bool(s.thres2_set), key1=s.key1,
                     key2=s.key2, len2=s.len2, rand=s.rand_start, step=s.step, nonfinite=bool(s.nonfinite),
                     compacted=bool(s.compacted), n_compacted=int(s.n_compacted),
                     phase_us=[(s.phase_ns[i + 1] - s.phase_ns[i]) / 1e3 for i in range(max(0, s.n_phases - 1))],
                     ef_compacted=bool(s.ef_compacted), nnz_not_counted=int(s.nnz_not_counted))

    def decompress_replicated(self, gathered, outs, nchunks=None):
        """tk_decompress_replicated: the rank-ordered decompression written to every tensor in outs
        (each out_len floats) - HiTopKComm's fused dense step 4 writes a segment to the node peers."""
        outs = list(outs)
        nch = self.chunks if nchunks is None else int(nchunks)
        arr = (ctypes.c_void_p * len(outs))(*[self._p(t, f"outs[{i}]", torch.float32, self.out_len).value
                                              for i, t in enumerate(outs)])
        self._check(_lib.tk_decompress_replicated(self._ctx, self._p(gathered, "gathered", torch.int32,
                                                                     nch * self.chunk_words), nch, arr, len(outs)))
        return outs

    def alloc_symmetric(self, numel: int):
        """tk_alloc_symmetric (collective over the GPUs of a virtual node): a float32 tensor of numel
        elements whose peers' copies libtk maps; pass it as g (or out) to step() to skip the copy-in
        (or to fuse the dense step 4).  Lives until free_symmetric / close."""
        p = ctypes.c_void_p()
        self._check(_lib.tk_alloc_symmetric(self._ctx, 4 * int(numel), ctypes.byref(p)))
        t = _DeviceView(p.value, int(numel), self.device).tensor()
        self._syms = getattr(self, "_syms", []) + [t]
        return t

    def free_symmetric(self, t):
        self._check(_lib.tk_free_symmetric(self._ctx, ctypes.c_void_p(t.data_ptr())))
        self._syms = [x for x in getattr(self, "_syms", []) if x.data_ptr() != t.data_ptr()]

    def input_buffer(self):
        """HiTopKComm ordered mode: a torch view of libtk's peer-visible gradient buffer (write the
        gradient here and pass it as g to step() to skip the copy-in); None in flat mode."""
        p = ctypes.c_void_p()
        self._check(_lib.tk_input_buffer(self._ctx, ctypes.byref(p)))
        if not p.value:
            return None
        # wrap the device pointer without copying (the buffer lives as long as the context)
        return _DeviceView(p.value, self.d, self.device).tensor()

    def set_step(self, step: int):
        self._check(_lib.tk_set_step(self._ctx, int(step)))

    def profile_begin(self, max_steps: int):
        self._check(_lib.tk_profile_begin(self._ctx, int(max_steps)))

    def profile_end(self) -> dict:
        """{stage name: (total ms, launches)} over the steps since profile_begin."""
        ms = (ctypes.c_double * NSTAGES)()
        ln = (ctypes.c_uint32 * NSTAGES)()
        self._check(_lib.tk_profile_end(self._ctx, ms, ln))
        return {_lib.tk_stage_name(i).decode(): (ms[i], ln[i]) for i in range(1, NSTAGES) if ln[i] > 0}

    @property
    def launches(self) -> int:
        return int(_lib.tk_launch_count(self._ctx))

    def close(self):
        if self._ctx:
            _lib.tk_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------------------------------
# Bucketed multi-tensor step (second half): the "tensor fusion" the paper names as
# the way gradient communication overlaps backpropagation (§2.2), reading Q32 of DESIGN.md: a bucket is the concatenation of its layers' gradients in list order, and
# one tk_step runs on it — one MSTopK selection over the fused d = sum d_l with k = rho * d
# (P:197), one sparse all-gather, one decompression.  The layers are zero-copy views of the
# bucket's flat buffers, so fusion costs no copy pass; this module only computes offsets.

def bucket_layout(shapes) -> list:
    """[(offset, numel, shape)] of each layer in the fused flat buffer: contiguous, in list
    order, no padding (padding would add zeros to the mean of Alg. 1 l.2)."""
    out, off = [], 0
    for s in shapes:
        shape = (int(s),) if isinstance(s, int) else tuple(int(x) for x in s)
        if any(x < 0 for x in shape):
            raise ValueError(f"negative dimension in layer shape {shape}")
        n = 1
        for x in shape:
            n *= x
        out.append((off, n, shape))
        off += n
    if off == 0:
        raise ValueError("a bucket needs at least one element")
    if off >= 1 << 32:
        raise ValueError("a bucket holds < 2^32 elements (u32 indices on the wire, Q15)")
    return out


class Bucket:
    """Many layers, one tk_step.  ``grads[i]`` / ``outputs[i]`` are views (layer shapes) of the
    flat gradient / aggregate buffers; write the layer gradients into ``grads`` (or let autograd
    accumulate into them), then ``step()`` or ``step_sgd(params_flat, lr)``.  Context keyword
    arguments (nranks, rank, uid, select, wire, group_size, ...) pass through to ``Context``."""

    def __init__(self, shapes, rho: float = 0.001, n_iters: int = 10, **ctx_kwargs):
        self.layout = bucket_layout(shapes)
        self.d = sum(n for _, n, _ in self.layout)
        self.ctx = Context(self.d, rho=rho, n_iters=n_iters, **ctx_kwargs)
        dev = self.ctx.device
        # HiTopKComm ordered mode: the gradient lives in libtk's peer-visible buffer (no copy-in)
        flat = self.ctx.input_buffer()
        self.flat_grad = torch.zeros(self.d, dtype=torch.float32, device=dev) if flat is None else flat
        self.flat_grad.zero_()
        # EF residual of this rank's part of the selection: the whole bucket (flat) or the
        # rank's segment of length d / n (HiTopKComm, Eq. 4-5)
        self.residual = torch.zeros(self.ctx.seg_len, dtype=torch.float32, device=dev)
        self.flat_out = torch.empty(self.d, dtype=torch.float32, device=dev)
        self.grads = self.views(self.flat_grad)
        self.outputs = self.views(self.flat_out)

    def views(self, flat):
        """Layer-shaped views of a flat buffer of the bucket's size (e.g. the parameters)."""
        if flat.numel() != self.d:
            raise ValueError(f"flat buffer has {flat.numel()} elements, the bucket {self.d}")
        return [flat[o:o + n].view(s) for o, n, s in self.layout]

    def step(self, gathered=None):
        """One iteration over the whole bucket; returns the layer-shaped aggregates."""
        self.ctx.step(self.flat_grad, self.residual, out=self.flat_out, gathered=gathered)
        return self.outputs

    def step_sgd(self, params_flat, lr: float, keep_out: bool = False):
        """One iteration plus Eq. 1's update of the bucket's flat parameter buffer, fused into
        the decompression (tk_step_sgd)."""
        self.ctx.step_sgd(self.flat_grad, self.residual, params_flat, lr,
                          out=self.flat_out if keep_out else None)
        return params_flat

    def close(self):
        self.ctx.close()
