"""CPU ORACLE for sparse aggregation — NaiveAG (§3.2) and HiTopKComm (Alg. 2,
P:217-248) — TEST INFRASTRUCTURE ONLY (see oracle/mstopk.py header).

All P ranks are simulated in one process with plain loops; no NCCL, no GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mstopk import RAND_SEEDED, compress, k_from_density


def pack(idx: np.ndarray, val: np.ndarray, wire: str = "f32") -> np.ndarray:
    """Wire layout of one rank's chunk (Q15): uint32[2k] = [idx k | bits(val) k]; FP16 wire (F3,
    Q31): [idx k | binary16(val) k, zero-padded to whole u32 words] (val must be fp16-exact)."""
    idx = idx.astype(np.uint32)
    val = np.ascontiguousarray(val, np.float32)
    if wire == "f32":
        return np.concatenate([idx, val.view(np.uint32)])
    h = val.astype(np.float16)
    assert np.array_equal(h.astype(np.float32).view(np.uint32), val.view(np.uint32)), "values not fp16-exact"
    if len(h) % 2:
        h = np.concatenate([h, np.zeros(1, np.float16)])
    return np.concatenate([idx, h.view(np.uint32)])


def chunk_words(k: int, wire: str = "f32") -> int:
    return 2 * k if wire == "f32" else k + (k + 1) // 2


def allgather(chunks: list) -> np.ndarray:
    """All-Gather: rank-major concatenation of every rank's packed chunk."""
    return np.concatenate(chunks)


def decompress(gathered: np.ndarray, P: int, k: int, d: int, wire: str = "f32") -> np.ndarray:
    """Index accumulation (Alg. 2 l.17-21): out = 0; for p = 0..P-1 in rank
    order, out[iota_p] += kappa_p in fp32 RN (Q16).  Indices within one rank are distinct,
    so the vectorised per-rank update equals the element-by-element loop.  FP16 wire: the
    binary16 values are widened to fp32 exactly first."""
    g = np.ascontiguousarray(gathered, dtype=np.uint32).reshape(P, chunk_words(k, wire))
    out = np.zeros(d, dtype=np.float32)
    for p in range(P):
        idx = g[p, :k].astype(np.int64)
        if wire == "f32":
            val = g[p, k:].view(np.float32)
        else:
            val = g[p, k:].copy().view(np.float16)[:k].astype(np.float32)
        out[idx] = (out[idx] + val).astype(np.float32)
    return out


@dataclass
class FlatResult:
    out: np.ndarray
    gathered: np.ndarray
    per_rank: list   # CompressResult per rank


def flat_step(grads: list, residuals: list, rho: float, n_iters: int, *, seed: int = 0, step: int = 0,
              rand_mode: int = RAND_SEEDED, error_feedback: bool = True, k: int | None = None,
              selector: str = "mstopk", wire: str = "f32") -> FlatResult:
    """NaiveAG TopK-SGD aggregation (§5.3) with error feedback (BJ):
    compress on every rank, all-gather the packed pairs, decompress in rank order."""
    P = len(grads)
    d = grads[0].shape[0]
    kk = k if k is not None else k_from_density(d, rho)
    per = [compress(grads[p], residuals[p] if error_feedback else None, kk, n_iters, seed=seed, step=step,
                    rank=p, rand_mode=rand_mode, error_feedback=error_feedback, selector=selector, wire=wire)
           for p in range(P)]
    gathered = allgather([pack(c.sel.idx, c.sent, wire) for c in per])
    return FlatResult(out=decompress(gathered, P, kk, d, wire), gathered=gathered, per_rank=per)


def reduce_scatter_ordered(grads: list, n: int, i: int, j: int) -> np.ndarray:
    """HiTopKComm step 1 (Eq. 4; Alg. 2 l.2-4): GPU (i,j)'s segment
    g^{[j]} = sum_{q=0..n-1} g_{i,q}[jL:(j+1)L], summed in ascending q, left to right,
    fp32 RN, starting from g_{i,0} (Q20, Q21: half-open segments, d % n == 0)."""
    d = grads[0].shape[0]
    L = d // n
    s = grads[i * n + 0][j * L:(j + 1) * L].astype(np.float32).copy()
    for q in range(1, n):
        s = (s + grads[i * n + q][j * L:(j + 1) * L]).astype(np.float32)
    return s


@dataclass
class HiTopKResult:
    out: np.ndarray          # identical on every rank
    segments: list           # reduced segment per rank (after step 1)
    per_rank: list           # CompressResult per rank (segment-local indices)
    column_gathered: list    # per j: uint32[m][2k~]


def hitopk_step(grads: list, residuals: list, m: int, n: int, rho: float, n_iters: int, *, seed: int = 0,
                step: int = 0, rand_mode: int = RAND_SEEDED, error_feedback: bool = True,
                selector: str = "mstopk", wire: str = "f32") -> HiTopKResult:
    """HiTopKComm (Alg. 2) on m x n GPUs; world rank = i*n + j.
    residuals[rank] is the segment residual in R^{d/n} (Q22)."""
    P = m * n
    assert len(grads) == P
    d = grads[0].shape[0]
    if d % n != 0:
        raise ValueError("d % n != 0 (Q21)")
    L = d // n
    kt = k_from_density(L, rho)  # Alg. 2 l.5: k~ = rho * d / n (Q13)
    segs, per = [], []
    for i in range(m):
        for j in range(n):
            segs.append(reduce_scatter_ordered(grads, n, i, j))
    for rank in range(P):  # Alg. 2 l.6-8: MSTopK on every segment
        per.append(compress(segs[rank], residuals[rank] if error_feedback else None, kt, n_iters, seed=seed,
                            step=step, rank=rank, rand_mode=rand_mode, error_feedback=error_feedback,
                            selector=selector, wire=wire))
    col = []
    G = []
    for j in range(n):  # Alg. 2 l.11-14: column All-Gather among GPUs (0..m-1, j)
        gathered = allgather([pack(per[i * n + j].sel.idx, per[i * n + j].sent, wire) for i in range(m)])
        col.append(gathered)
        G.append(decompress(gathered, m, kt, L, wire))  # Alg. 2 l.15-20, groups in order (Q16, Q18)
    out = np.concatenate(G)  # Alg. 2 l.21-23: intra-node All-Gather of segments (Q18, Q19)
    return HiTopKResult(out=out, segments=segs, per_rank=per, column_gathered=col)


def sgd_update(w: np.ndarray, out: np.ndarray, lr: float) -> np.ndarray:
    """Eq. 1 with the sparse aggregate in place of sum_p g_t^p:
    w_{t+1} = w_t - eta * g~, elementwise in fp32: fl32(w - fl32(eta * g~)) (reading Q29)."""
    w = np.ascontiguousarray(w, dtype=np.float32)
    prod = (np.float32(lr) * np.ascontiguousarray(out, dtype=np.float32)).astype(np.float32)
    return (w - prod).astype(np.float32)
