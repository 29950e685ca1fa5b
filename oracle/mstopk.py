"""CPU ORACLE for MSTopK (Alg. 1) and exact top-k (Eq. 2) — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this module.  The product path
(``paper_2010_10458_b200``) never does, and this module never imports the product.
It shares no code, header, table or constant generator with ``paper_2010_10458_b200/csrc``.

Citations: ``P:n`` = PAPER.md line n (arXiv 2010.10458, LaTeX source).  Every reading of a
silent / ambiguous passage is listed in DESIGN.md §"Readings" with its Q-number.

Precision: the paper fixes none.  Per DESIGN.md: fp32 data (Eq. 3 bills FP32 elements,
P:201), fp64 mean / thresholds (Q3, Q4), literal ``a >= thres`` comparisons done in fp64.

Parity pins: every function here is pinned by ``tests/test_oracle_pins.py`` against
hand-worked examples (tests/golden/*.json), closed forms, error bounds and brute force.
Un-pinnable: the authors' own bit-level choices (their TF kernel, RNG, fp32 mean) —
"parity unpinned" for paper-level numbers (Figs. 6-8 are stripped from PAPER.md).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .rng import window_hash

RAND_SEEDED = 0
RAND_FIRST = 1

F32_INF_BITS = 0x7F800000


def k_from_density(d: int, rho: float) -> int:
    """k = rho * d, read as max(1, floor(fl64(rho*d))) (Q13)."""
    if d < 1:
        raise ValueError("d must be >= 1")
    if not (0.0 < rho <= 1.0):
        raise ValueError("rho must lie in (0, 1]")
    return max(1, int(math.floor(float(rho) * float(d))))


def magnitudes(x: np.ndarray) -> np.ndarray:
    """Alg. 1 line 1: a = abs(x).  fp32 abs = clear the sign bit (exact)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    return np.abs(x)


def pairwise_sum_f64(a: np.ndarray) -> float:
    """Canonical fp64 pairwise sum (reading Q3; P:156 leaves the order unspecified).

    Leaves are (double)a_i, zero-padded to D = next power of two >= d; every level adds
    adjacent pairs: PW(lo,hi) = PW(lo,mid) + PW(mid,hi).  Level-by-level evaluation below
    pairs exactly the same nodes as the recursive definition.
    """
    d = a.shape[0]
    D = 1 if d <= 1 else 1 << (d - 1).bit_length()
    v = np.zeros(D, dtype=np.float64)
    v[:d] = a.astype(np.float64)
    while v.shape[0] > 1:
        v = v[0::2] + v[1::2]
    return float(v[0])


def ceil_f32_bits(t: float) -> int:
    """Bits of the smallest fp32 value >= t (t finite, >= 0).  Used only to REPORT the
    integer key that an implementation comparing fp32 bit patterns must use (Q4); the
    oracle's own comparisons are the literal fp64 ``a >= thres`` of Alg. 1."""
    if t <= 0.0:
        return 0
    f = np.float32(t)  # round to nearest even
    if float(f) < t:
        f = np.nextafter(f, np.float32(np.inf))
    return int(np.array([f], dtype=np.float32).view(np.uint32)[0])


@dataclass
class MSTopKResult:
    idx: np.ndarray            # uint32[k], ascending (Q11)
    val: np.ndarray            # float32[k], x[idx] bit-copied (Alg. 1 l.29)
    mean: float                # a-bar (fp64)
    u: float                   # max |x| (fp32 value, held as a Python float)
    k: int
    k1: int
    k2: int
    thres1: float
    thres2: float
    thres1_set: bool
    thres2_set: bool
    key1: int                  # ceil_f32 bits of thres1, or +inf bits when unset (Q8)
    key2: int                  # ceil_f32 bits of thres2, or 0 when unset (Q9)
    len2: int
    rand: int
    trials: list = field(default_factory=list)  # (ratio, thres, key, nnz) per iteration


def mstopk(x: np.ndarray, k: int, n_iters: int, *, seed: int = 0, step: int = 0, rank: int = 0,
           rand_mode: int = RAND_SEEDED) -> MSTopKResult:
    """MSTopK, Algorithm 1, step by step in the paper's order and notation."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    d = x.shape[0]
    if d < 1:
        raise ValueError("d must be >= 1")
    if not (1 <= k <= d):
        raise ValueError("k must lie in [1, d]")
    if not (1 <= n_iters <= 52):
        raise ValueError("N must lie in [1, 52] (Q5)")
    # l.1  a = abs(x)
    a = magnitudes(x)
    if not np.all(np.isfinite(a)):
        raise ValueError("non-finite input (Q24)")
    a64 = a.astype(np.float64)
    # l.2  a-bar = mean(a): canonical fp64 pairwise sum / d (Q3)
    abar = pairwise_sum_f64(a) / float(d)
    # l.3  u = max(a)
    u = float(a.max())
    # l.4-6
    l, r = 0.0, 1.0
    k1, k2 = 0, d
    thres1, thres2 = 0.0, 0.0
    set1, set2 = False, False
    trials = []
    # l.7-24
    for _ in range(n_iters):
        ratio = l + (r - l) / 2                      # l.8 (exact dyadic, Q5)
        thres = abar + ratio * (u - abar)            # l.9: three separate fp64 RN ops (Q4)
        nnz = int(np.count_nonzero(a64 >= thres))    # l.10
        trials.append((ratio, thres, ceil_f32_bits(thres), nnz))
        if nnz <= k:                                 # l.11
            r = ratio                                # l.12
            if nnz > k1:                             # l.13 (strict, Q7)
                k1 = nnz
                thres1 = thres
                set1 = True
        elif nnz > k:                                # l.17
            l = ratio                                # l.18
            if nnz < k2:                             # l.19 (strict, Q7)
                k2 = nnz
                thres2 = thres
                set2 = True
    # l.25  iota1 = nonzero_indices(a >= thres1); guard k1 == 0 -> empty (Q8)
    if k1 > 0:
        in1 = a64 >= thres1
    else:
        in1 = np.zeros(d, dtype=bool)
    # l.26  iota2 = nonzero_indices(a < thres1 and a >= thres2); thres2 unset = 0 (Q9)
    in2 = (~in1) & (a64 >= thres2)
    iota1 = np.nonzero(in1)[0]
    iota2 = np.nonzero(in2)[0]
    need = k - k1
    # l.27  rand = random(0, len(iota2) - (k - k1) + 1): half-open uniform integer (Q10)
    R = len(iota2) - need + 1
    if R < 1:
        raise AssertionError("window range R < 1 — impossible under readings Q8/Q9")
    if rand_mode == RAND_FIRST:
        rand = 0
    else:
        rand = (window_hash(seed, step, rank, 0) * R) >> 64
    # l.28  iota = concat(iota1, iota2[rand : rand + k - k1]); emitted ascending (Q11)
    iota = np.concatenate([iota1, iota2[rand:rand + need]])
    iota = np.sort(iota).astype(np.uint32)
    # l.29  kappa = x[iota] (signed values, bit-copied, Q12)
    kappa = x[iota.astype(np.int64)].copy()
    key1 = ceil_f32_bits(thres1) if set1 else F32_INF_BITS
    key2 = ceil_f32_bits(thres2) if set2 else 0
    return MSTopKResult(idx=iota, val=kappa, mean=abar, u=u, k=k, k1=k1, k2=k2, thres1=thres1,
                        thres2=thres2, thres1_set=set1, thres2_set=set2, key1=key1, key2=key2,
                        len2=int(len(iota2)), rand=int(rand), trials=trials)


def exact_topk(x: np.ndarray, k: int):
    """Exact top-k (Eq. 2), read as "the k largest |x_i|, ties -> lower index"
    (Q6): a full stable sort by (-|x_i|, i).  Returns (idx ascending uint32, val float32)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    d = x.shape[0]
    if not (1 <= k <= d):
        raise ValueError("k must lie in [1, d]")
    a64 = np.abs(x).astype(np.float64)
    order = np.lexsort((np.arange(d), -a64))  # primary: -|x|, secondary: index
    idx = np.sort(order[:k]).astype(np.uint32)
    return idx, x[idx.astype(np.int64)].copy()


@dataclass
class ExactResult:
    """Exact top-k (Eq. 2) of one vector, plus the order statistic that decides it."""
    idx: np.ndarray     # uint32[k], ascending
    val: np.ndarray     # float32[k], signed acc values (Q12)
    k: int
    kth_bits: int       # bits(|x|) of the k-th largest magnitude (T)
    k1: int             # #{i : bits(|x_i|) > T}   (all selected)
    k2: int             # #{i : bits(|x_i|) >= T}  (the first k - k1 of the ties at T, by index, are selected)


def exact_select(x: np.ndarray, k: int) -> ExactResult:
    """exact_topk plus its k-th order statistic, read off the sorted magnitudes (definitions only)."""
    idx, val = exact_topk(x, k)
    bits = magnitudes(np.ascontiguousarray(x, dtype=np.float32)).view(np.uint32)
    T = int(np.sort(bits)[::-1][k - 1])
    return ExactResult(idx=idx, val=val, k=k, kth_bits=T, k1=int(np.count_nonzero(bits > T)),
                       k2=int(np.count_nonzero(bits >= T)))


@dataclass
class CompressResult:
    sel: MSTopKResult
    acc: np.ndarray        # the vector MSTopK ran on (g + r with error feedback, else g)
    residual: np.ndarray   # r' (error feedback) — None when EF is off
    sent: np.ndarray       # the values put on the wire: sel.val, or their binary16 rounding (F3)


def compress(g: np.ndarray, r: np.ndarray | None, k: int, n_iters: int, *, seed: int = 0,
             step: int = 0, rank: int = 0, rand_mode: int = RAND_SEEDED,
             error_feedback: bool = True, selector: str = "mstopk", wire: str = "f32") -> CompressResult:
    """One rank's compression with error feedback (BJ north_star; Q14):
    acc = fl32(g + r); (kappa, iota) = MSTopK(acc) -- or, with selector="exact", the exact top-k
    of Eq. 2 (TopK-SGD; ties -> lower index, Q6); r' = acc with the sent entries := +0.0."""
    g = np.ascontiguousarray(g, dtype=np.float32)
    if error_feedback:
        acc = (g + np.ascontiguousarray(r, dtype=np.float32)).astype(np.float32)
    else:
        acc = g.copy()
    if selector == "exact":
        sel = exact_select(acc, k)
    elif selector == "mstopk":
        sel = mstopk(acc, k, n_iters, seed=seed, step=step, rank=rank, rand_mode=rand_mode)
    elif selector == "prose":
        sel = mstopk_prose(acc, k, n_iters, seed=seed, step=step, rank=rank, rand_mode=rand_mode)
    else:
        raise ValueError(f"unknown selector {selector!r}")
    if wire == "f32":
        sent = sel.val.copy()
    elif wire == "f16":
        # FP16 wire values (F3; Fig. 7 ran FP16; reading Q31): round-to-nearest binary16 of
        # the value clamped to the finite range, widened back exactly
        sent = np.clip(sel.val, np.float32(-65504.0), np.float32(65504.0)).astype(np.float16).astype(np.float32)
    else:
        raise ValueError(f"unknown wire format {wire!r}")
    res = None
    if error_feedback:
        res = acc.copy()
        ii = sel.idx.astype(np.int64)
        # Q14: the sent entries keep what was not sent: +0 (fp32 wire), fl32(v - sent) (FP16 wire)
        res[ii] = np.float32(0.0) if wire == "f32" else (sel.val - sent).astype(np.float32)
    return CompressResult(sel=sel, acc=acc, residual=res, sent=sent)


def mstopk_prose(x: np.ndarray, k: int, n_iters: int, *, seed: int = 0, step: int = 0, rank: int = 0,
                 rand_mode: int = RAND_SEEDED) -> MSTopKResult:
    """MSTopK with the threshold search the PROSE describes (SURVEY F3 `TK_SEARCH_PROSE`),
    reading Q33 of DESIGN.md, step by step in the prose's order:

    - "We first use the average value (a-bar) ... as the threshold (thres1)": trial 1 is t = a-bar.
    - "If the dimension of kappa is smaller (or larger) than k, then we half (or double) thres1 as
      thres2 ... we repeat the above search": while no trial has yet landed on each side of the
      k-th magnitude, the next trial is t/2 when nnz(a >= t) < k, 2t when nnz > k (exact in fp64).
      nnz == k counts as the "not larger" side, as in Alg. 1 l.11.
    - "then we can further narrow down the thresholds with the same pattern of search": once
      bracketed, the next trial is the fp64 midpoint of the two bracketing thresholds.
    - "We set a fixed number of searches (say N), and finally we select k elements using the
      chosen two thresholds": after N trials (k1, thres1) / (k2, thres2) are updated exactly as
      Alg. 1 l.11-20 does, and the selection is Alg. 1 l.25-29 unchanged (Q8-Q12).
    """
    x = np.ascontiguousarray(x, dtype=np.float32)
    d = x.shape[0]
    if d < 1:
        raise ValueError("d must be >= 1")
    if not (1 <= k <= d):
        raise ValueError("k must lie in [1, d]")
    if not (1 <= n_iters <= 52):
        raise ValueError("N must lie in [1, 52] (Q5)")
    a = magnitudes(x)
    if not np.all(np.isfinite(a)):
        raise ValueError("non-finite input (Q24)")
    a64 = a.astype(np.float64)
    abar = pairwise_sum_f64(a) / float(d)
    u = float(a.max())
    k1, k2 = 0, d
    thres1, thres2 = 0.0, 0.0
    set1, set2 = False, False
    t_hi = None   # smallest trial threshold seen with nnz <= k
    t_lo = None   # largest trial threshold seen with nnz > k
    t = abar
    trials = []
    for _ in range(n_iters):
        nnz = int(np.count_nonzero(a64 >= t))
        trials.append((float("nan"), t, ceil_f32_bits(t), nnz))
        if nnz <= k:
            t_hi = t if t_hi is None else min(t_hi, t)
            if nnz > k1:
                k1, thres1, set1 = nnz, t, True
        else:
            t_lo = t if t_lo is None else max(t_lo, t)
            if nnz < k2:
                k2, thres2, set2 = nnz, t, True
        if t_hi is None:
            t = 2.0 * t          # too many selected: double
        elif t_lo is None:
            t = t / 2.0          # too few selected: halve
        else:
            t = t_lo + (t_hi - t_lo) / 2.0
    in1 = a64 >= thres1 if k1 > 0 else np.zeros(d, dtype=bool)
    in2 = (~in1) & (a64 >= thres2)
    iota1 = np.nonzero(in1)[0]
    iota2 = np.nonzero(in2)[0]
    need = k - k1
    R = len(iota2) - need + 1
    if R < 1:
        raise AssertionError("window range R < 1 — impossible under readings Q8/Q9")
    rand = 0 if rand_mode == RAND_FIRST else (window_hash(seed, step, rank, 0) * R) >> 64
    iota = np.sort(np.concatenate([iota1, iota2[rand:rand + need]])).astype(np.uint32)
    kappa = x[iota.astype(np.int64)].copy()
    key1 = ceil_f32_bits(thres1) if set1 else F32_INF_BITS
    key2 = ceil_f32_bits(thres2) if set2 else 0
    return MSTopKResult(idx=iota, val=kappa, mean=abar, u=u, k=k, k1=k1, k2=k2, thres1=thres1,
                        thres2=thres2, thres1_set=set1, thres2_set=set2, key1=key1, key2=key2,
                        len2=int(len(iota2)), rand=int(rand), trials=trials)
