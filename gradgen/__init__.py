"""Seeded synthetic gradient generators shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no |x|, no mean, no threshold, no
selection, no accumulation).  It only produces input bytes: fp32 gradient vectors with
the value distributions and structure described in DESIGN.md §"Input recipe".  Both the
oracle (``oracle/``) and the GPU path (``paper_2010_10458_b200``) consume the exact same
bytes: the arrays are generated on the host with numpy's PCG64 and uploaded, never
regenerated on the GPU (libm differs).

Distributions (the paper states none: "different length of vectors", P:377
"randomly generated"):

* ``"G"``  iid N(0,1) fp32 (default).
* ``"L"``  layered, ResNet-like: d cut into 161 contiguous blocks (ResNet-50's layer
  count) at seeded sorted uniform cut points; block scale 10**U(-4,0) times N(0,1).
  The blocks and scales depend on (cfg, rank) only - the same network at every step - and
  the N(0,1) noise on the step.
* ``"H"``  Laplace(0,1) (heavy tailed).
* edge cases (correctness only): ``"zero"``, ``"const"``, ``"spike"``, ``"ties8"``
  (8 magnitude levels, massive ties), ``"denorm"``, ``"signed_zero"``.

Seeds: ``SeedSequence([201010458, cfg, rank, step])``.
"""
from __future__ import annotations

import numpy as np

BASE_SEED = 201010458
N_LAYERS = 161  # P:309, ResNet-50 layer count used for the layered profile

DISTS = ("G", "L", "H", "zero", "const", "spike", "ties8", "denorm", "signed_zero")


def rng_for(cfg: int, rank: int, step: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, int(cfg), int(rank), int(step)])))


def gradient(d: int, dist: str = "G", cfg: int = 0, rank: int = 0, step: int = 0) -> np.ndarray:
    """Return a seeded fp32 gradient of length ``d`` (C-contiguous, float32)."""
    d = int(d)
    g = rng_for(cfg, rank, step)
    if dist == "G":
        x = g.standard_normal(d, dtype=np.float32)
    elif dist == "L":
        x = g.standard_normal(d, dtype=np.float32)
        # the network (layer boundaries and per-layer scales) is the same at every step of a rank,
        # as in training; only the noise is drawn per step
        gl = rng_for(cfg, rank, 1 << 40)  # a step no caller uses: the network's own stream
        nl = min(N_LAYERS, max(1, d))
        cuts = np.sort(gl.integers(0, d + 1, size=nl - 1)) if nl > 1 else np.zeros(0, np.int64)
        bounds = np.concatenate([[0], cuts, [d]]).astype(np.int64)
        scales = (10.0 ** gl.uniform(-4.0, 0.0, size=nl)).astype(np.float32)
        for li in range(nl):
            lo, hi = bounds[li], bounds[li + 1]
            if hi > lo:
                x[lo:hi] *= scales[li]
    elif dist == "H":
        x = g.laplace(0.0, 1.0, size=d).astype(np.float32)
    elif dist == "zero":
        x = np.zeros(d, np.float32)
    elif dist == "const":
        x = np.full(d, np.float32(0.375), np.float32)
        x[g.random(d) < 0.5] *= np.float32(-1.0)
    elif dist == "spike":
        x = (g.standard_normal(d, dtype=np.float32) * np.float32(1e-3)).astype(np.float32)
        x[int(g.integers(0, d))] = np.float32(1e3)
    elif dist == "ties8":
        levels = np.array([0.0, 0.125, 0.25, 0.5, 1.0, 1.5, 2.0, 4.0], np.float32)
        x = levels[g.integers(0, 8, size=d)]
        x[g.random(d) < 0.5] *= np.float32(-1.0)
    elif dist == "denorm":
        x = (g.standard_normal(d, dtype=np.float32) * np.float32(1e-39)).astype(np.float32)
    elif dist == "signed_zero":
        x = g.standard_normal(d, dtype=np.float32)
        m = g.random(d)
        x[m < 0.3] = np.float32(0.0)
        x[(m >= 0.3) & (m < 0.6)] = np.float32(-0.0)
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    return np.ascontiguousarray(x, dtype=np.float32)


def residual_zero(d: int) -> np.ndarray:
    """Error-feedback residual at step 0 ('Residual: starts at 0')."""
    return np.zeros(int(d), np.float32)
