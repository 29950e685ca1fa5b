"""CPU oracle for the MSTopK + sparse-aggregation hot path — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct numpy implementations of what arXiv 2010.10458's
CommLib computes (Alg. 1 MSTopK, Eq. 2 exact top-k, §3.2 NaiveAG, Alg. 2 HiTopKComm),
written from PAPER.md and the readings listed in DESIGN.md.  Importable only from
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (``cpu_baseline`` and
``--impl reference``).  Shares no code with ``paper_2010_10458_b200``.
"""
from .mstopk import (RAND_FIRST, RAND_SEEDED, CompressResult, ExactResult, MSTopKResult, ceil_f32_bits,
                     compress, exact_select, exact_topk, k_from_density, magnitudes, mstopk, mstopk_prose,
                     pairwise_sum_f64)
from .aggregate import (FlatResult, HiTopKResult, allgather, chunk_words, decompress, flat_step, hitopk_step,
                        pack, reduce_scatter_ordered, sgd_update)
from .rng import splitmix64, window_hash

__all__ = [
    "RAND_FIRST", "RAND_SEEDED", "CompressResult", "ExactResult", "MSTopKResult", "exact_select", "ceil_f32_bits", "compress", "exact_topk",
    "k_from_density", "magnitudes", "mstopk", "mstopk_prose", "pairwise_sum_f64", "FlatResult", "HiTopKResult", "allgather",
    "decompress", "flat_step", "hitopk_step", "pack", "reduce_scatter_ordered", "sgd_update", "chunk_words", "splitmix64", "window_hash",
]
