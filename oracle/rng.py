"""CPU ORACLE — window RNG for Alg. 1 l.27 — TEST INFRASTRUCTURE ONLY.

The paper draws ``rand = random(0, len(iota2)-(k-k1)+1)`` without naming a generator
(reading Q10).  Both sides implement the same counter-based generator independently:
the SplitMix64 finaliser chained over (seed, step, rank, call).  Pinned by the published
SplitMix64 stream for seed 0 in tests/test_oracle_pins.py.
"""
MASK64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """One SplitMix64 step applied to state x (increment, then the finaliser), mod 2^64."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    z = x
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def window_hash(seed: int, step: int, rank: int, call: int) -> int:
    """H(s,t,p,c) = sm(sm(sm(sm(s) ^ t) ^ p) ^ c)."""
    h = splitmix64(seed & MASK64)
    h = splitmix64(h ^ (step & MASK64))
    h = splitmix64(h ^ (rank & MASK64))
    return splitmix64(h ^ (call & MASK64))
