"""GPU parity: libtk (through the C ABI via the thin binding) against the CPU oracle, element by
element on the same seeded inputs.  Bar (BASELINE.json north_star): thresholds, counts, index
sets, values and residuals bit-exact; rank-ordered aggregates bit-exact."""
import numpy as np
import pytest

import gradgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tk():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests selected but no CUDA device is visible")
    import paper_2010_10458_b200 as tk
    return tk


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _f32bits(t):
    return t.cpu().numpy().astype(np.float32).view(np.uint32)


NNZ_NOT_COUNTED = 0xFFFFFFFF


def _check_stats(st, ref, exact_counts=True):
    """Every field of the control block, bit for bit.  exact_counts (the parity suite's mode):
    every trial's nnz equals the oracle's count.  Default mode: a trial whose threshold lay below the
    EF-pass key reports NNZ_NOT_COUNTED and claims only nnz > k - checked exactly as claimed."""
    s = ref.sel
    assert st.mean == s.mean, (st.mean, s.mean)
    assert st.max_bits == int(np.float32(s.u).view(np.uint32))
    assert len(st.trials) == len(s.trials)
    if exact_counts:
        assert st.nnz_not_counted == 0
    for it, (a, b) in enumerate(zip(st.trials, s.trials)):
        same_ratio = (a[0] == b[0]) or (np.isnan(a[0]) and np.isnan(b[0]))  # prose search: no ratio
        assert same_ratio and a[1] == b[1] and a[2] == b[2], (it, a, b)
        if st.nnz_not_counted >> it & 1:
            assert a[3] == NNZ_NOT_COUNTED and b[3] > s.k, (it, a, b)
        else:
            assert a[3] == b[3], (it, a, b)
    assert (st.k1, st.k2) == (s.k1, s.k2)
    assert st.thres1_set == s.thres1_set and st.thres2_set == s.thres2_set
    assert st.thres1 == s.thres1 and st.thres2 == s.thres2
    assert (st.key1, st.key2) == (s.key1, s.key2)
    assert st.len2 == s.len2 and st.rand == s.rand


def _compress_case(tk, d, dist, k, N, *, ef=True, seed=0, step=0, rank=0, rand_mode="seeded", levels=0, cfg=1,
                   r_scale=0.0, select="mstopk"):
    g = gradgen.gradient(d, dist, cfg=cfg, rank=rank, step=step)
    r = (gradgen.gradient(d, "G", cfg=cfg + 100, rank=rank, step=step) * np.float32(r_scale)).astype(np.float32)
    ctx = tk.Context(d, k=k, n_iters=N, seed=seed, rand_mode=rand_mode, error_feedback=ef, levels_per_pass=levels,
                     select=select, exact_trial_counts=True)
    ctx.set_step(step)
    gd, rd = _dev(g), _dev(r)
    idx, val = ctx.compress(gd, rd if ef else None)
    torch.cuda.synchronize()
    ref = oracle.compress(g, r if ef else None, k, N, seed=seed, step=step, rank=rank,
                          rand_mode=oracle.RAND_FIRST if rand_mode == "first" else oracle.RAND_SEEDED,
                          error_feedback=ef, selector=select)
    st = ctx.stats()
    if select != "exact":
        _check_stats(st, ref)
    assert np.array_equal(_u32(idx), ref.sel.idx)
    assert np.array_equal(_f32bits(val), ref.sel.val.view(np.uint32))
    if ef:
        assert np.array_equal(_f32bits(rd), ref.residual.view(np.uint32))
    else:
        assert np.array_equal(_f32bits(gd), g.view(np.uint32))  # g never written
    ctx.close()
    _PATHS.add(st.compacted)
    return ref


_PATHS = set()  # which selection paths (compacted / whole-vector) the parity cases exercised


EDGE_D = [1, 2, 3, 4, 5, 127, 128, 129, 511, 4095, 4096, 4097, 8191, 12289, (1 << 20) + 3]


@pytest.mark.parametrize("d", EDGE_D)
def test_compress_edge_sizes(tk, d):
    _compress_case(tk, d, "G", max(1, d // 100), 10, r_scale=0.1)


@pytest.mark.parametrize("dist", gradgen.DISTS)
@pytest.mark.parametrize("d,rho,N", [(1000, 0.01, 10), (65537, 0.001, 10), (300001, 0.001, 20), (100000, 0.01, 5)])
def test_compress_distributions(tk, dist, d, rho, N):
    _compress_case(tk, d, dist, oracle.k_from_density(d, rho), N, seed=3, step=1, r_scale=0.05)


@pytest.mark.parametrize("levels", [1, 2, 3, 4, 5, 8, 9, 10])
@pytest.mark.parametrize("N", [1, 2, 3, 7, 10, 13, 30, 52])
def test_compress_levels_per_pass_invariance(tk, levels, N):
    _compress_case(tk, 50003, "L", 50, N, levels=levels, seed=5)


@pytest.mark.parametrize("k", [1, 2, 999, 10000])
def test_compress_k_extremes(tk, k):
    _compress_case(tk, 10000, "H", k, 10, seed=9)


def test_both_selection_paths_exercised(tk):
    # a typical case takes the compacted path; k = d / a low bracket forces the whole-vector path
    _compress_case(tk, 100_000, "G", 100, 10)
    _compress_case(tk, 100_000, "G", 60_000, 10)
    _compress_case(tk, 100_000, "H", 100_000, 10)
    assert _PATHS == {True, False}


def test_compress_no_error_feedback_and_first_mode(tk):
    _compress_case(tk, 1_000_000, "G", 1000, 10, ef=False)  # BASELINE config 1 (C1)
    _compress_case(tk, 77777, "ties8", 77, 10, rand_mode="first")


@pytest.mark.parametrize("case", ["E1_mstopk_bisection.json", "E2_thres2_unset.json", "E3_k1_zero_guard.json"])
def test_compress_worked_examples(tk, golden, case):
    gd = golden(case)
    x = np.array(gd["x"], np.float32)
    ctx = tk.Context(len(x), k=gd["k"], n_iters=gd["N"], rand_mode="first", error_feedback=False,
                     exact_trial_counts=True)
    idx, val = ctx.compress(_dev(x))
    st = ctx.stats()
    assert [(t[0], t[1], t[3]) for t in st.trials] == [tuple(t) for t in gd["trials"]]
    assert _u32(idx).tolist() == gd["idx"] and val.cpu().tolist() == gd["val"]


def test_error_feedback_multi_step(tk):
    d, k, N = 200003, 200, 10
    ctx = tk.Context(d, k=k, n_iters=N, seed=77, exact_trial_counts=True)
    r_ref = np.zeros(d, np.float32)
    rd = _dev(r_ref)
    for step in range(4):
        g = gradgen.gradient(d, "L", cfg=2, step=step)
        idx, val = ctx.compress(_dev(g), rd)
        ref = oracle.compress(g, r_ref, k, N, seed=77, step=step)
        _check_stats(ctx.stats(), ref)
        assert np.array_equal(_u32(idx), ref.sel.idx)
        assert np.array_equal(_f32bits(val), ref.sel.val.view(np.uint32))
        assert np.array_equal(_f32bits(rd), ref.residual.view(np.uint32))
        r_ref = ref.residual
        ctx.set_step(step + 1)


@pytest.mark.parametrize("P", [1, 2, 3, 8, 17])
@pytest.mark.parametrize("d,rho", [(5000, 0.01), (1 << 20, 0.001), (1_000_003, 0.01), (4097, 0.5)])
def test_decompress_rank_ordered(tk, P, d, rho):
    k = oracle.k_from_density(d, rho)
    gs = [gradgen.gradient(d, "G", cfg=20, rank=p) for p in range(P)]
    res = oracle.flat_step(gs, [np.zeros(d, np.float32)] * P, rho, 10, seed=1)
    ctx = tk.Context(d, k=k, n_iters=10)
    out = ctx.decompress(_dev(res.gathered.view(np.int32)), nchunks=P)
    assert np.array_equal(_f32bits(out), res.out.view(np.uint32))


def test_decompress_overlapping_indices_rank_order(tk):
    # every rank hits the same indices: the accumulation order decides the bits
    d, P, k = 10000, 8, 500
    rng = np.random.default_rng(4)
    idx = np.sort(rng.choice(d, k, replace=False)).astype(np.uint32)
    chunks = [oracle.pack(idx, (rng.standard_normal(k) * 10.0 ** rng.uniform(-8, 8, k)).astype(np.float32))
              for _ in range(P)]
    gathered = oracle.allgather(chunks)
    want = oracle.decompress(gathered, P, k, d)
    ctx = tk.Context(d, k=k, n_iters=10)
    out = ctx.decompress(_dev(gathered.view(np.int32)), nchunks=P)
    assert np.array_equal(_f32bits(out), want.view(np.uint32))


@pytest.mark.parametrize("d,rho,dist", [(1_000_000, 0.001, "G"), (3_000_017, 0.01, "L"), (4096, 1.0, "H")])
def test_flat_step_single_rank(tk, d, rho, dist):
    k = oracle.k_from_density(d, rho)
    ctx = tk.Context(d, rho=rho, n_iters=10, seed=2)
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    for step in range(3):
        g = gradgen.gradient(d, dist, cfg=30, step=step)
        gat = torch.empty(2 * k, dtype=torch.int32, device="cuda")
        out = ctx.step(_dev(g), rd, gathered=gat)
        ref = oracle.flat_step([g], [r], rho, 10, seed=2, step=step)
        assert np.array_equal(_u32(gat), ref.gathered)
        assert np.array_equal(_f32bits(out), ref.out.view(np.uint32))
        assert np.array_equal(_f32bits(rd), ref.per_rank[0].residual.view(np.uint32))
        r = ref.per_rank[0].residual


@pytest.mark.parametrize("d,rho,dist", [(3_000_017, 0.01, "L"), (3_000_017, 0.01, "G"), (1_000_000, 0.001, "G")])
def test_step_p1_writes_every_element_of_out(tk, d, rho, dist):
    """At P = 1 tk_step's k_compress writes the whole aggregate (Alg. 2 l.15-20 with one chunk: +0,
    then the k values) and no decompression runs: every element of out must be written, whatever out
    held before (a NaN pattern here) - on the first call (whole-vector search) and on later calls
    (the fast search).  Guards the round-2 race in which late warps skipped zeroing their slab."""
    k = oracle.k_from_density(d, rho)
    ctx = tk.Context(d, rho=rho, n_iters=10, seed=3)
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    for step in range(8):
        g = gradgen.gradient(d, dist, cfg=32, step=step)
        out = torch.full((d,), float("nan"), device="cuda")
        gat = torch.empty(2 * k, dtype=torch.int32, device="cuda")
        ctx.step(_dev(g), rd, out=out, gathered=gat)
        ref = oracle.flat_step([g], [r], rho, 10, seed=3, step=step)
        assert np.array_equal(_u32(gat), ref.gathered), step
        assert np.array_equal(_f32bits(out), ref.out.view(np.uint32)), step
        assert np.array_equal(_f32bits(rd), ref.per_rank[0].residual.view(np.uint32)), step
        r = ref.per_rank[0].residual
    ctx.close()


def test_step_host_matches_device_path(tk):
    d, rho = 500_000, 0.001
    ctx = tk.Context(d, rho=rho, n_iters=10, seed=8)
    r = np.zeros(d, np.float32)
    for step in range(2):
        g = gradgen.gradient(d, "G", cfg=31, step=step)
        gat = np.empty(2 * ctx.k, np.uint32)
        out = np.empty(d, np.float32)
        ctx.step_host(g, gat, out)
        ref = oracle.flat_step([g], [r], rho, 10, seed=8, step=step)
        assert np.array_equal(gat, ref.gathered)
        assert np.array_equal(out.view(np.uint32), ref.out.view(np.uint32))
        r = ref.per_rank[0].residual


def test_nonfinite_is_reported(tk):
    d = 10000
    g = gradgen.gradient(d, "G", cfg=1)
    g[1234] = np.inf
    ctx = tk.Context(d, k=10, n_iters=10, error_feedback=False)
    ctx.compress(_dev(g))
    assert ctx.stats().nonfinite


def test_rejects_cpu_and_wrong_dtype(tk):
    ctx = tk.Context(1000, k=10, n_iters=10)
    with pytest.raises(ValueError):
        ctx.compress(torch.zeros(1000), torch.zeros(1000))
    with pytest.raises(TypeError):
        ctx.compress(torch.zeros(1000, dtype=torch.float64, device="cuda"), torch.zeros(1000, device="cuda"))


@pytest.mark.parametrize("step", [0, 1])
def test_compress_full_size_c2(tk, step):
    """BASELINE config 2 at full size (d = 25.6M, rho = 1e-3, N = 10, error feedback), in the
    launch configuration bench.py times; every field compared."""
    d, rho, N = 25_600_000, 0.001, 10
    k = oracle.k_from_density(d, rho)
    r = (gradgen.gradient(d, "G", cfg=2, step=99) * np.float32(0.3 * step)).astype(np.float32)
    g = gradgen.gradient(d, "G", cfg=2, step=step)
    ctx = tk.Context(d, rho=rho, n_iters=N, seed=1234, exact_trial_counts=True)
    ctx.set_step(step)
    rd = _dev(r)
    idx, val = ctx.compress(_dev(g), rd)
    ref = oracle.compress(g, r, k, N, seed=1234, step=step)
    _check_stats(ctx.stats(), ref)
    assert np.array_equal(_u32(idx), ref.sel.idx)
    assert np.array_equal(_f32bits(val), ref.sel.val.view(np.uint32))
    assert np.array_equal(_f32bits(rd), ref.residual.view(np.uint32))


def test_compress_full_size_c3(tk):
    """BASELINE config 3's gradient (d = 110M, rho = 1e-3) on one rank, two EF steps."""
    d, rho, N = 110_000_000, 0.001, 10
    k = oracle.k_from_density(d, rho)
    ctx = tk.Context(d, rho=rho, n_iters=N, seed=77, exact_trial_counts=True)
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    for step in range(2):
        g = gradgen.gradient(d, "G", cfg=3, step=step)
        idx, val = ctx.compress(_dev(g), rd)
        ref = oracle.compress(g, r, k, N, seed=77, step=step)
        _check_stats(ctx.stats(), ref)
        assert np.array_equal(_u32(idx), ref.sel.idx)
        assert np.array_equal(_f32bits(val), ref.sel.val.view(np.uint32))
        assert np.array_equal(_f32bits(rd), ref.residual.view(np.uint32))
        r = ref.residual
        ctx.set_step(step + 1)


# ------------------------------------------------------------------ EF-pass compaction (predicted key)
_EF_PATHS = set()
_EF_STEPS = []


def _multi_step(tk, d, dist, k, N, steps, *, scales=None, levels=0, seed=12, cfg=60, exact_counts=True,
                select="mstopk", expect_ef=False):
    """consecutive compressions on one context: from the second call on, the EF pass compacts at a
    key predicted by the previous call; every call is compared with the oracle bit for bit"""
    ctx = tk.Context(d, k=k, n_iters=N, seed=seed, levels_per_pass=levels, exact_trial_counts=exact_counts,
                     select=select)
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    for step in range(steps):
        g = gradgen.gradient(d, dist, cfg=cfg, step=step)
        if scales is not None:
            g = (g * np.float32(scales[step])).astype(np.float32)
        ctx.set_step(step)
        idx, val = ctx.compress(_dev(g), rd)
        ref = oracle.compress(g, r, k, N, seed=seed, step=step, selector=select)
        st = ctx.stats()
        _check_stats(st, ref, exact_counts)
        if expect_ef and step > 0:
            assert st.ef_compacted, step  # the timed path: the EF pass compacted at the predicted key
        assert np.array_equal(_u32(idx), ref.sel.idx), step
        assert np.array_equal(_f32bits(val), ref.sel.val.view(np.uint32)), step
        assert np.array_equal(_f32bits(rd), ref.residual.view(np.uint32)), step
        if step > 0:
            _EF_PATHS.add(st.ef_compacted)
        _EF_STEPS.append(st.ef_compacted)
        r = ref.residual
    ctx.close()
    return st


@pytest.mark.parametrize("dist", ["G", "L", "H", "ties8", "spike"])
@pytest.mark.parametrize("d,rho,N", [(300_001, 0.001, 10), (1_000_003, 0.01, 20), (65537, 0.001, 5)])
def test_ef_compaction_multi_step(tk, dist, d, rho, N):
    _multi_step(tk, d, dist, oracle.k_from_density(d, rho), N, 5)


@pytest.mark.parametrize("levels", [1, 3, 8])
def test_ef_compaction_levels(tk, levels):
    _multi_step(tk, 200_003, "G", 200, 13, 4, levels=levels)


def test_ef_compaction_restart_on_shift(tk):
    # the scale jumps: the predicted key is far too low (entries overflow) or too high (a trial
    # falls below it); both calls must restart the search and stay bit-exact
    _multi_step(tk, 400_003, "G", 400, 10, 6, scales=[1, 1, 1000, 1e-3, 1e-3, 1])


def test_ef_compaction_paths_exercised(tk):
    _multi_step(tk, 100_003, "G", 100, 10, 3)
    _multi_step(tk, 100_003, "G", 100, 10, 4, scales=[1, 1, 1e4, 1])
    assert _EF_PATHS == {True, False}


# ------------------------------------------------------------------ the bench's timed path at full size
@pytest.mark.parametrize("dist", ["G", "L"])
def test_full_size_c2_multi_step_ef_compacted(tk, dist):
    """BASELINE config 2 at full size (d = 25.6M, rho = 1e-3, N = 10) on ONE context for 6 steps with
    the residual carried - the regime bench.py times: every trial counted exactly (exact_trial_counts)
    and every step bit-exact; with N(0,1) gradients the EF pass compacts at the predicted key on every
    step >= 1 (asserted), with the layered profile on most of them (a failed prediction restarts)."""
    _EF_STEPS.clear()
    _multi_step(tk, 25_600_000, dist, 25_600, 10, 6, cfg=2, expect_ef=(dist == "G"))
    assert sum(_EF_STEPS[1:]) >= (5 if dist == "G" else 3), _EF_STEPS


def test_full_size_c2_default_mode(tk):
    """The same in the bench's default mode (no extra count pass): identical selection, residual and
    control block; the trials whose count was skipped are flagged and exceed k in the oracle."""
    st = _multi_step(tk, 25_600_000, "G", 25_600, 10, 4, cfg=3, exact_counts=False, expect_ef=True)
    assert st.ef_compacted


@pytest.mark.parametrize("regime", ["G_ef", "U_noef"])
def test_default_mode_matches_exact_count_mode_c2(tk, regime):
    """C2 size, fresh inputs per step on one context: the default mode and the exact-count mode give
    bit-identical selections, residuals and control blocks, except that the default mode skips the
    counts of trials below the EF-pass key - whose exact counts (from the exact-count mode, itself
    pinned to the oracle above) exceed k, as the flag claims.  G_ef: the bench regime (N(0,1), EF);
    U_noef: U(-1,1) without EF, a light tail that puts the first trials (near a-bar + (u - a-bar)/2)
    far below the k-th magnitude, so counts are skipped on every step after the first."""
    d, k, steps = 25_600_000, 25_600, 5
    ef = regime == "G_ef"
    gen = torch.Generator(device="cuda")
    gen.manual_seed(9)
    gs = [torch.randn(d, generator=gen, device="cuda") if ef else torch.rand(d, generator=gen, device="cuda") * 2 - 1
          for _ in range(steps)]
    runs = {}
    for exact in (False, True):
        ctx = tk.Context(d, k=k, n_iters=10, seed=3, exact_trial_counts=exact, error_feedback=ef)
        r = torch.zeros(d, device="cuda")
        log = []
        for step in range(steps):
            ctx.set_step(step)
            idx, val = ctx.compress(gs[step], r if ef else None)
            log.append((_u32(idx).copy(), _f32bits(val).copy(), _f32bits(r).copy(), ctx.stats()))
        runs[exact] = log
        ctx.close()
    flagged = 0
    for (i0, v0, r0, s0), (i1, v1, r1, s1) in zip(runs[False], runs[True]):
        assert np.array_equal(i0, i1) and np.array_equal(v0, v1) and np.array_equal(r0, r1)
        assert s1.nnz_not_counted == 0
        assert (s0.k1, s0.k2, s0.key1, s0.key2, s0.len2, s0.rand, s0.mean) == (s1.k1, s1.k2, s1.key1, s1.key2,
                                                                               s1.len2, s1.rand, s1.mean)
        for it, (a, b) in enumerate(zip(s0.trials, s1.trials)):
            assert a[:3] == b[:3]
            if s0.nnz_not_counted >> it & 1:
                assert a[3] == NNZ_NOT_COUNTED and b[3] > k
                flagged += 1
            else:
                assert a[3] == b[3]
    if not ef:
        assert flagged > 0  # the light-tailed regime does skip counts


# ------------------------------------------------------------------ prose search
@pytest.mark.parametrize("d", [1, 5, 129, 4097, 65537, (1 << 20) + 3])
def test_prose_edge_sizes(tk, d):
    _compress_case(tk, d, "G", max(1, d // 100), 10, r_scale=0.1, select="prose")


@pytest.mark.parametrize("dist", gradgen.DISTS)
@pytest.mark.parametrize("d,rho,N", [(1000, 0.01, 10), (300001, 0.001, 20), (100000, 0.01, 5)])
def test_prose_distributions(tk, dist, d, rho, N):
    _compress_case(tk, d, dist, oracle.k_from_density(d, rho), N, seed=3, step=1, r_scale=0.05, select="prose")


@pytest.mark.parametrize("levels", [1, 2, 4, 10])
@pytest.mark.parametrize("N", [1, 3, 10, 30, 52])
def test_prose_levels_per_pass_invariance(tk, levels, N):
    _compress_case(tk, 50003, "L", 50, N, levels=levels, seed=5, select="prose")


@pytest.mark.parametrize("k", [1, 2, 9999, 10000])
def test_prose_k_extremes(tk, k):
    _compress_case(tk, 10000, "H", k, 10, seed=9, select="prose")


def test_prose_no_ef_and_first_mode(tk):
    _compress_case(tk, 1_000_000, "G", 1000, 10, ef=False, select="prose")
    _compress_case(tk, 77777, "ties8", 77, 10, rand_mode="first", select="prose")
    _compress_case(tk, 4096, "zero", 40, 10, select="prose")


def test_prose_hand_worked_examples(tk):
    # the trial sequences of tests/test_oracle_prose.py, worked by hand from P:148
    x = np.array([1, -2, 3, 4, -5, 6, 7, -8], np.float32)
    ctx = tk.Context(8, k=2, n_iters=4, rand_mode="first", error_feedback=False, select="prose",
                     exact_trial_counts=True)
    idx, val = ctx.compress(_dev(x))
    st = ctx.stats()
    assert [t[1] for t in st.trials] == [4.5, 9.0, 6.75, 5.625] and [t[3] for t in st.trials] == [4, 0, 2, 3]
    assert _u32(idx).tolist() == [6, 7] and val.cpu().tolist() == [7.0, -8.0]
    x = np.array([100, 1, -1, 1], np.float32)
    ctx = tk.Context(4, k=3, n_iters=6, rand_mode="first", error_feedback=False, select="prose",
                     exact_trial_counts=True)
    idx, _ = ctx.compress(_dev(x))
    assert [t[1] for t in ctx.stats().trials] == [25.75, 12.875, 6.4375, 3.21875, 1.609375, 0.8046875]
    assert _u32(idx).tolist() == [0, 1, 2]


@pytest.mark.parametrize("dist", ["G", "L", "H"])
def test_prose_multi_step_ef_compaction(tk, dist):
    _multi_step(tk, 300_001, dist, 300, 10, 5, select="prose", cfg=61)


def test_prose_restart_on_shift(tk):
    _multi_step(tk, 400_003, "G", 400, 10, 6, scales=[1, 1, 1000, 1e-3, 1e-3, 1], select="prose", cfg=62)


def test_prose_full_size_c2(tk):
    """F3's bench configuration: C2 at full size, 4 steps on one context, EF-pass compaction."""
    _multi_step(tk, 25_600_000, "G", 25_600, 10, 4, select="prose", cfg=63, expect_ef=True)


# ------------------------------------------------------------------ all-zero input (reading Q34)
@pytest.mark.parametrize("rand_mode", ["first", "seeded"])
def test_all_zero_input_worked_example(tk, golden, rand_mode):
    gd = golden("E9_all_zero.json")
    x = np.array(gd["x"], np.float32)
    ctx = tk.Context(len(x), k=gd["k"], n_iters=gd["N"], rand_mode=rand_mode, error_feedback=False,
                     exact_trial_counts=True)
    idx, val = ctx.compress(_dev(x))
    st = ctx.stats()
    assert [(t[0], t[1], t[3]) for t in st.trials] == [tuple(t) for t in gd["trials"]]
    assert (st.k1, st.k2, st.len2, st.thres1_set, st.thres2_set) == (gd["k1"], gd["k2"], gd["len2"], False, False)
    ref = oracle.mstopk(x, gd["k"], gd["N"], rand_mode=oracle.RAND_FIRST if rand_mode == "first" else 0)
    assert st.rand == ref.rand and _u32(idx).tolist() == ref.idx.tolist()
    assert _f32bits(val).tolist() == ref.val.view(np.uint32).tolist()
    if rand_mode == "first":
        assert _u32(idx).tolist() == gd["first_idx"] and _f32bits(val).tolist() == gd["first_val_bits"]


@pytest.mark.parametrize("select", ["mstopk", "prose", "exact"])
def test_all_zero_input_large(tk, select):
    if select == "exact":
        ctx = tk.Context(100_000, k=100, n_iters=10, select="exact")
        idx, _ = ctx.compress(torch.zeros(100_000, device="cuda"), torch.zeros(100_000, device="cuda"))
        assert _u32(idx).tolist() == list(range(100))  # Eq. 2 with every |x| tied: the lowest indices
        return
    _compress_case(tk, 100_000, "zero", 100, 10, select=select)
