"""GPU parity of the exact top-k selector (TK_SELECT_EXACT; Eq. 2, ties ->
lower index, Q6) against the CPU oracle (oracle.compress(selector="exact") = a full stable sort):
indices, values, residuals bit-exact; the k-th order statistic and the counts around it exact."""
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


def _bits(t):
    return t.cpu().numpy().view(np.uint32)


_PATHS = set()


def _check(ctx, idx, val, rd, ref, ef):
    st = ctx.stats()
    e = ref.sel
    assert (st.key2, st.key1) == (e.kth_bits, e.kth_bits + 1)
    assert (st.k1, st.k2) == (e.k1, e.k2)
    assert np.array_equal(_bits(idx), e.idx)
    assert np.array_equal(_bits(val), e.val.view(np.uint32))
    if ef:
        assert np.array_equal(_bits(rd), ref.residual.view(np.uint32))
    _PATHS.add(st.compacted)


def _case(tk, d, dist, k, *, ef=True, steps=1, cfg=1, r_scale=0.0):
    ctx = tk.Context(d, k=k, select="exact", error_feedback=ef)
    r = (gradgen.gradient(d, "G", cfg=cfg + 100) * np.float32(r_scale)).astype(np.float32)
    rd = _dev(r)
    for step in range(steps):
        g = gradgen.gradient(d, dist, cfg=cfg, step=step)
        gd = _dev(g)
        idx, val = ctx.compress(gd, rd if ef else None)
        ref = oracle.compress(g, r if ef else None, k, 10, error_feedback=ef, selector="exact")
        _check(ctx, idx, val, rd, ref, ef)
        if ef:
            r = ref.residual
        else:
            assert np.array_equal(_bits(gd), g.view(np.uint32))
    ctx.close()


EDGE_D = [1, 2, 3, 4, 5, 127, 128, 129, 511, 4095, 4096, 4097, 12289, (1 << 20) + 3]


@pytest.mark.parametrize("d", EDGE_D)
def test_exact_edge_sizes(tk, d):
    _case(tk, d, "G", max(1, d // 100), r_scale=0.1)


@pytest.mark.parametrize("d", [1, 5, 4097, 100_003])
@pytest.mark.parametrize("which", ["one", "all"])
def test_exact_k_extremes(tk, d, which):
    _case(tk, d, "H", 1 if which == "one" else d)


@pytest.mark.parametrize("dist", gradgen.DISTS)
@pytest.mark.parametrize("d,rho", [(1000, 0.01), (65537, 0.001), (300001, 0.001), (1_000_003, 0.01)])
def test_exact_distributions(tk, dist, d, rho):
    _case(tk, d, dist, oracle.k_from_density(d, rho), cfg=3, r_scale=0.05)


@pytest.mark.parametrize("dist", ["G", "L", "H"])
def test_exact_error_feedback_multi_step(tk, dist):
    """the k-th statistic of the previous step seeds the next one's first pass (results independent)"""
    _case(tk, 400_009, dist, 400, steps=4, cfg=5)


def test_exact_no_error_feedback(tk):
    _case(tk, 1_000_000, "G", 1000, ef=False)  # C1 shape


def test_exact_both_paths(tk):
    # compacted (typical) and whole-vector (large k / ties everywhere) narrowing
    _case(tk, 100_000, "G", 100)
    _case(tk, 100_000, "G", 60_000)
    _case(tk, 100_000, "zero", 77)
    _case(tk, 100_000, "ties8", 5000)
    assert _PATHS == {True, False}


@pytest.mark.parametrize("d,rho,dist", [(1_000_000, 0.001, "G"), (3_000_017, 0.01, "L")])
def test_exact_flat_step_single_rank(tk, d, rho, dist):
    k = oracle.k_from_density(d, rho)
    ctx = tk.Context(d, rho=rho, select="exact")
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    for step in range(3):
        g = gradgen.gradient(d, dist, cfg=30, step=step)
        gat = torch.empty(2 * k, dtype=torch.int32, device="cuda")
        out = ctx.step(_dev(g), rd, gathered=gat)
        ref = oracle.flat_step([g], [r], rho, 10, step=step, selector="exact")
        assert np.array_equal(_bits(gat), ref.gathered)
        assert np.array_equal(_bits(out), ref.out.view(np.uint32))
        assert np.array_equal(_bits(rd), ref.per_rank[0].residual.view(np.uint32))
        r = ref.per_rank[0].residual


def test_exact_full_size_c2(tk):
    """BASELINE config 2's shape (d = 25.6M, rho = 1e-3, error feedback), two steps."""
    _case(tk, 25_600_000, "G", 25_600, steps=2, cfg=2)


def test_exact_restart_on_shift(tk):
    """scale jumps make the predicted compaction key useless (overflow / above T): still exact"""
    d, k = 300_007, 300
    ctx = tk.Context(d, k=k, select="exact")
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    used = set()
    for step, sc in enumerate([1, 1, 1000, 1e-3, 1e-3, 1]):
        g = (gradgen.gradient(d, "G", cfg=9, step=step) * np.float32(sc)).astype(np.float32)
        idx, val = ctx.compress(_dev(g), rd)
        ref = oracle.compress(g, r, k, 10, selector="exact")
        _check(ctx, idx, val, rd, ref, True)
        if step:
            used.add(ctx.stats().ef_compacted)
        r = ref.residual
    assert used == {True, False}
