"""Bucketed multi-tensor step (tensor fusion; DESIGN reading Q32): a bucket of
layers is the concatenation of their gradients in list order and one tk_step runs on it.

CPU: the layout (contiguous offsets, no padding, the degenerate layers).  GPU: the layer-shaped
aggregates and residuals of ``Bucket.step`` / ``Bucket.step_sgd`` bit for bit against the oracle's
flat_step over ``np.concatenate`` of the same layer gradients, over several steps (EF carries)."""
import numpy as np
import pytest

import gradgen
import oracle

torch = pytest.importorskip("torch")

# a ResNet-ish mix: conv kernels, a BN pair, an empty layer, a ragged FC (d = 1 048 627)
SHAPES = [(64, 3, 7, 7), (64,), (64,), (0,), (256, 64, 3, 3), (7, 11, 13), (1000, 885), (1,)]


def _tk():
    import paper_2010_10458_b200 as tk
    return tk


def test_layout_is_contiguous_in_list_order():
    tk = _tk()
    lay = tk.bucket_layout(SHAPES)
    off = 0
    for (o, n, s), shape in zip(lay, SHAPES):
        assert o == off and s == tuple(shape) and n == int(np.prod(shape))
        off += n
    assert off == 9408 + 64 + 64 + 0 + 147456 + 1001 + 885000 + 1
    # an int is a 1-D layer
    assert tk.bucket_layout([5, (2, 3)]) == [(0, 5, (5,)), (5, 6, (2, 3))]


def test_layout_rejects_degenerate_buckets():
    tk = _tk()
    with pytest.raises(ValueError):
        tk.bucket_layout([])
    with pytest.raises(ValueError):
        tk.bucket_layout([(0,), (3, 0)])
    with pytest.raises(ValueError):
        tk.bucket_layout([(2, -1)])
    with pytest.raises(ValueError):
        tk.bucket_layout([(1 << 31,), (1 << 31,)])


def _layers(step, cfg=90):
    return [gradgen.gradient(int(np.prod(s)), "L" if i % 2 else "G", cfg=cfg + i, step=step).reshape(s)
            for i, s in enumerate(SHAPES)]


def _bits(t):
    return t.detach().cpu().numpy().astype(np.float32).view(np.uint32).ravel()


@pytest.mark.gpu
@pytest.mark.parametrize("select,wire", [("mstopk", "f32"), ("exact", "f32"), ("mstopk", "f16")])
def test_bucket_step_matches_oracle_on_the_concatenation(select, wire):
    if not torch.cuda.is_available():
        pytest.fail("GPU tests selected but no CUDA device is visible")
    tk = _tk()
    rho = 0.002
    b = tk.Bucket(SHAPES, rho=rho, seed=11, select=select, wire=wire)
    d = b.d
    r = np.zeros(d, np.float32)
    for step in range(3):
        layers = _layers(step)
        for view, g in zip(b.grads, layers):
            view.copy_(torch.from_numpy(g))
        outs = b.step()
        flat = np.concatenate([g.ravel() for g in layers])
        ref = oracle.flat_step([flat], [r], rho, 10, seed=11, step=step, selector=select, wire=wire)
        assert [tuple(o.shape) for o in outs] == [tuple(s) for s in SHAPES]
        for (o, n, _), view in zip(b.layout, outs):
            assert np.array_equal(_bits(view), ref.out[o:o + n].view(np.uint32)), (step, o)
        assert np.array_equal(_bits(b.residual), ref.per_rank[0].residual.view(np.uint32)), step
        r = ref.per_rank[0].residual
    b.close()


@pytest.mark.gpu
def test_bucket_step_sgd_updates_the_layer_views():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests selected but no CUDA device is visible")
    tk = _tk()
    rho, lr = 0.001, 0.05
    b = tk.Bucket(SHAPES, rho=rho, seed=3)
    w = gradgen.gradient(b.d, "G", cfg=99)
    wd = torch.from_numpy(w.copy()).cuda()
    params = b.views(wd)
    r = np.zeros(b.d, np.float32)
    for step in range(2):
        layers = _layers(step, cfg=120)
        for view, g in zip(b.grads, layers):
            view.copy_(torch.from_numpy(g))
        b.step_sgd(wd, lr)
        ref = oracle.flat_step([np.concatenate([g.ravel() for g in layers])], [r], rho, 10, seed=3, step=step)
        w = oracle.sgd_update(w, ref.out, lr)
        r = ref.per_rank[0].residual
        for (o, n, _), p in zip(b.layout, params):
            assert np.array_equal(_bits(p), w[o:o + n].view(np.uint32)), (step, o)
    with pytest.raises(ValueError):
        b.views(torch.zeros(b.d + 1, device="cuda"))
    b.close()


def test_bucket_has_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("checks the CPU-only failure mode")
    tk = _tk()
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        tk.Bucket(SHAPES)
