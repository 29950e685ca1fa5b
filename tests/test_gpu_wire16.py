"""GPU parity of FP16 wire values (TK_WIRE_F16; Fig. 7 ran FP16; reading Q31):
the binary16 values sent, the packed [idx | binary16] chunks, the residual that keeps the rounding
error, and the rank-ordered aggregate, bit for bit against the oracle (wire="f16")."""
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


@pytest.mark.parametrize("d,k,dist,select", [(1000, 10, "G", "mstopk"), (100_003, 101, "H", "mstopk"),
                                             (1_000_000, 1000, "L", "mstopk"), (300_007, 300, "G", "exact"),
                                             (4097, 4097, "G", "mstopk"), (5, 3, "spike", "mstopk")])
def test_compress_fp16_wire(tk, d, k, dist, select):
    ctx = tk.Context(d, k=k, seed=6, wire="f16", select=select)
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    for step in range(3):
        g = (gradgen.gradient(d, dist, cfg=80, step=step) * np.float32(30000.0 if dist == "spike" else 1.0))
        g = g.astype(np.float32)
        ctx.set_step(step)
        idx, val = ctx.compress(_dev(g), rd)
        ref = oracle.compress(g, r, k, 10, seed=6, step=step, selector=select, wire="f16")
        assert np.array_equal(_bits(idx), ref.sel.idx)
        assert np.array_equal(_bits(val), ref.sent.view(np.uint32))
        assert np.array_equal(_bits(rd), ref.residual.view(np.uint32))
        gat = ctx.sparse_allgather(idx, val)
        assert np.array_equal(_bits(gat), oracle.pack(ref.sel.idx, ref.sent, "f16"))
        out = ctx.decompress(gat, nchunks=1)
        assert np.array_equal(_bits(out), oracle.decompress(oracle.pack(ref.sel.idx, ref.sent, "f16"), 1, k, d,
                                                             "f16").view(np.uint32))
        r = ref.residual


@pytest.mark.parametrize("d,rho", [(25_600_000, 0.001), (3_000_017, 0.01)])
def test_step_fp16_wire(tk, d, rho):
    ctx = tk.Context(d, rho=rho, seed=7, wire="f16")
    r = np.zeros(d, np.float32)
    rd = _dev(r)
    for step in range(2):
        g = gradgen.gradient(d, "G", cfg=81, step=step)
        gat = torch.empty(ctx.chunk_words, dtype=torch.int32, device="cuda")
        out = ctx.step(_dev(g), rd, gathered=gat)
        ref = oracle.flat_step([g], [r], rho, 10, seed=7, step=step, wire="f16")
        assert np.array_equal(_bits(gat), ref.gathered)
        assert np.array_equal(_bits(out), ref.out.view(np.uint32))
        assert np.array_equal(_bits(rd), ref.per_rank[0].residual.view(np.uint32))
        r = ref.per_rank[0].residual


def test_step_host_fp16_wire(tk):
    d, rho = 500_000, 0.001
    ctx = tk.Context(d, rho=rho, seed=8, wire="f16")
    r = np.zeros(d, np.float32)
    for step in range(2):
        g = gradgen.gradient(d, "G", cfg=82, step=step)
        gat = np.empty(ctx.chunk_words, np.uint32)
        out = np.empty(d, np.float32)
        ctx.step_host(g, gat, out)
        ref = oracle.flat_step([g], [r], rho, 10, seed=8, step=step, wire="f16")
        assert np.array_equal(gat, ref.gathered)
        assert np.array_equal(out.view(np.uint32), ref.out.view(np.uint32))
        r = ref.per_rank[0].residual
