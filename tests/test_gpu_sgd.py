"""GPU parity of the fused SGD update (tk_step_sgd; Eq. 1): the parameters
after w -= lr * aggregate, bit for bit against oracle.sgd_update of the oracle's aggregate."""
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


@pytest.mark.parametrize("d,rho,select,keep_out", [(1_000_003, 0.001, "mstopk", True), (4097, 0.01, "mstopk", False),
                                                   (3_000_017, 0.01, "exact", False), (5, 0.5, "mstopk", True)])
def test_step_sgd_single_rank(tk, d, rho, select, keep_out):
    lr = 0.0625 if select == "mstopk" else 0.013
    ctx = tk.Context(d, rho=rho, seed=4, select=select)
    r = np.zeros(d, np.float32)
    w = gradgen.gradient(d, "G", cfg=70)
    rd, wd = _dev(r), _dev(w)
    for step in range(3):
        g = gradgen.gradient(d, "L", cfg=71, step=step)
        out = torch.empty(d, dtype=torch.float32, device="cuda") if keep_out else None
        ctx.step_sgd(_dev(g), rd, wd, lr, out=out)
        ref = oracle.flat_step([g], [r], rho, 10, seed=4, step=step, selector=select)
        w = oracle.sgd_update(w, ref.out, lr)
        assert np.array_equal(_bits(wd), w.view(np.uint32)), step
        if keep_out:
            assert np.array_equal(_bits(out), ref.out.view(np.uint32))
        assert np.array_equal(_bits(rd), ref.per_rank[0].residual.view(np.uint32))
        r = ref.per_rank[0].residual


def test_step_sgd_rejects_bad_arguments(tk):
    ctx = tk.Context(1000, k=10)
    g = torch.zeros(1000, device="cuda")
    r = torch.zeros(1000, device="cuda")
    with pytest.raises(tk.TkError):
        ctx.step_sgd(g, r, torch.zeros(1000, device="cuda"), float("nan"))
    with pytest.raises(tk.TkError):
        ctx.step_sgd(g, r, g, 0.1)  # w aliases g
