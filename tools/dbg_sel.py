"""debug: C2-size two-step compression vs the oracle; report how the selection differs"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gradgen, oracle
import paper_2010_10458_b200 as tk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
k = d // 1000
ctx = tk.Context(d, k=k, n_iters=10, seed=12, exact_trial_counts=True)
r = np.zeros(d, np.float32); rd = torch.from_numpy(r.copy()).cuda()
for step in range(int(os.environ.get("STEPS", "3"))):
    g = gradgen.gradient(d, "G", cfg=int(os.environ.get("CFG", "60")), step=step)
    ctx.set_step(step)
    idx, val = ctx.compress(torch.from_numpy(g).cuda(), rd)
    st = ctx.stats()
    ref = oracle.compress(g, r, k, 10, seed=12, step=step)
    gi = idx.cpu().numpy().view(np.uint32).astype(np.int64)
    ri = ref.sel.idx.astype(np.int64)
    print("step", step, "ef", st.ef_compacted, "n_comp", st.n_compacted, "k1", st.k1, ref.sel.k1, "k2", st.k2, ref.sel.k2,
          "rand", st.rand, ref.sel.rand, "len2", st.len2, ref.sel.len2)
    bad = np.nonzero(gi != ri)[0]
    print("  mismatches", len(bad), "first", bad[:10].tolist(), "gpu", gi[bad[:5]].tolist(), "ref", ri[bad[:5]].tolist(),
          "sorted", bool(np.all(np.diff(gi) > 0)), "inrange", bool(gi.max() < d), "set_diff", len(set(gi) - set(ri)), len(set(ri) - set(gi)))
    rr = rd.cpu().numpy().view(np.uint32); print("  resid mism", int((rr != ref.residual.view(np.uint32)).sum()))
    r = ref.residual
