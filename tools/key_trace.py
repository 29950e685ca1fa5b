"""Per-step trace of the search's key2 (the final bracket's lower key), the EF-pass entries kept and
whether the EF-pass path was taken, in the bench regime (fresh N(0,1) gradient per step, EF)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_10458_b200 as tk

d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
ctx = tk.Context(d, rho=0.001, n_iters=10, seed=1)
gen = torch.Generator(device="cuda")
gen.manual_seed(5)
g = torch.empty(d, device="cuda")
r = torch.zeros(d, device="cuda")
out = torch.empty(d, device="cuda")
prev = None
for s in range(steps):
    g.normal_(generator=gen)
    ctx.step(g, r, out)
    st = ctx.stats()
    if s < 10 or s % 20 == 0 or not st.ef_compacted:
        dk = None if prev is None else st.key2 - prev
        print(f"step {s}: key2 {st.key2:#x} dkey2 {dk} entries/k {st.n_compacted / ctx.k:.2f} ef {st.ef_compacted}")
    prev = st.key2
