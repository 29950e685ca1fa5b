"""Per-step path and phases of k_compress on a given distribution (bench regime: fresh gradients,
residual carried): which search path ran (EF-pass entries or whole-vector restart), entries kept."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gradgen
import paper_2010_10458_b200 as tk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
dist = sys.argv[2] if len(sys.argv) > 2 else "L"
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 12
ctx = tk.Context(d, rho=0.001, n_iters=10, seed=1)
gs = [torch.from_numpy(gradgen.gradient(d, dist, cfg=2, step=s)).cuda() for s in range(4)]
r = torch.zeros(d, device="cuda"); out = torch.empty(d, device="cuda")
for s in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ctx.step(gs[s % 4], r, out); e1.record(); torch.cuda.synchronize()
    st = ctx.stats()
    print(f"step {s:2d} {e0.elapsed_time(e1)*1e3:7.1f} us  ef_compacted={int(st.ef_compacted)} compacted={int(st.compacted)} "
          f"n_compacted={st.n_compacted:8d} key2={st.key2:#x} phases={[round(x,1) for x in st.phase_us]}")
