"""A short bench-regime run for ncu captures: C2 steps with fresh N(0,1) gradients and EF."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("TK_PKG_PATH"):
    sys.path.insert(0, os.environ["TK_PKG_PATH"])
import torch
import paper_2010_10458_b200 as tk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 24
ctx = tk.Context(d, rho=0.001, n_iters=10, seed=1)
gen = torch.Generator(device="cuda"); gen.manual_seed(5)
gs = [torch.randn(d, generator=gen, device="cuda") for _ in range(4)]
r = torch.zeros(d, device="cuda"); out = torch.empty(d, device="cuda")
for s in range(steps):
    ctx.step(gs[s % 4], r, out)
torch.cuda.synchronize()
print("ok", ctx.stats().ef_compacted)
