"""BASELINE config 1 (d = 1M, rho = 1e-3, N = 10, EF off, P = 1): tk_compress latency per call on fresh
N(0,1) gradients (CUDA events over 200 back-to-back calls) and the k_compress phase split."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("TK_PKG_PATH"):
    sys.path.insert(0, os.environ["TK_PKG_PATH"])
import torch
import paper_2010_10458_b200 as tk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
stream = torch.cuda.Stream()
ctx = tk.Context(d, rho=0.001, n_iters=10, seed=1, error_feedback=False, stream=stream)
torch.cuda.set_stream(stream)
gen = torch.Generator(device="cuda"); gen.manual_seed(3)
gs = [torch.randn(d, generator=gen, device="cuda") for _ in range(32)]
idx = torch.empty(ctx.k, dtype=torch.int32, device="cuda"); val = torch.empty(ctx.k, device="cuda")
for i in range(50):
    ctx.compress(gs[i % 32], None, idx, val)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 400
e0.record()
for i in range(n):
    ctx.compress(gs[i % 32], None, idx, val)
e1.record(); torch.cuda.synchronize()
t_stream = e0.elapsed_time(e1) * 1e3 / n
# the same calls captured in a CUDA graph (no host launch cost between kernels)
s = ctx.stream
g = torch.cuda.CUDAGraph()
reps = 20
with torch.cuda.graph(g, stream=s):
    for i in range(reps):
        ctx.compress(gs[i % 32], None, idx, val)
g.replay(); torch.cuda.synchronize()
e0.record(s)
for _ in range(n // reps):
    g.replay()
e1.record(s); torch.cuda.synchronize()
t_graph = e0.elapsed_time(e1) * 1e3 / (n // reps * reps)
st = ctx.stats()
print(f"C1 d={d}: {t_stream:.2f} us per tk_compress launched from Python, {t_graph:.2f} us per call in a CUDA graph; phases",
      [round(x, 1) for x in st.phase_us], "sum", round(sum(st.phase_us), 1), "ef_compacted", st.ef_compacted)
