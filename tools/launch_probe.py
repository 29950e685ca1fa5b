"""Where the k_compress event interval goes at C2 (EF, fresh N(0,1) gradients, residual carried):
per-call device time of compress-only loops (CUDA events at the loop ends only, so consecutive
launches overlap through programmatic dependent launch), the same loop with an event pair around
every launch (the bench's per-stage method), whole steps, and CTA 0's phase sum."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_10458_b200 as tk

d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
ef = os.environ.get("EF", "1") == "1"
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ctx = tk.Context(d, rho=0.001, n_iters=10, seed=1, error_feedback=ef, stream=stream)
gen = torch.Generator(device="cuda"); gen.manual_seed(5)
gs = [torch.randn(d, generator=gen, device="cuda") for _ in range(8)]
r = torch.zeros(d, device="cuda") if ef else None
out = torch.empty(d, device="cuda")
idx = torch.empty(ctx.k, dtype=torch.int32, device="cuda"); val = torch.empty(ctx.k, device="cuda")
for i in range(60):
    ctx.compress(gs[i % 8], r, idx, val)
torch.cuda.synchronize()
n = 200
E = lambda: torch.cuda.Event(enable_timing=True)
e0, e1 = E(), E()
e0.record(stream)
for i in range(n):
    ctx.compress(gs[i % 8], r, idx, val)
e1.record(stream); torch.cuda.synchronize()
t_loop = e0.elapsed_time(e1) * 1e3 / n
ev = [(E(), E()) for _ in range(n)]
for i in range(n):
    ev[i][0].record(stream)
    ctx.compress(gs[i % 8], r, idx, val)
    ev[i][1].record(stream)
torch.cuda.synchronize()
t_ev = sum(a.elapsed_time(b) for a, b in ev) * 1e3 / n
ph = ctx.stats().phase_us
e0.record(stream)
for i in range(n):
    ctx.step(gs[i % 8], r, out)
e1.record(stream); torch.cuda.synchronize()
t_step = e0.elapsed_time(e1) * 1e3 / n
# one launch alone (stream idle before it): the launch latency is fully exposed
solo = []
for i in range(20):
    torch.cuda.synchronize()
    e0.record(stream)
    ctx.compress(gs[i % 8], r, idx, val)
    e1.record(stream); torch.cuda.synchronize()
    solo.append(e0.elapsed_time(e1) * 1e3)
print(f"d={d} EF={ef}: compress loop {t_loop:.1f} us/call; event pair per call {t_ev:.1f} us; solo {sorted(solo)[10]:.1f} us; "
      f"step loop {t_step:.1f} us; CTA0 phase sum {sum(ph):.1f} us {[round(x, 1) for x in ph]}")
