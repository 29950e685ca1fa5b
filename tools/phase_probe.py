"""Per-phase device time of k_compress in the bench regime (fresh N(0,1) gradients, EF from r=0),
with the SM clock sampled by nvidia-smi during the measured calls (phase times of the latency-bound
tail scale with it)."""
import os
import subprocess
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("TK_PKG_PATH"):  # experiments: another build of the package (e.g. round 1's)
    sys.path.insert(0, os.environ["TK_PKG_PATH"])
import torch
import paper_2010_10458_b200 as tk

d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
select = sys.argv[2] if len(sys.argv) > 2 else "mstopk"
steps = 400
ctx = tk.Context(d, rho=0.001, n_iters=10, seed=1, select=select)
gen = torch.Generator(device="cuda")
gen.manual_seed(5)
gs = [torch.randn(d, generator=gen, device="cuda") for _ in range(8)]
r = torch.zeros(d, device="cuda")
out = torch.empty(d, device="cuda")
smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "20"],
                       stdout=subprocess.PIPE, text=True)
acc, n = None, 0
t0 = time.time()
for s in range(steps):
    ctx.step(gs[s % 8], r, out)
    if s >= 20 and s % 4 == 0:
        st = ctx.stats()
        acc = st.phase_us if acc is None else [a + b for a, b in zip(acc, st.phase_us)]
        n += 1
torch.cuda.synchronize()
smi.terminate()
clk = [float(x) for x in smi.communicate()[0].split() if x.strip().replace(".", "").isdigit()]
names = ["ef", "root"] + [f"pass{i}" for i in range(len(acc) - 5)] + ["replay", "prefix", "select"]
if st.ef_compacted and select != "exact":  # fast search: pass, counts, replay per pass, then verify
    names = ["ef", "root"] + sum([[f"pass{i}", f"counts{i}", f"replay{i}"] for i in range((len(acc) - 4) // 3)], []) + ["verify", "prefix", "select"]
if select == "exact":
    names = ["ef", "root"] + [f"pass{i}" for i in range(len(acc) - 4)] + ["prefix", "select"]
print(select, f"d={d}", "phases (us):", {names[i] if i < len(names) else i: round(v / n, 1) for i, v in enumerate(acc)},
      "total", round(sum(acc) / n, 1), "compacted", st.compacted, "n_compacted", st.n_compacted,
      "frac", round(st.n_compacted / d, 4), "sm_mhz", (min(clk), sorted(clk)[len(clk) // 2], max(clk)) if clk else None)
