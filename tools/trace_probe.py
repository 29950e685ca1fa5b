"""Per-CTA phase timeline of k_compress (TK_PHASE_TRACE variant build): for each stamp, the spread over
CTAs relative to the earliest CTA start, and each barrier's arrival spread (who is late)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2010_10458_b200 as tk
d = int(sys.argv[1]) if len(sys.argv) > 1 else 25_600_000
ef = os.environ.get("EF", "1") == "1"
ctx = tk.Context(d, rho=0.001, n_iters=10, seed=1, error_feedback=ef)
gen = torch.Generator(device="cuda"); gen.manual_seed(5)
gs = [torch.randn(d, generator=gen, device="cuda") for _ in range(8)]
r = torch.zeros(d, device="cuda"); out = torch.empty(d, device="cuda")
lib = ctypes.CDLL(tk.lib_path())
buf = np.zeros((2, 32, 2048), np.uint64)
G = None
acc = []
for s in range(200):
    if ef:
        ctx.step(gs[s % 8], r, out)
    else:
        ctx.compress(gs[s % 8], None)
    if s >= 40 and s % 10 == 0:
        torch.cuda.synchronize()
        assert lib.tk_debug_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
        st = buf[0].astype(np.int64)
        G = int((st[0] > 0).sum())
        t0 = st[0, :G].min()
        acc.append((buf.astype(np.int64)[:, :, :G] - t0))
a = np.stack(acc)  # [samples][2][32][G]
smid = buf[1, 30, :G].astype(np.int64)
np.savez(os.environ.get("TRACE_OUT", "/tmp/trace.npz"), a=a, smid=smid)
n = len(acc)
print(f"EF={ef} d={d} CTAs={G} samples={n} (us, relative to the earliest CTA start; median over samples of min/med/max over CTAs)")
for kind, name in ((0, "stamp"), (1, "arrive")):
    for slot in range(32):
        v = a[:, kind, slot, :]
        if (v[:, 0] <= 0).all() and slot != 0:
            continue
        mn, md, mx = (np.median(v.min(1)) / 1e3, np.median(np.median(v, 1)) / 1e3, np.median(v.max(1)) / 1e3)
        late = np.bincount(v.argmax(1), minlength=G).argmax()
        print(f"  {name:6s} {slot:2d}: min {mn:7.2f} med {md:7.2f} max {mx:7.2f}  (latest CTA most often: {late})")
# EF-pass arrival (barrier 1) by SM load: CTAs with a run (arrival > 5 us) per SM, and arrival percentiles
arr = np.median(a[:, 1, 1, :], 0) / 1e3
busy = arr > 5.0
per_sm = np.bincount(smid, weights=busy.astype(float), minlength=smid.max() + 1)
load = per_sm[smid]
print("  ef arrivals of busy CTAs: p10 %.2f p50 %.2f p90 %.2f p99 %.2f max %.2f" % tuple(np.percentile(arr[busy], [10, 50, 90, 99, 100])))
for nb in sorted(set(load[busy].astype(int))):
    sel = busy & (load == nb)
    print(f"  SMs with {nb} busy CTAs: {sel.sum()} CTAs, arrival p50 {np.median(arr[sel]):.2f} max {arr[sel].max():.2f}")
