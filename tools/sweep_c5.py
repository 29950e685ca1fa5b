"""BASELINE config 5 (the paper's Fig. 6 analogue): size / density / N sweep of the
compression on one B200 - MSTopK (Alg. 1), the exact top-k of Eq. 2 (libtk's F1 selector) and, as
context, torch.topk on |x| - with MSTopK's recall against the exact top-k.  Writes JSONL.

Per configuration: a fresh context, 6 warm-up calls, then 20 timed calls on fresh N(0,1) gradients
(4 buffers cycled) with error feedback (the regime of a training step), CUDA events on the context
stream; recall from one call of each selector on the same gradient without error feedback."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2010_10458_b200 as tk

SIZES = [262_144, 1_000_000, 4_000_000, 16_000_000, 25_600_000, 64_000_000, 110_000_000, 134_217_728, 336_000_000]
RHOS = [1e-4, 1e-3, 1e-2]
NS = [5, 10, 20, 30]
out = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5_sweep.jsonl", "w")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
gen = torch.Generator(device="cuda")
gen.manual_seed(201010458)


def timed(fn, gs, reps=20, warm=6):
    for i in range(warm):
        fn(gs[i % len(gs)])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(reps):
        fn(gs[i % len(gs)])
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for d in SIZES:
    gs = [torch.randn(d, generator=gen, device="cuda") for _ in range(4)]
    torch.cuda.synchronize()
    for rho in RHOS:
        k = tk.k_from_density(d, rho)
        # exact top-k (F1) and torch.topk once per (d, rho)
        r = torch.zeros(d, device="cuda")
        ce = tk.Context(d, rho=rho, select="exact", stream=stream)
        idx_e = torch.empty(k, dtype=torch.int32, device="cuda"); val_e = torch.empty(k, device="cuda")
        t_exact = timed(lambda g: ce.compress(g, r, idx_e, val_e), gs)
        ce.close()
        t_torch = timed(lambda g: torch.topk(g.abs(), k, sorted=False), gs)
        cx = tk.Context(d, rho=rho, select="exact", error_feedback=False, stream=stream)
        ix, _ = cx.compress(gs[0])
        ix = ix.long(); cx.close()
        for N in NS:
            r.zero_()
            c = tk.Context(d, rho=rho, n_iters=N, stream=stream)
            idx = torch.empty(k, dtype=torch.int32, device="cuda"); val = torch.empty(k, device="cuda")
            t_ms = timed(lambda g: c.compress(g, r, idx, val), gs)
            st = c.stats()
            c.close()
            c0 = tk.Context(d, rho=rho, n_iters=N, error_feedback=False, stream=stream)
            i0, v0 = c0.compress(gs[0])
            torch.cuda.synchronize()
            recall = int(torch.isin(i0.long(), ix).sum().item()) / k
            mag = float(v0.abs().double().sum().item()) / float(gs[0].abs()[ix].double().sum().item())
            c0.close()
            rec = {"d": d, "rho": rho, "k": k, "N": N, "P": 1, "ef": True, "dist": "G",
                   "mstopk_us": t_ms, "exact_us": t_exact, "torch_topk_us": t_torch,
                   "mstopk_elements_per_s": d / (t_ms * 1e-6), "hbm_floor_GBps": (12 * d + 12 * k) / (t_ms * 1e-6) / 1e9,
                   "recall_vs_exact": recall, "magnitude_ratio_vs_exact": mag,
                   "ef_compacted": st.ef_compacted, "n_compacted": st.n_compacted}
            out.write(json.dumps(rec) + "\n"); out.flush()
            print(json.dumps(rec), flush=True)
    del gs
    torch.cuda.empty_cache()
