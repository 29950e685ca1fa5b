#!/usr/bin/env python
"""Benchmark of the MSTopK + sparse-aggregation hot path (arXiv 2010.10458 CommLib) on B200.

    python bench.py [--gpus N --steps K --warmup W]                 # libtk (this repo)
    python bench.py --impl reference [--gpus N --steps K --warmup W] # the CPU oracle (reference arm)
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One step = one whole iteration of the hot path on every rank: error feedback, MSTopK (N = 10
samplings), compaction into (index, value) pairs, the sparse All-Gather across the P ranks,
rank-ordered decompression into the dense aggregate, residual write-back.
Workload (BASELINE.json configs[1], C2): d = 25.6M fp32 gradient per rank, rho = 1e-3
(k = 25 600), N = 10, error feedback on; P = N GPUs, flat NaiveAG (weak scaling: every rank
brings its own d-vector).  Metric: elements/s = P*d / (max-over-ranks device time per step).

Rank 0 prints ONE JSON line.  See DESIGN.md §Measurement for the roofline accounting.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import gradgen  # noqa: E402  (seeded inputs only; no method arithmetic)

METRIC = "MSTopK+aggregation elements/s"
UNIT = "elements/s"
HBM_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="tk", choices=["tk", "reference"])
    ap.add_argument("--d", "--dim", dest="d", type=int, default=25_600_000)
    ap.add_argument("--rho", type=float, default=0.001)
    ap.add_argument("--n-iters", type=int, default=10)
    ap.add_argument("--dist", default="G")
    ap.add_argument("--group-size", type=int, default=1, help="HiTopKComm n (1 = flat NaiveAG)")
    ap.add_argument("--step4", default="dense", choices=["dense", "sparse"])
    ap.add_argument("--levels", type=int, default=0, help="bisection levels per count pass (0 = default)")
    ap.add_argument("--ag-mode", default="push", choices=["push", "nccl"], help="flat all-gather: fused peer push or NCCL")
    ap.add_argument("--rs-mode", default="ordered", choices=["ordered", "nccl"],
                    help="HiTopKComm step-1 reduce-scatter: ordered peer reads (bit-exact) or NCCL")
    ap.add_argument("--select", default="mstopk", choices=["mstopk", "exact"],
                    help="selector: MSTopK (Alg. 1) or the exact top-k of Eq. 2 (SURVEY F1)")
    ap.add_argument("--wire", default="f32", choices=["f32", "f16"],
                    help="value format on the wire: fp32 or binary16 (SURVEY F3, Fig. 7's FP16)")
    ap.add_argument("--sgd", type=float, default=0.0,
                    help="lr > 0: time tk_step_sgd (Eq. 1's update fused into the decompression, SURVEY F4)")
    ap.add_argument("--no-symmetric", action="store_true",
                    help="HiTopKComm: plain gradient / output tensors (copy-in, NCCL row all-gather)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra single-GPU configurations")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--ncu", action="store_true", help="short run for ncu: no soak, no e2e, no cpu baseline")
    return ap.parse_args()


def workload_name(a, P):
    if a.group_size > 1:
        return f"C4 HiTopKComm {P // a.group_size}x{a.group_size} d={a.d} rho={a.rho} N={a.n_iters}"
    tag = "C2" if a.d == 25_600_000 else ("C3" if a.d == 110_000_000 else "custom")
    if a.select == "exact":
        return f"{tag} exact top-k (Eq. 2) + flat sparse allgather d={a.d} rho={a.rho} EF P={P}"
    return f"{tag} flat sparse allgather d={a.d} rho={a.rho} N={a.n_iters} EF P={P}"


def k_of(d, rho):
    import math
    return max(1, int(math.floor(float(rho) * float(d))))


def measured_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.proc = None
        self.path = f"/tmp/tk_clocks_{os.getpid()}.csv"
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------ dist
def dist_setup(a):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.gpus != ws:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={ws}: launch N>1 with torchrun")
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.is_available() and a.impl == "tk":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda" if torch.cuda.is_available() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, ws):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ------------------------------------------------------------------------------------------ CPU oracle
def time_oracle_step(d, rho, N, P, n, seed=1, dist="G", selector="mstopk", wire="f32", gs=None):
    """One full simulated step of the oracle (all P ranks in one process); returns seconds."""
    import oracle
    if gs is None:
        gs = [gradgen.gradient(d, dist, cfg=2, rank=p, step=0) for p in range(P)]
    t0 = time.perf_counter()
    if n == 1:
        rs = [np.zeros(d, np.float32) for _ in range(P)]
        oracle.flat_step(gs, rs, rho, N, seed=seed, selector=selector, wire=wire)
    else:
        rs = [np.zeros(d // n, np.float32) for _ in range(P)]
        oracle.hitopk_step(gs, rs, P // n, n, rho, N, seed=seed, selector=selector, wire=wire)
    return time.perf_counter() - t0


def _oracle_worker(args):
    """One host core: repeat whole simulated oracle steps (P ranks, d per rank) for budget_s seconds.
    Returns (steps done, seconds spent in them)."""
    d, rho, N, P, n, dist, selector, wire, budget_s, wid = args
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    gs = [gradgen.gradient(d, dist, cfg=2, rank=p, step=wid) for p in range(P)]
    steps, spent = 0, 0.0
    while spent < budget_s or steps == 0:
        spent += time_oracle_step(d, rho, N, P, n, dist=dist, selector=selector, wire=wire, gs=gs)
        steps += 1
    return steps, spent


def host_cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def host_ram_gb():
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable"):
                return int(line.split()[1]) / 1e6
    except OSError:
        pass
    return 8.0


def oracle_throughput(d, rho, N, P, n, dist, selector, wire, budget_s, workers):
    """The oracle as it stands, run as `workers` independent instances on as many host cores (one
    process each, numpy single-threaded): elements of whole simulated steps per wall second."""
    import multiprocessing as mp
    args = [(d, rho, N, P, n, dist, selector, wire, budget_s, w) for w in range(workers)]
    t0 = time.perf_counter()
    if workers == 1:
        res = [_oracle_worker(args[0])]
    else:
        with mp.get_context("spawn").Pool(workers) as pool:
            res = pool.map(_oracle_worker, args)
    wall = time.perf_counter() - t0
    steps = sum(r[0] for r in res)
    busy = max(r[1] for r in res)  # the slowest worker's time inside its steps (excludes start-up)
    return P * d * steps / busy, steps, busy, wall


def oracle_workers(d, P):
    """as many processes as host cores, bounded by host RAM (~40 B per element and rank in flight)"""
    cores = host_cores() or 1
    per = max(1e-3, 40.0 * d * P / 1e9)
    return max(1, min(cores, int(host_ram_gb() * 0.6 / per)))


def cpu_baseline(a, P, budget_s=12.0):
    d_s = a.d
    val1, steps1, busy1, _ = oracle_throughput(d_s, a.rho, a.n_iters, 1, 1, a.dist, a.select, a.wire, budget_s, 1)
    w = oracle_workers(d_s, 1)
    valn, stepsn, busyn, _ = oracle_throughput(d_s, a.rho, a.n_iters, 1, 1, a.dist, a.select, a.wire, budget_s, w)
    return {"value": valn, "unit": UNIT, "cores": w, "kind": "oracle",
            "sample": f"{stepsn} full single-rank oracle steps at d={d_s}, rho={a.rho}, N={a.n_iters}, EF, run as {w} "
                      f"independent numpy processes (1 thread each) on the host's {host_cores()} cores "
                      f"({host_cpu_model()}); {busyn:.1f} s each",
            "single_core": {"value": val1, "cores": 1, "sample": f"{steps1} steps on one core, {busy1:.1f} s"}}


def run_reference(a, ws, rank, emit):
    if rank != 0:
        return
    P = ws
    n = a.group_size
    d_s = max(n * 4096, (min(a.d, 25_600_000 // P) // n) * n)  # bounded sample of the workload per step
    w = oracle_workers(d_s, P)
    # warm-up: a.warmup whole steps on one core (the oracle has no state to warm; this loads numpy)
    for _ in range(max(1, a.warmup)):
        time_oracle_step(d_s, a.rho, a.n_iters, P, n, dist=a.dist, selector=a.select, wire=a.wire)
    # timed: the oracle on every host core, each core repeating whole simulated P-rank steps; at
    # least a.steps steps in total
    budget = max(5.0, min(60.0, 2.0 * a.steps * time_oracle_step(d_s, a.rho, a.n_iters, P, n, dist=a.dist,
                                                                   selector=a.select, wire=a.wire) / w))
    val, steps, busy, wall = oracle_throughput(d_s, a.rho, a.n_iters, P, n, a.dist, a.select, a.wire, budget, w)
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": ws, "steps": steps, "warmup": a.warmup,
            "ms_per_step": P * d_s / val * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(a, P), "d": a.d, "rho": a.rho, "n_iters": a.n_iters, "P": P,
                       "group_size": n, "dist": a.dist, "sample_d_per_rank": d_s},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": w, "kind": "oracle",
                             "sample": f"{steps} whole {P}-rank steps simulated on d={d_s} per rank (bounded sample of "
                                       f"d={a.d}), {w} independent numpy processes (1 thread each) on the host's "
                                       f"{host_cores()} cores ({host_cpu_model()}); {busy:.1f} s each, "
                                       f"{wall:.1f} s wall; ms_per_step = one step's elements / throughput"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ------------------------------------------------------------------------------------------ libtk arm
def stage_bytes(name, L, d, k, P, ef, chunks, fused_out=False):
    """Algorithmic HBM bytes of ONE launch of a stage."""
    if name == "k_compress":
        # the floor of any correct implementation: the EF pass (read g, read r, write acc - or read
        # g without EF), the k (index, value) pairs and the k residual writes.  This design moves
        # only that plus the compacted entries (~0.4 % of n, data dependent, not counted).  P = 1
        # tk_step without the fused update: the kernel also writes the dense aggregate (its zeros,
        # 4 B/element, and its k values, 4 B/pair) - there is no decompression then.
        return ((12 if ef else 4) * L + 8 * k + (4 * k if ef else 0) +
                ((4 * L + 4 * k) if fused_out else 0))
    if name == "k_decompress":
        return 4 * d + 8 * chunks * k
    if name == "k_tile_ranges":
        return 4 * chunks * k
    return None


NVLINK_GBS = 770.0  # measured peer copy per direction per GPU (B200_PROFILING.md); 900 nominal


def nvlink_report(a, stages, P, n, L, k, t_step_ms, cw):
    """Bytes each GPU must move over NVLink per step for every exchange of the path, and the
    achieved rate over the stage that carries it, against the measured 770 GB/s per direction
    (Eq. 3 for the flat all-gather, Eqs. 7-10 for HiTopKComm's steps)."""
    if P == 1:
        return None
    m = P // n

    def st(name):
        v = stages.get(name)
        return v["ms_per_launch"] * v["launches_per_step"] if v else None

    def entry(nbytes, ms, carried_by):
        out = {"bytes_per_gpu": nbytes, "stage": carried_by}
        if ms:
            out.update({"ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9, "frac": nbytes / (ms * 1e-3) / 1e9 / NVLINK_GBS})
        return out
    rep = {"peak_GBps": NVLINK_GBS, "peak_source": "measured peer copy per direction (B200_PROFILING.md; 900 nominal)"}
    if n == 1:
        ag = 4 * (P - 1) * cw  # received: every other rank's packed chunk (8k B with fp32 values)
        if a.ag_mode == "push":
            # fused: the packets are pushed by k_compress and consumed by k_decompress; the exchange
            # has no stage of its own, so the whole step bounds it
            rep["allgather"] = entry(ag, t_step_ms, "fused into k_compress + k_decompress (step time as the bound)")
        else:
            rep["allgather"] = entry(ag, st("allgather"), "ncclAllGather")
        rep["allgather"]["time_at_peak_us"] = ag / NVLINK_GBS / 1e3
        return rep
    rs = 4 * (n - 1) * L  # H1: the peer segments this GPU reads (ordered RS fused into the EF pass)
    rep["h1_reduce_scatter"] = entry(rs, st("k_compress") if a.rs_mode == "ordered" else st("reduce_scatter"),
                                     "k_compress (peer loads)" if a.rs_mode == "ordered" else "ncclReduceScatter")
    rep["h3_column_allgather"] = entry(4 * (m - 1) * cw, st("allgather"), "ncclAllGather (column)")
    if a.step4 == "dense":
        s4 = 4 * (n - 1) * L
        t4 = (st("k_decompress") or 0) + (st("step4_allgather") or 0)
        rep["h5_row_allgather"] = entry(s4, t4, "k_decompress replica stores + row barrier" if not a.no_symmetric
                                        else "k_decompress + ncclAllGather (row)")
    else:
        rep["h5_row_allgather"] = entry(4 * (n - 1) * m * cw, st("step4_allgather"), "ncclAllGather (row, pairs)")
    for key in ("h1_reduce_scatter", "h3_column_allgather", "h5_row_allgather"):
        rep[key]["time_at_peak_us"] = rep[key]["bytes_per_gpu"] / NVLINK_GBS / 1e3
    return rep


def extra_configs(a, tk, stream, gs, dev):
    """Single-GPU context numbers measured after the timed region (device time, CUDA events on the
    context stream, fresh gradients): BASELINE config 1 (d = 1M, EF off, tk_compress only, from a
    CUDA graph so the host's launch cost is excluded); the first call of a fresh context (no
    prediction) and a forced restart (the gradient scale jumps x1000); the C2 step with the layered
    ResNet-like profile, with the prose search (F3) and with the exact selector (F1)."""
    import torch
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def steps_us(ctx, bufs, n, r):
        for i in range(3):
            ctx.step(bufs[i % len(bufs)], r)
        e0, e1 = ev(), ev()
        e0.record(stream)
        for i in range(n):
            ctx.step(bufs[i % len(bufs)], r)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / n

    res = {}
    with torch.cuda.stream(stream):
        # C1
        d1 = 1_000_000
        c1 = tk.Context(d1, rho=a.rho, n_iters=a.n_iters, error_feedback=False, stream=stream, device=dev)
        g1 = [torch.randn(d1, device="cuda") for _ in range(16)]
        idx = torch.empty(c1.k, dtype=torch.int32, device="cuda")
        val = torch.empty(c1.k, device="cuda")
        for i in range(40):
            c1.compress(g1[i % 16], None, idx, val)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            for i in range(16):
                c1.compress(g1[i], None, idx, val)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(20):
            graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        res["C1_compress_us"] = e0.elapsed_time(e1) * 1e3 / 320
        res["C1_phases_us"] = [round(x, 2) for x in c1.stats().phase_us]
        c1.close()
        del g1
        # C2 k_compress back to back: tk_compress calls on fresh gradients with the residual carried,
        # CUDA events around the whole loop only (no event between launches, so consecutive
        # launches overlap through programmatic dependent launch as they do inside a step)
        c = tk.Context(a.d, rho=a.rho, n_iters=a.n_iters, stream=stream, device=dev)
        r = torch.zeros(a.d, device="cuda")
        cidx = torch.empty(c.k, dtype=torch.int32, device="cuda")
        cval = torch.empty(c.k, device="cuda")
        for i in range(20):
            c.compress(gs[i % len(gs)], r, cidx, cval)
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for i in range(100):
            c.compress(gs[i % len(gs)], r, cidx, cval)
        e1.record(stream)
        torch.cuda.synchronize()
        res["C2_compress_back_to_back_us"] = e0.elapsed_time(e1) * 1e3 / 100
        c.close()
        del r
        # first call / restart at C2 (median of 3 fresh contexts / 3 forced restarts)
        first, restart, whole = [], [], []
        for rep in range(3):
            c = tk.Context(a.d, rho=a.rho, n_iters=a.n_iters, stream=stream, device=dev)
            r = torch.zeros(a.d, device="cuda")
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record(stream)
            c.step(gs[rep % len(gs)], r)
            e1.record(stream)
            torch.cuda.synchronize()
            first.append(e0.elapsed_time(e1) * 1e3)
            for i in range(10):
                c.step(gs[(i + 1) % len(gs)], r)
            big = gs[rep % len(gs)] * 1000.0
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record(stream)
            c.step(big, r)
            e1.record(stream)
            torch.cuda.synchronize()
            restart.append(e0.elapsed_time(e1) * 1e3)
            whole.append(not c.stats().ef_compacted)
            c.close()
            del big, r
        res["C2_first_step_us"] = sorted(first)[1]
        res["C2_restart_step_us"] = sorted(restart)[1]
        res["C2_restart_took_whole_vector_path"] = all(whole)
        # layered profile
        gl = [torch.from_numpy(gradgen.gradient(a.d, "L", cfg=2, step=s_)).cuda() for s_ in range(4)]
        c = tk.Context(a.d, rho=a.rho, n_iters=a.n_iters, stream=stream, device=dev)
        res["C2_dist_L_step_us"] = steps_us(c, gl, 20, torch.zeros(a.d, device="cuda"))
        c.close()
        del gl
        for sel in ("prose", "exact"):
            c = tk.Context(a.d, rho=a.rho, n_iters=a.n_iters, stream=stream, device=dev, select=sel)
            res[f"C2_{sel}_step_us"] = steps_us(c, gs, 20, torch.zeros(a.d, device="cuda"))
            c.close()
    res["note"] = ("device time per call / step (CUDA events, fresh gradients); C1 replays 16 tk_compress calls "
                   "per CUDA graph; C2_compress_back_to_back: 100 tk_compress calls between two events (the "
                   "roofline's per-launch events sit inside the steps instead); prose = TK_SELECT_PROSE (P:148), "
                   "exact = TK_SELECT_EXACT (Eq. 2)")
    return res


def log(*x):
    print(f"[bench {time.strftime('%H:%M:%S')}]", *x, file=sys.stderr, flush=True)


def main():
    # C-level stdout (e.g. NCCL's version banner) goes to stderr: stdout carries exactly one JSON line
    json_fd = os.dup(1)
    os.dup2(2, 1)

    def emit(obj):
        os.write(json_fd, (json.dumps(obj) + "\n").encode())

    a = parse()
    ws, rank, local = dist_setup(a)
    log("rank", rank, "of", ws, "up")
    if a.impl == "reference":
        run_reference(a, ws, rank, emit)
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    import torch
    import paper_2010_10458_b200 as tk
    torch.cuda.set_device(local)
    P = ws
    n = a.group_size
    uid = tk.broadcast_unique_id() if P > 1 else None
    stream = torch.cuda.Stream()
    ctx = tk.Context(a.d, rho=a.rho, n_iters=a.n_iters, nranks=P, rank=rank, group_size=n, seed=2010_10458,
                     step4=a.step4, levels_per_pass=a.levels, uid=uid, stream=stream, device=local, ag_mode=a.ag_mode,
                     select=a.select, rs_mode=a.rs_mode, wire=a.wire)
    L, k = ctx.seg_len, ctx.k
    log("ctx up")
    # inputs: a fresh seeded N(0,1) gradient for every warm-up / timed / profiled step, generated on
    # the device before any timing (pool capped at ~16 GB per rank; reused cyclically beyond that)
    need = a.warmup + 2 * a.steps
    nbuf = max(2, min(need, int(16e9 // (4 * a.d))))
    # HiTopKComm with the ordered reduce-scatter: the gradients live in symmetric (IPC-mapped)
    # buffers, as a training loop would produce them (no per-step copy-in), and so does out (the
    # dense step 4 is then fused into the decompression)
    sym = n > 1 and a.rs_mode == "ordered" and not a.no_symmetric
    if sym:
        nbuf = min(nbuf, 8)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(201010458 + 1000 * rank)
    with torch.cuda.stream(stream):
        gs = [ctx.alloc_symmetric(a.d) if sym else torch.empty(a.d, device="cuda") for _ in range(nbuf)]
        for s_, gt in enumerate(gs):
            if a.dist == "G":
                gt.normal_(generator=gen)
            else:
                gt.copy_(torch.from_numpy(gradgen.gradient(a.d, a.dist, cfg=2, rank=rank, step=s_)))
        r = torch.zeros(L, dtype=torch.float32, device="cuda")
        r_soak = torch.zeros(L, dtype=torch.float32, device="cuda")
        out = ctx.alloc_symmetric(a.d) if sym else torch.empty(a.d, dtype=torch.float32, device="cuda")
        w = torch.randn(a.d, generator=gen, device="cuda", dtype=torch.float32) if a.sgd else None
    stream.synchronize()
    cursor = [0]
    log("inputs generated")

    def run(steps, rr=None):
        rr = r if rr is None else rr
        for _ in range(steps):
            if a.sgd:  # F4: Eq. 1's update fused into the decompression (no dense aggregate written)
                ctx.step_sgd(gs[cursor[0] % nbuf], rr, w, a.sgd)
            else:
                ctx.step(gs[cursor[0] % nbuf], rr, out)
            cursor[0] += 1

    sampler = None if a.ncu else ClockSampler(local)
    if not a.ncu:
        # keep the GPU under this load ~1 s (on a scratch residual) so the clock samples describe
        # the timed region's regime; every rank runs the same number of steps (collectives match)
        torch.cuda.synchronize()
        t0 = time.time()
        with torch.cuda.stream(stream):
            run(50, r_soak)
        stream.synchronize()
        per = max_over_ranks((time.time() - t0) / 50, ws)
        n_soak = int(min(20000, max(10, 1.0 / max(per, 1e-6))))
        with torch.cuda.stream(stream):
            for i in range(0, n_soak, 50):
                run(min(50, n_soak - i), r_soak)
                stream.synchronize()
    log("soak done")
    cursor[0] = 0
    ctx.set_step(0)
    with torch.cuda.stream(stream):
        r.zero_()
        run(a.warmup)
    stream.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        run(a.steps)
        e1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    barrier(ws)
    clocks = sampler.stop() if sampler else None
    log("timed region done")
    launches = ctx.launches - l0
    t_step = max_over_ranks(e0.elapsed_time(e1) / a.steps, ws)  # ms, max over ranks
    gpu_launches = int(sum_over_ranks(launches, ws))
    value = P * a.d / (t_step * 1e-3)

    # per-stage breakdown over K more steps with stage events (same stream, same buffers)
    ctx.profile_begin(a.steps)
    with torch.cuda.stream(stream):
        run(a.steps)
    prof = ctx.profile_end()
    log("profile done")
    chunks = P if n == 1 else P // n
    stages = {}
    for name, (ms, cnt) in prof.items():
        stages[name] = {"ms_per_launch": ms / cnt, "launches_per_step": cnt / a.steps,
                        "share": ms / a.steps / t_step if t_step > 0 else None}
    compute = {kname: v for kname, v in stages.items() if kname.startswith("k_")}
    dom = max(compute, key=lambda kn: compute[kn]["ms_per_launch"] * compute[kn]["launches_per_step"])
    peak, peak_src = measured_hbm()
    fused_out = n == 1 and P == 1 and not a.sgd  # P = 1 tk_step: k_compress writes the aggregate whole
    bytes_launch = stage_bytes(dom, L, a.d, k, P, True, chunks, fused_out)
    achieved = bytes_launch / (stages[dom]["ms_per_launch"] * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tr = json.load(open(tp))
            key = f"{dom}@d={L}"
            traffic = tr.get(key)
        except Exception:
            traffic = None
    literal = None
    if dom == "k_compress":  # bytes Alg. 1 moves as written: EF + N count passes + 2 index passes
        literal = ((16 + 4 * a.n_iters) * L + 12 * k) / (stages[dom]["ms_per_launch"] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "effective_literal_alg1_GBps": literal,
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": bytes_launch,
                "ms_per_launch": stages[dom]["ms_per_launch"],
                "note": ("achieved = algorithmic bytes per launch (the floor: " +
                         ("16 B/elem (EF: read g, r; write acc; write the dense aggregate, which at P = 1 this "
                          "kernel writes) + 16 B/pair" if fused_out else
                          "12 B/elem (EF: read g, r; write acc) + 12 B/pair") +
                         ") / mean CUDA-event duration of that launch inside the profiled steps")}

    nvlink = nvlink_report(a, stages, P, n, L, k, t_step, ctx.chunk_words)
    # comparator: the dense all-reduce of the whole fp32 gradient the sparse path replaces (the paper's
    # TreeAR / dense baseline): ncclAllReduce of 4d bytes, max over ranks
    allreduce = None
    if P > 1 and not a.ncu:
        import torch.distributed as dist
        buf = gs[0].clone()
        for _ in range(3):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        barrier(ws)
        ka = max(5, min(a.steps, 20))
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record()
        for _ in range(ka):
            dist.all_reduce(buf)
        eb.record()
        torch.cuda.synchronize()
        t_ar = max_over_ranks(ea.elapsed_time(eb) / ka, ws)
        allreduce = {"ms": t_ar, "elements_per_s": P * a.d / (t_ar * 1e-3),
                     "bus_GBps": 2 * (P - 1) / P * 4 * a.d / (t_ar * 1e-3) / 1e9,
                     "sparse_step_speedup": t_ar / t_step,
                     "note": "torch.distributed.all_reduce (NCCL) of the dense fp32 gradient, max over ranks"}
        del buf

    # end-to-end through the public host-buffer API: pinned H2D of g + D2H of the gathered pairs
    e2e = None
    if not a.no_e2e and not a.ncu:
        ctx_h = ctx
        hg = [torch.from_numpy(gradgen.gradient(a.d, a.dist, cfg=2, rank=rank, step=s)).pin_memory() for s in range(2)]
        gat_h = torch.empty(chunks * ctx.chunk_words, dtype=torch.int32).pin_memory()
        for i in range(3):
            ctx_h.step_host(hg[i % 2], gat_h)
        barrier(ws)
        ks = max(5, min(a.steps, 50))
        t0 = time.perf_counter()
        for i in range(ks):
            ctx_h.step_host(hg[i % 2], gat_h)
        t_e2e = max_over_ranks((time.perf_counter() - t0) / ks, ws)
        log("e2e done")
        e2e = {"value": P * a.d / t_e2e, "unit": UNIT, "ms_per_step": t_e2e * 1e3,
               "h2d_bytes_per_step": 4 * a.d, "d2h_bytes_per_step": 4 * chunks * ctx.chunk_words,
               "api": "tk_step_host (pinned host gradient in, gathered (index, value) pairs out; residual device-resident)"}

    # MSTopK's recall against the exact top-k of Eq. 2 (the comparison of the paper's Fig. 6), both
    # selections made by libtk's kernels on the same step-0 gradient (no error feedback), outside
    # the timed region: |iota_MSTopK ∩ iota_exact| / k and the ratio of the selected |x| mass
    recall = None
    if rank == 0 and P == 1 and n == 1 and a.select == "mstopk" and not a.ncu:
        sel = {}
        for kind in ("mstopk", "exact"):
            c = tk.Context(a.d, rho=a.rho, n_iters=a.n_iters, seed=2010_10458, select=kind, error_feedback=False,
                           device=local)
            idx, val = c.compress(gs[0])
            torch.cuda.synchronize()
            sel[kind] = (idx.long(), val.abs().double().sum().item())
            c.close()
        hit = int(torch.isin(sel["mstopk"][0], sel["exact"][0]).sum().item())
        recall = {"index_recall": hit / k, "magnitude_ratio": sel["mstopk"][1] / sel["exact"][1],
                  "note": "MSTopK vs exact top-k (Eq. 2) on the step-0 gradient, both on the GPU, EF off"}

    extra = None
    if rank == 0 and P == 1 and n == 1 and not a.ncu and not a.no_extra:
        extra = extra_configs(a, tk, stream, gs, local)
        log("extra configurations done")

    cpu = None
    if rank == 0 and P == 1 and not a.no_cpu_baseline and not a.ncu:
        cpu = cpu_baseline(a, P)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": P, "steps": a.steps, "warmup": a.warmup,
                "ms_per_step": t_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": workload_name(a, P), "d": a.d, "rho": a.rho, "k": k, "n_iters": a.n_iters,
                           "P": P, "group_size": n, "step4": a.step4 if n > 1 else None, "dist": a.dist,
                           "allgather": (a.ag_mode if n == 1 and P > 1 else None), "selector": a.select,
                           "wire": a.wire, "fused_sgd_lr": a.sgd or None,
                           "levels_per_pass": a.levels or 10, "input_buffers": nbuf,
                           "inputs": "fresh seeded N(0,1) gradient per step (torch CUDA generator, pre-generated in "
                                     "HBM); residual carried from r=0 at step 0; timed steps W..W+K-1",
                           "l2": "inputs larger than L2: each step reads a fresh g (4d B), reads and writes r and "
                                 f"writes out: {16 * a.d / 1e6:.0f} MB per rank per step vs 126 MB L2; no explicit flush"},
                "gpu_launches": gpu_launches, "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu,
                "e2e": e2e, "stages": stages, "recall_vs_exact": recall, "nvlink": nvlink,
                "dense_allreduce_comparator": allreduce, "extra_configs": extra}
        emit(line)
    ctx.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
