"""Multi-GPU parity worker, launched by tests/test_multigpu.py under torchrun (one rank per GPU).

Every rank runs libtk's tk_step on its own seeded gradient; rank 0 regenerates all ranks'
gradients, runs the CPU oracle (oracle.flat_step / oracle.hitopk_step, all ranks simulated in one
process) and compares bit for bit: the gathered (index, value) pairs, the aggregated gradient of
EVERY rank, and every rank's residual, at every step.  Writes a JSON verdict to --out.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gradgen  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, required=True)
    ap.add_argument("--rho", type=float, default=0.001)
    ap.add_argument("--n-iters", type=int, default=10)
    ap.add_argument("--group-size", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--dist", default="G")
    ap.add_argument("--step4", default="dense")
    ap.add_argument("--rs-mode", default="ordered")
    ap.add_argument("--ag-mode", default="push")
    ap.add_argument("--select", default="mstopk")
    ap.add_argument("--wire", default="f32")
    ap.add_argument("--sgd", type=float, default=0.0, help="also run Eq. 1's fused update with this lr")
    ap.add_argument("--zero-copy", action="store_true", help="write g into the context's input buffer")
    ap.add_argument("--bucket", action="store_true", help="drive the step through tk.Bucket (3 layer views)")
    ap.add_argument("--symmetric", action="store_true",
                    help="g and out in tk_alloc_symmetric buffers (in-place step 1, fused dense step 4)")
    ap.add_argument("--no-ef", action="store_true", help="error feedback off")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()

    rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2010_10458_b200 as tk

    def log(*x):
        if os.environ.get("TK_WORKER_LOG"):
            print(f"[rank {rank}]", *x, flush=True)

    uid = tk.broadcast_unique_id()
    log("uid ok")
    n = a.group_size
    kw = dict(n_iters=a.n_iters, nranks=ws, rank=rank, group_size=n, seed=99, uid=uid, step4=a.step4,
              rs_mode=a.rs_mode, ag_mode=a.ag_mode, device=local, select=a.select, wire=a.wire,
              error_feedback=not a.no_ef)
    bucket = None
    if a.bucket:  # the same flat gradient, seen as three layers of one bucket (reading Q32)
        q = a.dim // 3
        bucket = tk.Bucket([(q,), (1,), (a.dim - q - 1,)], rho=a.rho, **kw)
        ctx = bucket.ctx
    else:
        ctx = tk.Context(a.dim, rho=a.rho, **kw)
    L, k = ctx.seg_len, ctx.k
    log("ctx ok", L, k)
    chunks = ws if n == 1 else ws // n
    r = torch.zeros(L, dtype=torch.float32, device="cuda") if bucket is None else bucket.residual
    results = []
    ok = True
    r_ref = [np.zeros(L, np.float32) for _ in range(ws)]
    inbuf = ctx.input_buffer() if a.zero_copy else None
    sym_g = [ctx.alloc_symmetric(a.dim) for _ in range(2)] if a.symmetric else None  # alternate between two
    sym_out = ctx.alloc_symmetric(a.dim) if a.symmetric else None
    w_ref = gradgen.gradient(a.dim, "G", cfg=41)
    wd = torch.from_numpy(w_ref.copy()).cuda()
    for step in range(a.steps):
        g = torch.from_numpy(gradgen.gradient(a.dim, a.dist, cfg=40, rank=rank, step=step)).cuda()
        if inbuf is not None:
            inbuf.copy_(g)
            g = inbuf
        if sym_g is not None:
            sym_g[step % 2].copy_(g)
            g = sym_g[step % 2]
        gat = torch.empty(chunks * ctx.chunk_words, dtype=torch.int32, device="cuda")
        if bucket is not None:
            for (o, cnt, _), view in zip(bucket.layout, bucket.grads):
                view.copy_(g[o:o + cnt])
            bucket.step(gathered=gat)
            out = bucket.flat_out
        elif a.sgd:
            out = torch.empty(a.dim, dtype=torch.float32, device="cuda")
            ctx.step_sgd(g, r, wd, a.sgd, out=out, gathered=gat)
        else:
            out = ctx.step(g, r if not a.no_ef else None, out=sym_out, gathered=gat)
        torch.cuda.synchronize()
        log("step", step, "done")
        outs = [torch.empty_like(out) for _ in range(ws)]
        gats = [torch.empty_like(gat) for _ in range(ws)]
        rs = [torch.empty_like(r) for _ in range(ws)]
        wds = [torch.empty_like(wd) for _ in range(ws)]
        dist.all_gather(wds, wd)
        dist.all_gather(outs, out)
        dist.all_gather(gats, gat)
        dist.all_gather(rs, r)
        if rank == 0:
            import oracle
            grads = [gradgen.gradient(a.dim, a.dist, cfg=40, rank=p, step=step) for p in range(ws)]
            if n == 1:
                ref = oracle.flat_step(grads, r_ref, a.rho, a.n_iters, seed=99, step=step, selector=a.select,
                                       wire=a.wire, error_feedback=not a.no_ef)
                ref_gat = [ref.gathered] * ws
            else:
                ref = oracle.hitopk_step(grads, r_ref, ws // n, n, a.rho, a.n_iters, seed=99, step=step,
                                         selector=a.select, wire=a.wire, error_feedback=not a.no_ef)
                ref_gat = [ref.column_gathered[p % n] for p in range(ws)]
            rec = {"step": step}
            rec["out_equal"] = [bool(np.array_equal(o.cpu().numpy().view(np.uint32), ref.out.view(np.uint32)))
                                for o in outs]
            rec["gathered_equal"] = [bool(np.array_equal(gg.cpu().numpy().view(np.uint32), ref_gat[p]))
                                     for p, gg in enumerate(gats)]
            rec["residual_equal"] = [a.no_ef or bool(np.array_equal(rr.cpu().numpy().view(np.uint32),
                                                                    ref.per_rank[p].residual.view(np.uint32)))
                                     for p, rr in enumerate(rs)]
            if a.sgd:
                w_ref = oracle.sgd_update(w_ref, ref.out, a.sgd)
                rec["w_equal"] = [bool(np.array_equal(x.cpu().numpy().view(np.uint32), w_ref.view(np.uint32)))
                                  for x in wds]
                ok = ok and all(rec["w_equal"])
            rec["max_abs_diff"] = max(float(np.max(np.abs(o.cpu().numpy() - ref.out))) for o in outs)
            rec["nnz_out"] = int(np.count_nonzero(ref.out))
            ok = ok and all(rec["out_equal"]) and all(rec["gathered_equal"]) and all(rec["residual_equal"])
            results.append(rec)
            if not a.no_ef:
                r_ref = [ref.per_rank[p].residual for p in range(ws)]
        dist.barrier()
    if rank == 0:
        with open(a.out, "w") as f:
            json.dump({"ok": ok, "P": ws, "n": n, "d": a.dim, "k": k, "steps": results}, f, indent=1)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
