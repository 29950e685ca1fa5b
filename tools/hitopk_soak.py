"""HiTopKComm soak (run under torchrun on 4 GPUs): ROUNDS x {1x4 sparse step 4, 2x2 dense step 4} fresh
contexts, each with symmetric (IPC-mapped) gradient / output buffers and EF-pass compaction, STEPS
steps on fresh N(0,1) gradients.  After every context: the device error flags (tk_get_stats), and the
aggregate must be identical on every rank (Alg. 2: every GPU ends with the same g~) - checked as
the max - min over ranks of a bit hash of `out`.  Prints one line per context; exits non-zero on
the first inconsistency (a crash shows as a non-zero torchrun exit).
    torchrun --nproc-per-node 4 tools/hitopk_soak.py [ROUNDS] [STEPS]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2010_10458_b200 as tk

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 50
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
rank, ws, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
d = 25_600_000
gen = torch.Generator(device="cuda")
gen.manual_seed(7 + rank)
t0 = time.time()
for it in range(rounds):
    for n, step4 in ((4, "sparse"), (2, "dense")):
        uid = tk.broadcast_unique_id()
        stream = torch.cuda.Stream()
        ctx = tk.Context(d, rho=0.001, n_iters=10, nranks=ws, rank=rank, group_size=n, seed=it, step4=step4, uid=uid,
                         stream=stream, device=local)
        with torch.cuda.stream(stream):
            gs = [ctx.alloc_symmetric(d) for _ in range(4)]
            out = ctx.alloc_symmetric(d)
            r = torch.zeros(ctx.seg_len, device="cuda")
            for s in range(steps):
                gs[s % 4].normal_(generator=gen)
                ctx.step(gs[s % 4], r, out)
        stream.synchronize()
        st = ctx.stats()
        h = torch.tensor([int(out.view(torch.int32).to(torch.int64).mul_(2654435761).sum().item()) & ((1 << 62) - 1)],
                         dtype=torch.int64, device="cuda")
        hmax, hmin = h.clone(), h.clone()
        dist.all_reduce(hmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(hmin, op=dist.ReduceOp.MIN)
        ok = bool(hmax.item() == hmin.item())
        if rank == 0:
            print(f"round {it} {1 if n == 4 else 2}x{n} {step4}: {steps} steps ok={ok} ef_compacted={st.ef_compacted} "
                  f"t={time.time() - t0:.0f}s", flush=True)
        del gs, out
        ctx.close()
        if not ok:
            sys.exit(3)
dist.destroy_process_group()
