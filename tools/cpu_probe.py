"""Host enqueue time per tk_step vs device time per step (is the GPU starved by the CPU?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2010_10458_b200 as tk
ws = int(os.environ.get("WORLD_SIZE", "1")); rank = int(os.environ.get("RANK", "0")); local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
uid = None
if ws > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = tk.broadcast_unique_id()
mode = sys.argv[1] if len(sys.argv) > 1 else "push"
d = 25_600_000
ctx = tk.Context(d, rho=0.001, n_iters=10, nranks=ws, rank=rank, uid=uid, device=local, ag_mode=mode)
gs = [torch.randn(d, device="cuda") for _ in range(4)]
r = torch.zeros(d, device="cuda"); out = torch.empty(d, device="cuda")
for i in range(20): ctx.step(gs[i % 4], r, out)
torch.cuda.synchronize()
if ws > 1: dist.barrier()
n = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter(); e0.record()
for i in range(n): ctx.step(gs[i % 4], r, out)
t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
print(f"rank {rank} ws {ws} {mode}: host enqueue {1e6*(t1-t0)/n:.1f} us/step, device {1e3*e0.elapsed_time(e1)/n:.1f} us/step", flush=True)
ctx.profile_begin(n)
for i in range(n): ctx.step(gs[i % 4], r, out)
prof = ctx.profile_end()
print(f"rank {rank} ws {ws} {mode} stages:", {k: round(ms / c * 1e3, 1) for k, (ms, c) in prof.items()}, flush=True)
st = ctx.stats()
print(f"rank {rank} phases:", [round(x, 1) for x in st.phase_us], "compacted", st.compacted, st.n_compacted, flush=True)
