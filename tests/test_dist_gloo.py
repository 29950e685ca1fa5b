"""CPU, world_size 2 (gloo): the multi-process host logic of the N > 1 path.

* the NCCL unique-id bootstrap of the binding (rank 0 creates it with libtk, torch.distributed
  broadcasts the 128 bytes) gives every rank the same id;
* the distributed decomposition of the path — each rank compresses its own gradient, the packed
  chunks are all-gathered rank-major, every rank decompresses in rank order — reproduces the
  single-process simulation (oracle.flat_step) bit for bit on every rank;
* the HiTopKComm decomposition (row groups reduce-scatter in rank order, per-segment MSTopK,
  column all-gather, row all-gather) with m x n = 1 x 2 and 2 x 1 process groups matches
  oracle.hitopk_step.
The arithmetic is the oracle's (the CUDA path is covered by tests/test_multigpu.py on GPUs)."""
import functools
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gradgen
import oracle


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        q.put((rank, fn(rank, ws)))
    except Exception as e:  # surfaced in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _spawn(fn, ws=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, fn, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=180) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
    return out


def _uid(rank, ws):
    import paper_2010_10458_b200 as tk
    return tk.broadcast_unique_id()


def test_unique_id_broadcast():
    out = _spawn(_uid)
    assert isinstance(out[0], bytes) and len(out[0]) == 128
    assert out[0] == out[1]


D, RHO, N, STEPS = 20_008, 0.01, 10, 3


def _flat(selector, wire, rank, ws):
    r = np.zeros(D, np.float32)
    outs = []
    k = oracle.k_from_density(D, RHO)
    for step in range(STEPS):
        g = gradgen.gradient(D, "G", cfg=50, rank=rank, step=step)
        c = oracle.compress(g, r, k, N, seed=3, step=step, rank=rank, selector=selector, wire=wire)
        chunk = torch.from_numpy(oracle.pack(c.sel.idx, c.sent, wire).view(np.int32))
        gathered = [torch.empty_like(chunk) for _ in range(ws)]
        dist.all_gather(gathered, chunk)
        g_all = torch.cat(gathered).numpy().view(np.uint32)
        outs.append(oracle.decompress(g_all, ws, k, D, wire).view(np.uint32).tobytes())
        r = c.residual
    return outs


@pytest.mark.parametrize("selector,wire", [("mstopk", "f32"), ("exact", "f32"), ("mstopk", "f16")])
def test_flat_decomposition_matches_simulation(selector, wire):
    """the per-rank compress / packed all-gather / rank-ordered decompress decomposition (also with the
    exact selector, F1, and FP16 wire values, F3) reproduces the single-process simulation"""
    out = _spawn(functools.partial(_flat, selector, wire))
    r = [np.zeros(D, np.float32) for _ in range(2)]
    for step in range(STEPS):
        gs = [gradgen.gradient(D, "G", cfg=50, rank=p, step=step) for p in range(2)]
        ref = oracle.flat_step(gs, r, RHO, N, seed=3, step=step, selector=selector, wire=wire)
        for rank in range(2):
            assert out[rank][step] == ref.out.view(np.uint32).tobytes()
        r = [c.residual for c in ref.per_rank]


def _hitopk_body(m, n, rank, ws):
    i, j = rank // n, rank % n
    rows = [dist.new_group([a * n + b for b in range(n)]) for a in range(m)]
    cols = [dist.new_group([a * n + b for a in range(m)]) for b in range(n)]
    L = D // n
    kt = oracle.k_from_density(L, RHO)
    r = np.zeros(L, np.float32)
    outs = []
    for step in range(STEPS):
        g = torch.from_numpy(gradgen.gradient(D, "G", cfg=51, rank=rank, step=step))
        # step 1: rank-ordered reduce-scatter inside the row
        parts = [torch.empty_like(g) for _ in range(n)]
        dist.all_gather(parts, g, group=rows[i])
        seg = parts[0].numpy()[j * L:(j + 1) * L].copy()
        for q in range(1, n):
            seg = (seg + parts[q].numpy()[j * L:(j + 1) * L]).astype(np.float32)
        # step 2: MSTopK on the segment
        c = oracle.compress(seg, r, kt, N, seed=4, step=step, rank=rank)
        # step 3: column all-gather + accumulation in group order
        chunk = torch.from_numpy(oracle.pack(c.sel.idx, c.sel.val).view(np.int32))
        gat = [torch.empty_like(chunk) for _ in range(m)]
        dist.all_gather(gat, chunk, group=cols[j])
        G = oracle.decompress(torch.cat(gat).numpy().view(np.uint32), m, kt, L)
        # step 4: row all-gather of the segments
        segs = [torch.empty(L, dtype=torch.float32) for _ in range(n)]
        dist.all_gather(segs, torch.from_numpy(G), group=rows[i])
        outs.append(torch.cat(segs).numpy().view(np.uint32).tobytes())
        r = c.residual
    return outs


@pytest.mark.parametrize("m,n", [(1, 2), (2, 1)])
def test_hitopk_decomposition_matches_simulation(m, n):
    out = _spawn(functools.partial(_hitopk_body, m, n))
    r = [np.zeros(D // n, np.float32) for _ in range(2)]
    for step in range(STEPS):
        gs = [gradgen.gradient(D, "G", cfg=51, rank=p, step=step) for p in range(2)]
        ref = oracle.hitopk_step(gs, r, m, n, RHO, N, seed=4, step=step)
        for rank in range(2):
            assert out[rank][step] == ref.out.view(np.uint32).tobytes(), (m, n, step, rank)
        r = [c.residual for c in ref.per_rank]


# ---------------------------------------------------------------- world size 8 (the 8-GPU box layout)
def _flat_ws(rank, ws):
    return _flat("mstopk", "f32", rank, ws)


def test_flat_decomposition_world_size_8():
    """flat NaiveAG at P = 8 (BASELINE configs 2-3's 8-GPU aggregation): 8 processes, each its own
    gradient and residual, one rank-major all-gather, rank-ordered decompression on every rank"""
    ws = 8
    out = _spawn(_flat_ws, ws=ws)
    r = [np.zeros(D, np.float32) for _ in range(ws)]
    for step in range(STEPS):
        gs = [gradgen.gradient(D, "G", cfg=50, rank=p, step=step) for p in range(ws)]
        ref = oracle.flat_step(gs, r, RHO, N, seed=3, step=step)
        for rank in range(ws):
            assert out[rank][step] == ref.out.view(np.uint32).tobytes(), (step, rank)
        r = [c.residual for c in ref.per_rank]


@pytest.mark.parametrize("m,n", [(2, 4), (4, 2), (2, 2)])
def test_hitopk_decomposition_world_size_8(m, n):
    """HiTopKComm's virtual-node layouts of BASELINE config 4 (2x4 and 4x2 on 8 processes; 2x2 on 4):
    row groups (rank // n), column groups (rank % n), ordered reduce-scatter, per-segment MSTopK,
    column all-gather, row all-gather - every rank's aggregate equals oracle.hitopk_step's"""
    ws = m * n
    out = _spawn(functools.partial(_hitopk_body, m, n), ws=ws)
    r = [np.zeros(D // n, np.float32) for _ in range(ws)]
    for step in range(STEPS):
        gs = [gradgen.gradient(D, "G", cfg=51, rank=p, step=step) for p in range(ws)]
        ref = oracle.hitopk_step(gs, r, m, n, RHO, N, seed=4, step=step)
        for rank in range(ws):
            assert out[rank][step] == ref.out.view(np.uint32).tobytes(), (m, n, step, rank)
        r = [c.residual for c in ref.per_rank]
