"""Single-GPU parity of the multi-GPU kernels, with every rank of a
P-GPU job emulated on ONE GPU (libtk `loopback` contexts, no communicator):

* HiTopKComm (Alg. 2): each emulated GPU (i, j) runs `tk_compress_segment` - the same
  `k_compress<EF, NP>` kernel `tk_step` launches with CUDA-IPC peer pointers - on the n local
  buffers of its virtual node (H1, ordered reduce-scatter fused into the EF pass, Eq. 4; H2, MSTopK
  on the segment, Eq. 5); the column all-gather (H3, an NCCL call in tk_step) is a concatenation
  here; the group-ordered accumulation (H4) and step 4 (H5, dense: concatenation of the segments;
  sparse: every GPU decompresses every segment's gathered pairs) run through `tk_decompress`.
* The fused push all-gather (F2): every emulated rank runs `tk_loopback_push` - the
  compression kernel with its tagged-packet stores into every rank's packet buffer - then every
  rank runs the packet-consuming decompression (`k_decompress<TaggedChunks>`).  All pushes finish
  before any decompression starts (one stream), so no kernel waits on another launch.

Everything is compared bit for bit with the CPU oracle (oracle.hitopk_step / oracle.flat_step),
per step, with the residuals carried."""
import numpy as np
import pytest

import gradgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def tk():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests selected but no CUDA device is visible")
    import paper_2010_10458_b200 as tk
    return tk


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _u32(t):
    return t.cpu().numpy().view(np.uint32)


def _bits(t):
    return t.cpu().numpy().astype(np.float32).view(np.uint32)


def _check_stats(st, sel):
    """every field of the control block, bit for bit (exact_trial_counts contexts)"""
    assert st.mean == sel.mean and st.max_bits == int(np.float32(sel.u).view(np.uint32))
    assert st.nnz_not_counted == 0
    assert [t[1:] for t in st.trials] == [(b[1], b[2], b[3]) for b in sel.trials]
    assert (st.k1, st.k2, st.key1, st.key2, st.len2, st.rand) == (sel.k1, sel.k2, sel.key1, sel.key2, sel.len2,
                                                                 sel.rand)
    assert st.thres1 == sel.thres1 and st.thres2 == sel.thres2


# ------------------------------------------------------------------------------ HiTopKComm
def _hitopk_loopback(tk, d, m, n, rho, N, steps, *, dist="G", ef=True, step4="dense", select="mstopk", wire="f32",
                     seed=31, cfg=70):
    P = m * n
    L = d // n
    ctxs = [tk.Context(d, rho=rho, n_iters=N, nranks=P, rank=p, group_size=n, seed=seed, error_feedback=ef,
                       step4=step4, select=select, wire=wire, loopback=True, exact_trial_counts=True)
            for p in range(P)]
    kt = ctxs[0].k
    assert kt == oracle.k_from_density(L, rho) and ctxs[0].seg_len == L
    res = [np.zeros(L, np.float32) for _ in range(P)]
    rd = [_dev(r) for r in res]
    for step in range(steps):
        grads = [gradgen.gradient(d, dist, cfg=cfg, rank=p, step=step) for p in range(P)]
        gd = [_dev(g) for g in grads]
        ref = oracle.hitopk_step(grads, res, m, n, rho, N, seed=seed, step=step, error_feedback=ef, selector=select,
                                 wire=wire)
        chunks = {}
        for i in range(m):
            for j in range(n):
                p = i * n + j
                c = ctxs[p]
                c.set_step(step)
                # H1 + H2: the n buffers of virtual node i, segment j, summed in ascending row rank
                srcs = [gd[i * n + q][j * L:(j + 1) * L] for q in range(n)]
                chunk = torch.empty(c.chunk_words, dtype=torch.int32, device="cuda")
                idx = chunk[:kt]
                if wire == "f32":
                    val = chunk[kt:].view(torch.float32)
                    c.compress_segment(srcs, rd[p] if ef else None, idx=idx, val=val)
                else:
                    val = torch.empty(kt, dtype=torch.float32, device="cuda")
                    c.compress_segment(srcs, rd[p] if ef else None, idx=idx, val=val)
                    chunk = _pack16(idx, val, c.chunk_words)
                cr = ref.per_rank[p]
                if select != "exact":
                    _check_stats(c.stats(), cr.sel)
                assert np.array_equal(_u32(idx), cr.sel.idx), (step, p)
                assert np.array_equal(_bits(val), cr.sent.view(np.uint32)), (step, p)
                if ef:
                    assert np.array_equal(_bits(rd[p]), cr.residual.view(np.uint32)), (step, p)
                chunks[p] = chunk
        # H3: column all-gather (groups i = 0..m-1 at position j); H4: group-ordered accumulation
        segs = []
        for j in range(n):
            col = torch.cat([chunks[i * n + j] for i in range(m)])
            assert np.array_equal(_u32(col), ref.column_gathered[j]), (step, j)
            segs.append(ctxs[j].decompress(col, nchunks=m))
        # H5 dense: every GPU of a node concatenates the n segments (identical on every GPU)
        out = torch.cat(segs)
        assert np.array_equal(_bits(out), ref.out.view(np.uint32)), step
        if step4 == "sparse":
            # H5 sparse (Eq. 10): a GPU decompresses every segment's m*k~ gathered pairs itself
            for p in (0, P - 1):
                parts = [ctxs[p].decompress(torch.cat([chunks[i * n + j] for i in range(m)]), nchunks=m)
                         for j in range(n)]
                assert np.array_equal(_bits(torch.cat(parts)), ref.out.view(np.uint32)), (step, p)
        if ef:
            res = [ref.per_rank[p].residual for p in range(P)]
    for c in ctxs:
        c.close()


def _pack16(idx, val, cw):
    """[idx k | binary16 val k (zero pad)] - the FP16 wire chunk (values already fp16-exact)"""
    k = idx.numel()
    h = val.to(torch.float16)
    if k % 2:
        h = torch.cat([h, torch.zeros(1, dtype=torch.float16, device=h.device)])
    return torch.cat([idx, h.view(torch.int32)])[:cw]


@pytest.mark.parametrize("m,n", [(1, 2), (2, 2), (1, 4), (2, 4), (4, 2), (1, 8)])
def test_hitopk_loopback_small(tk, m, n):
    _hitopk_loopback(tk, 400_000, m, n, 0.001, 10, 3)


@pytest.mark.parametrize("m,n", [(2, 4), (4, 2)])
def test_hitopk_loopback_dense_rho_1e2(tk, m, n):
    # C4 at the paper's Fig. 8 density
    _hitopk_loopback(tk, 1_000_000, m, n, 0.01, 10, 2, dist="L")


@pytest.mark.parametrize("ef", [True, False])
def test_hitopk_loopback_error_feedback_off(tk, ef):
    # EF off: the peer sum is stored in the segment scratch (the ordered-RS kernel has no residual)
    _hitopk_loopback(tk, 300_000, 2, 2, 0.001, 10, 2, ef=ef)


def test_hitopk_loopback_sparse_step4(tk):
    _hitopk_loopback(tk, 300_000, 2, 4, 0.001, 10, 2, step4="sparse")


@pytest.mark.parametrize("select", ["exact", "prose"])
def test_hitopk_loopback_selectors(tk, select):
    _hitopk_loopback(tk, 200_000, 2, 2, 0.001, 10, 2, select=select)


def test_hitopk_loopback_wire16(tk):
    _hitopk_loopback(tk, 200_000, 2, 2, 0.001, 10, 2, wire="f16")


@pytest.mark.parametrize("m,n", [(2, 4), (4, 2)])
def test_hitopk_loopback_full_size_c4(tk, m, n):
    """BASELINE config 4 at full size (d = 25.6M, rho = 1e-3, N = 10, EF): the 2x4 and 4x2
    virtual-node shapes, three steps with the segment residuals carried (the later steps take the
    EF-pass compaction of the peer-sum kernel)."""
    _hitopk_loopback(tk, 25_600_000, m, n, 0.001, 10, 3)


def test_hitopk_peer_sum_compaction_soak(tk):
    """many consecutive steps of the peer-sum kernel with the EF-pass compaction (the path the
    round-1 build had disabled for NP > 0): every step bit-exact, and compacted after step 0"""
    d, n, rho, N = 2_000_000, 4, 0.001, 10
    L = d // n
    c = tk.Context(d, rho=rho, n_iters=N, nranks=n, rank=1, group_size=n, seed=5, loopback=True,
                   exact_trial_counts=True)
    r = np.zeros(L, np.float32)
    rd = _dev(r)
    used = []
    for step in range(12):
        grads = [gradgen.gradient(d, "G", cfg=80, rank=q, step=step) for q in range(n)]
        srcs = [_dev(g[L:2 * L]) for g in grads]
        c.set_step(step)
        idx, val = c.compress_segment(srcs, rd)
        seg = oracle.reduce_scatter_ordered(grads, n, 0, 1)
        ref = oracle.compress(seg, r, c.k, N, seed=5, step=step, rank=1)
        st = c.stats()
        _check_stats(st, ref.sel)
        assert np.array_equal(_u32(idx), ref.sel.idx) and np.array_equal(_bits(val), ref.sel.val.view(np.uint32))
        assert np.array_equal(_bits(rd), ref.residual.view(np.uint32))
        used.append(st.ef_compacted)
        r = ref.residual
    assert all(used[1:]), used


# ------------------------------------------------------------------------------ fused push all-gather
def _push_loopback(tk, d, P, rho, N, steps, *, dist="G", wire="f32", seed=41, cfg=90):
    ctxs = [tk.Context(d, rho=rho, n_iters=N, nranks=P, rank=p, seed=seed, wire=wire, loopback=True,
                       exact_trial_counts=True) for p in range(P)]
    k, cw = ctxs[0].k, ctxs[0].chunk_words
    # every rank's packet buffer: [P][k] 16-byte packets (zero = tag 0, never a step's tag)
    bufs = [torch.zeros(P * 2 * k, dtype=torch.int64, device="cuda") for _ in range(P)]
    res = [np.zeros(d, np.float32) for _ in range(P)]
    rd = [_dev(r) for r in res]
    for step in range(steps):
        tag = step + 1
        grads = [gradgen.gradient(d, dist, cfg=cfg, rank=p, step=step) for p in range(P)]
        ref = oracle.flat_step(grads, res, rho, N, seed=seed, step=step, wire=wire)
        for p in range(P):
            ctxs[p].set_step(step)
            chunk = torch.empty(cw, dtype=torch.int32, device="cuda")
            slots = [bufs[q][2 * k * p:2 * k * (p + 1)] for q in range(P)]
            ctxs[p].loopback_push(_dev(grads[p]), rd[p], chunk, slots, tag)
            assert np.array_equal(_u32(chunk), ref.gathered[p * cw:(p + 1) * cw]), (step, p)
            assert np.array_equal(_bits(rd[p]), ref.per_rank[p].residual.view(np.uint32)), (step, p)
            _check_stats(ctxs[p].stats(), ref.per_rank[p].sel)
        for q in (range(P) if d <= 4_000_000 else (0, P - 1)):
            plain = torch.empty(P * cw, dtype=torch.int32, device="cuda")
            out = ctxs[q].loopback_decompress(bufs[q], P, tag, plain_out=plain)
            assert np.array_equal(_u32(plain), ref.gathered), (step, q)
            assert np.array_equal(_bits(out), ref.out.view(np.uint32)), (step, q)
        res = [ref.per_rank[p].residual for p in range(P)]
    for c in ctxs:
        c.stats()  # no timeout, no non-finite input
        c.close()


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_push_allgather_loopback(tk, P):
    _push_loopback(tk, 500_003, P, 0.001, 10, 3)


def test_push_allgather_loopback_wire16(tk):
    _push_loopback(tk, 300_000, 4, 0.001, 10, 2, wire="f16")


def test_push_allgather_loopback_full_size_c2(tk):
    """BASELINE config 2 at full size (d = 25.6M) with P = 8 emulated ranks: the packets every rank
    pushes and the rank-ordered aggregate every rank decompresses, two steps."""
    _push_loopback(tk, 25_600_000, 8, 0.001, 10, 2)


def test_push_allgather_timeout_reports_error(tk):
    """a packet that never arrives: the decompression gives up after push_timeout_ms (no trap, no
    hang), stays memory-safe, and the next tk_get_stats reports TK_ERR_TIMEOUT"""
    d, P = 100_000, 2
    c = tk.Context(d, rho=0.001, n_iters=10, nranks=P, rank=0, loopback=True, push_timeout_ms=30)
    k = c.k
    buf = torch.zeros(P * 2 * k, dtype=torch.int64, device="cuda")
    r = torch.zeros(d, device="cuda")
    chunk = torch.empty(c.chunk_words, dtype=torch.int32, device="cuda")
    c.loopback_push(_dev(gradgen.gradient(d, "G", cfg=91)), r, chunk, [buf[:2 * k]], 1)  # rank 1 never pushes
    c.loopback_decompress(buf, P, 1)
    torch.cuda.synchronize()
    with pytest.raises(tk.TkError) as e:
        c.stats()
    assert e.value.status == 9
    c.close()


# ------------------------------------------------------------------------------ fused dense step 4
@pytest.mark.parametrize("m,n", [(2, 4), (4, 2), (1, 8)])
def test_hitopk_fused_dense_step4_replicated_decompress(tk, m, n):
    """HiTopKComm's dense step 4 fused into step 3's accumulation (Alg. 2 l.15-23): GPU (i, j)
    decompresses its column-gathered pairs once and writes segment j into the out buffer of every GPU
    of its node (tk_decompress_replicated - on a node the replicas are the peers' CUDA-IPC mapped
    outs); after all n positions ran, every GPU's out must equal the oracle's aggregate bit for bit."""
    d, rho, N = 400_000, 0.001, 10
    P, L = m * n, 400_000 // n
    ctxs = [tk.Context(d, rho=rho, n_iters=N, nranks=P, rank=p, group_size=n, seed=8, loopback=True) for p in range(P)]
    kt = ctxs[0].k
    grads = [gradgen.gradient(d, "G", cfg=95, rank=p) for p in range(P)]
    res = [np.zeros(L, np.float32) for _ in range(P)]
    ref = oracle.hitopk_step(grads, res, m, n, rho, N, seed=8)
    gd = [_dev(g) for g in grads]
    chunks = {}
    for i in range(m):
        for j in range(n):
            c = ctxs[i * n + j]
            chunk = torch.empty(c.chunk_words, dtype=torch.int32, device="cuda")
            c.compress_segment([gd[i * n + q][j * L:(j + 1) * L] for q in range(n)], _dev(res[i * n + j]),
                               idx=chunk[:kt], val=chunk[kt:].view(torch.float32))
            chunks[i * n + j] = chunk
    for i in range(m):  # node i: n output buffers, filled by the n positions' replicated decompressions
        outs = [torch.full((d,), float("nan"), device="cuda") for _ in range(n)]
        for j in range(n):
            col = torch.cat([chunks[a * n + j] for a in range(m)])
            ctxs[i * n + j].decompress_replicated(col, [o[j * L:(j + 1) * L] for o in outs], nchunks=m)
        for q in range(n):
            assert np.array_equal(_bits(outs[q]), ref.out.view(np.uint32)), (i, q)
    for c in ctxs:
        c.close()
