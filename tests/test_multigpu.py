"""Multi-GPU parity (flat NaiveAG at P = 2/4/8 and HiTopKComm virtual nodes) through torchrun:
one process per GPU, NCCL over NVLink, every rank's aggregate / residual / gathered pairs
compared bit for bit with the CPU oracle (tests/mp_worker.py).  Cases needing more GPUs than
the box has are skipped."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(P, tmp_path, **kw):
    if not torch.cuda.is_available():
        pytest.fail("GPU tests selected but no CUDA device is visible")
    if torch.cuda.device_count() < P:
        pytest.skip(f"needs {P} GPUs, box has {torch.cuda.device_count()}")
    out = tmp_path / "res.json"
    extra = []
    for key, v in kw.items():
        if v is True:
            extra.append("--" + key.replace("_", "-"))
        else:
            extra += ["--" + key.replace("_", "-"), str(v)]
    for attempt in range(3):  # the free port can be taken between probe and bind: retry on EADDRINUSE
        args = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
                "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "mp_worker.py"),
                "--out", str(out)] + extra
        proc = subprocess.Popen(args, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT,
                                start_new_session=True)
        try:
            so, se = proc.communicate(timeout=150)
        except subprocess.TimeoutExpired:
            os.killpg(proc.pid, 9)  # the whole torchrun process group, workers included
            so, se = proc.communicate()
            pytest.fail("multi-GPU worker timed out:\n" + so[-2000:] + se[-3000:])
        if proc.returncode == 0 or "EADDRINUSE" not in se:
            break
    assert proc.returncode == 0, so[-3000:] + se[-3000:]
    verdict = json.loads(out.read_text())
    assert verdict["ok"], json.dumps(verdict["steps"], indent=1)[:4000]
    return verdict


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("ag", ["push", "nccl"])
def test_flat_sparse_allgather(P, ag, tmp_path):
    _run(P, tmp_path, dim=1_000_003, rho=0.001, steps=3, ag_mode=ag)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_flat_c2_full_size(P, tmp_path):
    """BASELINE config 2 (d = 25.6M, rho = 1e-3, N = 10, error feedback) at P GPUs."""
    _run(P, tmp_path, dim=25_600_000, rho=0.001, steps=2)


@pytest.mark.parametrize("P,n,step4,rs", [(2, 2, "dense", "ordered"), (2, 2, "sparse", "nccl"), (4, 2, "dense", "ordered"),
                                          (4, 4, "dense", "ordered"), (4, 4, "sparse", "ordered"),
                                          (4, 2, "sparse", "ordered"), (8, 4, "dense", "ordered"),
                                          (8, 2, "dense", "ordered"), (8, 4, "sparse", "ordered")])
def test_hitopk_virtual_nodes(P, n, step4, rs, tmp_path):
    """HiTopKComm (Alg. 2): m = P/n virtual nodes of n GPUs (2x4 / 4x2 on 8 GPUs, BASELINE config 4).
    The NCCL reduce-scatter is bit-exact only for n = 2 (a two-term sum commutes)."""
    _run(P, tmp_path, dim=8 * 131_076, rho=0.001, group_size=n, step4=step4, rs_mode=rs, steps=3)


def test_hitopk_zero_copy_input(tmp_path):
    _run(2, tmp_path, dim=2 * 100_004, rho=0.01, group_size=2, zero_copy=True, steps=3)


@pytest.mark.parametrize("P,n", [(4, 2), (8, 4), (8, 2)])
def test_hitopk_c4_full_size(P, n, tmp_path):
    """BASELINE config 4: d = 25.6M HiTopKComm (2x4, 4x2 on 8 GPUs; 2x2 on 4)."""
    _run(P, tmp_path, dim=25_600_000, rho=0.001, group_size=n, steps=2)


@pytest.mark.parametrize("P,n", [(2, 1), (4, 1), (4, 2)])
def test_exact_selector_multi_gpu(P, n, tmp_path):
    """the exact top-k selector (Eq. 2) on the flat push path and HiTopKComm"""
    _run(P, tmp_path, dim=8 * 131_076, rho=0.001, group_size=n, select="exact", steps=3)


@pytest.mark.parametrize("P,n,step4", [(2, 1, "dense"), (4, 2, "dense"), (4, 2, "sparse")])
def test_fused_sgd_update_multi_gpu(P, n, step4, tmp_path):
    """Eq. 1's update fused into the decompression (flat), or after the row all-gather (dense step 4)"""
    _run(P, tmp_path, dim=8 * 131_076, rho=0.001, group_size=n, step4=step4, sgd=0.05, steps=3)


@pytest.mark.parametrize("P,n,ag,step4", [(2, 1, "push", "dense"), (4, 1, "push", "dense"), (2, 1, "nccl", "dense"),
                                          (4, 2, "push", "dense"), (4, 2, "push", "sparse")])
def test_fp16_wire_multi_gpu(P, n, ag, step4, tmp_path):
    """FP16 wire values (F3) through the fused push all-gather, NCCL and HiTopKComm"""
    _run(P, tmp_path, dim=1_049_616, rho=0.001, group_size=n, ag_mode=ag, step4=step4, wire="f16", steps=3)


@pytest.mark.parametrize("P,n", [(2, 1), (4, 1), (2, 2), (4, 2)])
def test_bucketed_step_multi_gpu(P, n, tmp_path):
    """the bucketed multi-tensor step (reading Q32): three layer views of one bucket,
    flat or HiTopKComm (whose bucket gradient is libtk's peer-visible input buffer)"""
    _run(P, tmp_path, dim=8 * 131_076 if n > 1 else 1_000_003, rho=0.001, group_size=n, bucket=True, steps=3)


@pytest.mark.parametrize("P,n,step4", [(2, 2, "dense"), (4, 4, "dense"), (4, 2, "dense"), (4, 2, "sparse"),
                                       (8, 4, "dense"), (8, 2, "dense")])
def test_hitopk_symmetric_buffers(P, n, step4, tmp_path):
    """g and out in tk_alloc_symmetric buffers: the ordered reduce-scatter reads the peers' gradients
    in place (no copy-in) and the dense step 4 is fused into the decompression (NVLink replica stores
    into every node peer's out, then a row barrier) - Alg. 2 bit for bit, five steps"""
    _run(P, tmp_path, dim=8 * 131_076, rho=0.001, group_size=n, step4=step4, symmetric=True, steps=5)


@pytest.mark.parametrize("P,n,step4", [(2, 2, "dense"), (4, 2, "sparse")])
def test_hitopk_no_error_feedback(P, n, step4, tmp_path):
    """HiTopKComm with the ordered reduce-scatter and error feedback off (the peer sum is stored to a
    segment scratch; round 1 crashed here)"""
    _run(P, tmp_path, dim=8 * 131_076, rho=0.001, group_size=n, step4=step4, no_ef=True, steps=3)


@pytest.mark.parametrize("P,n", [(4, 2), (4, 4), (8, 4), (8, 2)])
def test_hitopk_c4_full_size_symmetric(P, n, tmp_path):
    """BASELINE config 4 at full size with symmetric buffers, 4 steps (the EF-pass compaction of the
    peer-sum kernel from step 1 on)"""
    _run(P, tmp_path, dim=25_600_000, rho=0.001, group_size=n, symmetric=True, steps=4)
