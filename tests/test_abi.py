"""C-ABI contract checks that need no GPU: libtk.so loads, exports every symbol include/tk.h
declares, and its pure host helpers behave (no compute call is made without a GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "tk.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tk_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ["tk_init", "tk_compress", "tk_sparse_allgather", "tk_decompress", "tk_step"]:
        assert n in names


def test_library_loads_and_exports_every_declared_symbol():
    import paper_2010_10458_b200 as tk
    lib = ctypes.CDLL(tk.lib_path())
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(tk.EXPORTS) == _declared()


def test_library_is_sm100a_and_links_nccl():
    import subprocess
    import paper_2010_10458_b200 as tk
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", tk.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", tk.lib_path()], capture_output=True, text=True).stdout
    assert "libnccl.so.2" in deps


def test_tk_k_rounding():
    import paper_2010_10458_b200 as tk
    for d, rho, k in [(1000, 0.001, 1), (1048576, 0.001, 1048), (8, 1.0, 8), (25600000, 0.001, 25600),
                      (110000000, 0.001, 110000), (134217728, 0.001, 134217), (10, 1e-4, 1)]:
        assert tk.k_from_density(d, rho) == k
    with pytest.raises(ValueError):
        tk.k_from_density(0, 0.1)
    with pytest.raises(ValueError):
        tk.k_from_density(10, 1.5)


def test_status_strings():
    import paper_2010_10458_b200 as tk
    lib = tk._lib
    assert lib.tk_status_string(0) == b"ok"
    assert lib.tk_status_string(4) == b"non-finite input"
    assert lib.tk_status_string(99) == b"unknown status"


def test_init_rejects_bad_config_before_touching_the_gpu():
    import paper_2010_10458_b200 as tk
    lib = tk._lib

    def init(**kw):
        base = dict(d=1000, rho=0.01, k=0, n_iters=10, nranks=1, rank=0, group_size=1, seed=0, rand_mode=0,
                    error_feedback=1, step4=0, levels_per_pass=0, device=-1)
        base.update(kw)
        cfg = tk._Config(**base)
        ctx = ctypes.c_void_p()
        return lib.tk_init(ctypes.byref(cfg), None, None, ctypes.byref(ctx))

    assert init(d=0) == 1
    assert init(d=1 << 32) == 1
    assert init(rho=0.0) == 1
    assert init(rho=1.5) == 1
    assert init(n_iters=0) == 1
    assert init(n_iters=53) == 1
    assert init(rank=1) == 1
    assert init(nranks=2, rank=0) == 3            # no NCCL unique id
    assert init(nranks=6, group_size=4) == 3      # P % n != 0
    assert init(d=1001, nranks=2, group_size=2) == 3  # d % n != 0
    assert init(d=1004, nranks=4, group_size=4) == 3  # (d / n) % 4 != 0: unaligned segments
    assert init(k=1001) == 2                      # k > d
    assert init(levels_per_pass=11) == 1


def test_product_has_no_cpu_path():
    import torch
    import paper_2010_10458_b200 as tk
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        tk.Context(1000, 0.01, 10)
