"""Build libtk.so in-tree for sm_100a with nvcc (no JIT cache: the .so travels with the repo).

    python paper_2010_10458_b200/build.py            # release build (never imports the package)
    python paper_2010_10458_b200/build.py --verbose  # also print ptxas register/spill report
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtk.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("the venv's nvidia-nccl package (torch's NCCL) is required")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith(".cu")]


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = sources()
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "tk.h"))
    if not force and os.path.exists(OUT) and all(os.path.getmtime(OUT) >= os.path.getmtime(d) for d in deps):
        return OUT
    inc, lib = nccl_dirs()
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "--split-compile=0", "-Xcompiler", "-fPIC,-O2",
           "-shared", "-o", OUT, *srcs, "-I", os.path.join(ROOT, "include"), "-I", inc, "-L", lib,
           "-l:libnccl.so.2", f"-Xlinker=-rpath,{lib}", "-lcudart"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    return OUT


if __name__ == "__main__":
    build(verbose="--verbose" in sys.argv, force=True)
