"""A few small tk_step iterations (flat, P = 1) for compute-sanitizer (memcheck /
racecheck / synccheck of the kernels at small d).  Run: compute-sanitizer --tool memcheck
--error-exitcode 7 python tools/sanitize_step.py [--select exact] [--wire f16] [--sgd]."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import gradgen  # noqa: E402
import paper_2010_10458_b200 as tk  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=100_003)
    ap.add_argument("--rho", type=float, default=0.01)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--select", default="mstopk")
    ap.add_argument("--wire", default="f32")
    ap.add_argument("--sgd", action="store_true")
    a = ap.parse_args()
    ctx = tk.Context(a.d, rho=a.rho, seed=1, select=a.select, wire=a.wire)
    r = torch.zeros(a.d, device="cuda")
    w = torch.zeros(a.d, device="cuda")
    for step in range(a.steps):
        g = torch.from_numpy(gradgen.gradient(a.d, "L", cfg=7, step=step)).cuda()
        if a.sgd:
            ctx.step_sgd(g, r, w, 0.1)
        else:
            ctx.step(g, r)
    torch.cuda.synchronize()
    print("ok", ctx.launches)
    ctx.close()


if __name__ == "__main__":
    main()
