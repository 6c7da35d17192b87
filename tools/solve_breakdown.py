"""Where BatchSolver.solve's end-to-end time goes (pageable numpy in, host
coefficients out): problem upload, the solve call, the copy back, the last
history row.  Usage: solve_breakdown.py [--config c1]"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_10392_b200 import make_solver  # noqa: E402
from paper_2109_10392_b200.scenes import CONFIGS, make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
W = make_workload(args.config)
iters = CONFIGS[args.config].iters
solver = make_solver(W.n, W.t_f, W.degree, W.m)


def timeit(fn, reps=args.reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return float(np.median(ts))


def full():
    st, info = solver.solve(W, max_iter=iters, tol=0.0)
    return st.c_x, info.residual_history[-1]


prob = solver._problem(W)
sol = solver.solve_device(prob, iters, 0.0)
print(f"{args.config}: solve + c_x + history[-1] {timeit(full):.3f} ms | _problem (upload) "
      f"{timeit(lambda: solver._problem(W)):.3f} | solve_device {timeit(lambda: solver.solve_device(prob, iters, 0.0)):.3f} | "
      f"block D2H {timeit(lambda: sol.block.cpu().numpy()):.3f} | solve_device want_v=False "
      f"{timeit(lambda: solver.solve_device(prob, iters, 0.0, want_v=False)):.3f}")
