"""Minimal driver for ncu: one warm-up + one timed launch of the persistent AM
kernel on a BASELINE config (default c1).  Usage:
  python tools/profile_solve.py [--config c1] [--iters 100] [--scenes S] [--l L]
  ncu --set full --clock-control none --import-source on -k regex:am_solve -s 1 -c 1 \
      -o gpurun_out/prof python tools/profile_solve.py
"""
import argparse
import ctypes
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2109_10392_b200 import _native as nat  # noqa: E402
from paper_2109_10392_b200 import device as D  # noqa: E402
from paper_2109_10392_b200 import make_solver  # noqa: E402
from paper_2109_10392_b200.scenes import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--scenes", type=int, default=None)
ap.add_argument("--l", type=int, default=None)
ap.add_argument("--warps", type=int, default=0)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
args = ap.parse_args()

from paper_2109_10392_b200.scenes import CONFIGS  # noqa: E402

cfg = CONFIGS[args.config]
W = make_workload(args.config, scenes=args.scenes, l=args.l)
iters = args.iters or cfg.iters
solver = make_solver(W.n, W.t_f, W.degree, W.m)
ctx = solver._context()
dev = torch.device("cuda", 0)
prob = D.DeviceProblem.from_host(W.n, W.xi_x, W.xi_y, W.b_xy, W.b_psi, W.l, W.a, W.b, W.v_min,
                                 W.v_max, W.a_max, device=dev)
sol = D.alloc_solution(solver.basis.n_b, W.n, W.L, iters, False, dev)
opts = nat.SolveOpts(max_iter=iters, tol=0.0, warps_per_block=args.warps,
                     precision=1 if args.precision == "fp32" else 0)
out = D.solution_struct(sol)
out.history = None  # the plan path does not write the residual history either
ps = prob.c_struct()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
lib = nat.load()
times = []
for r in range(1 + args.reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    nat.check(lib.bmpc_sweeps(ctx, ctypes.byref(ps), ctypes.byref(opts), iters, 0, 0, None, 0,
                              ctypes.byref(out), sp))
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b))
print(f"{args.config} L={W.L} iters={iters}: launch ms {['%.3f' % t for t in times]}")
