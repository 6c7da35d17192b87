"""Per-phase cycle breakdown of the persistent AM kernel (clock64 build).

Build the profiling variant first (BMPC_VARIANT=prof python
paper_2109_10392_b200/_build.py), then run:
  python tools/phase_prof.py [--config c1] [--iters 100] [--warps 0]
Cycles are summed over warps (lane 0 of each) and reported per warp and
sweep; they include the time the warp waits for its SMSP, so they are the
wall share of each phase, not its issue cost.
"""
import argparse
import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
os.environ.setdefault("BMPC_LIB", str(ROOT / "paper_2109_10392_b200/_lib/libbatchmpc_b200_prof.so"))

import torch  # noqa: E402

from paper_2109_10392_b200 import _native as nat  # noqa: E402
from paper_2109_10392_b200 import device as D  # noqa: E402
from paper_2109_10392_b200 import make_solver  # noqa: E402
from paper_2109_10392_b200.scenes import CONFIGS, make_workload  # noqa: E402

PHASES = ["init", "xy_qp", "passA", "unwrap+pth", "psi_qp", "obst:slots", "G_reduce", "lam+res",
          "score", "outputs", "obst:xy", "obst:loop", "passB", "obst:contract"]

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
ap.add_argument("--iters", type=int, default=0)
ap.add_argument("--warps", type=int, default=0)
ap.add_argument("--l", type=int, default=None)
ap.add_argument("--scenes", type=int, default=None)
ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32"])
args = ap.parse_args()

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
ps = prob.c_struct()
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
lib = nat.load()
rd = getattr(lib, f"bmpc_phase_prof_nb{solver.basis.n_b}")
rd.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
buf = (ctypes.c_ulonglong * 20)()
for rep in range(2):  # warm-up, then measured
    assert rd(buf, 1) == 0
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    nat.check(lib.bmpc_sweeps(ctx, ctypes.byref(ps), ctypes.byref(opts), iters, 0, 0, None, 0,
                              ctypes.byref(out), sp))
    b.record()
    torch.cuda.synchronize()
assert rd(buf, 0) == 0
ms = a.elapsed_time(b)
tot = sum(buf[i] for i in range(len(PHASES)))
per = W.L * iters
print(f"{args.config} L={W.L} iters={iters} launch {ms:.3f} ms (profiling build)")
for i, name in enumerate(PHASES):
    print(f"  {name:12s} {buf[i] / per:10.1f} cycles/warp/sweep  {100.0 * buf[i] / tot:5.1f}%")
print(f"  {'total':12s} {tot / per:10.1f}")
if buf[14]:
    print(f"  obstacle slots tested {buf[14] / per:.2f} per warp-sweep, skipped {100.0 * buf[15] / buf[14]:.1f}%, "
          f"failed with a never-skip sample {100.0 * buf[16] / buf[14]:.1f}%, failing samples per warp-sweep {buf[17] / per:.2f}")
