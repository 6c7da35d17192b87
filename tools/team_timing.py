"""Kernel time per team size (warps per instance) on BASELINE configs."""
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
from paper_2109_10392_b200.scenes import CONFIGS, make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", nargs="+", default=["c0", "c1"])
ap.add_argument("--teams", nargs="+", type=int, default=[1, 2, 4])
ap.add_argument("--warps", type=int, default=0, help="warps per block (0 = auto)")
a = ap.parse_args()
for cfg_name in a.configs:
    cfg = CONFIGS[cfg_name]
    W = make_workload(cfg_name, scenes=min(cfg.scenes, 8))
    solver = make_solver(W.n, W.t_f, W.degree, W.m)
    ctx = solver._context()
    dev = torch.device("cuda", 0)
    prob = D.DeviceProblem.from_host(W.n, W.xi_x, W.xi_y, W.b_xy, W.b_psi, W.l, W.a, W.b, W.v_min,
                                     W.v_max, W.a_max, device=dev)
    sol = D.alloc_solution(solver.basis.n_b, W.n, W.L, cfg.iters, False, dev)
    out = D.solution_struct(sol)
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for tw in a.teams:
        opts = nat.SolveOpts(max_iter=cfg.iters, tol=0.0, team_warps=tw, warps_per_block=a.warps)
        ts = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nat.check(nat.load().bmpc_sweeps(ctx, ctypes.byref(prob.c_struct()), ctypes.byref(opts),
                                             cfg.iters, 0, 0, None, 0, ctypes.byref(out), sp))
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f"{cfg_name} L={W.L} team={tw}: {min(ts[1:]):.3f} ms")
