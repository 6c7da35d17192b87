"""Small solves for compute-sanitizer (racecheck / synccheck / memcheck): every
kernel variant on a short run -- 4-warp teams (c0), one warp per instance with
staged predictions (c1 subset), culling (c2f, m = 30), long horizon (c4f,
n = 200, n_b = 16), the polled early exit (tol > 0), fused scoring + argmin."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2109_10392_b200 import device as D  # noqa: E402
from paper_2109_10392_b200 import make_solver  # noqa: E402
from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch  # noqa: E402


class _S:
    def __init__(self, z, l=None):
        L0 = int(z["l"])
        l = l or L0
        S = np.atleast_2d(z["xi_x"]).shape[0]
        self.xi_x, self.xi_y = np.atleast_2d(z["xi_x"]), np.atleast_2d(z["xi_y"])
        cols = np.concatenate([np.arange(s * L0, s * L0 + l) for s in range(S)])
        self.b_xy, self.b_psi = np.ascontiguousarray(z["b_xy"][:, cols]), np.ascontiguousarray(z["b_psi"][:, cols])
        self.l, self.S = l, S
        self.a, self.b = float(z["a"]), float(z["b"])
        self.v_min, self.v_max, self.a_max = float(z["v_min"]), float(z["v_max"]), float(z["a_max"])


def run(name, iters, team=0, l=None, tol=0.0):
    z = dict(np.load(ROOT / "tests" / "golden" / f"{name}.npz"))
    solver = make_solver(int(z["n"]), float(z["t_f"]), int(z["degree"]), int(z["m"]))
    S = _S(z, l)
    prob = D.DeviceProblem.from_host(int(z["n"]), S.xi_x, S.xi_y, S.b_xy, S.b_psi, S.l, S.a, S.b, S.v_min,
                                     S.v_max, S.a_max)
    sol = solver.solve_device(prob, max_iter=iters, tol=tol, team_warps=team)
    res = plan_batch(solver, S, max_iter=iters, tol=tol, spec=MetaCostSpec("cruise", v_cruise=20.0),
                     limits=FilterLimits())
    torch.cuda.synchronize()
    print(f"{name} team={team} l={S.l} iters={sol.iterations} best={res.best_index}", flush=True)


run("c0", 8, team=4, l=16)
run("c0", 8, team=2, l=16)
run("c1", 8, l=256)
run("c2f", 6, l=64)
run("c4f", 4, l=16)
run("demo", 60, tol=3.0)          # polled early exit (team build, one warp per instance)
run("demo", 60, team=4, tol=3.0)  # polled early exit in 4-warp teams
print("sanitize drive done")
