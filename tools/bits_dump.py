"""Dump solve outputs (bits) for library A/B comparisons.
Usage: BMPC_LIB=... [PREC=fp32] python tools/bits_dump.py NAME OUT.npz [team_warps] [tol]"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2109_10392_b200 import device as D  # noqa: E402
from paper_2109_10392_b200 import make_solver  # noqa: E402

name, out = sys.argv[1], sys.argv[2]
team = int(sys.argv[3]) if len(sys.argv) > 3 else 0
tol = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
z = dict(np.load(ROOT / "tests" / "golden" / f"{name}.npz"))
solver = make_solver(int(z["n"]), float(z["t_f"]), int(z["degree"]), int(z["m"]))
xi_x, xi_y = np.atleast_2d(z["xi_x"]), np.atleast_2d(z["xi_y"])
prob = D.DeviceProblem.from_host(int(z["n"]), xi_x, xi_y, z["b_xy"], z["b_psi"], int(z["l"]), float(z["a"]),
                                 float(z["b"]), float(z["v_min"]), float(z["v_max"]), float(z["a_max"]))
sol = solver.solve_device(prob, max_iter=int(z.get("iters", 40)), tol=tol, team_warps=team,
                          precision=os.environ.get("PREC", "fp64"))
np.savez(out, c_x=sol.c_x.cpu().numpy(), c_y=sol.c_y.cpu().numpy(), c_psi=sol.c_psi.cpu().numpy(),
         it=sol.iterations)
print(name, "iterations", sol.iterations)
