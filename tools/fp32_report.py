"""fp32 mode accuracy report (under gpurun): every golden fixture solved in
fp64 and fp32 mode; per fixture the max / median relative trajectory error of
each mode against the reference on its screen-stable columns, the fp32 error
against our own fp64 solve, and whether the best / argmin indices agree.
Usage: python tools/fp32_report.py [names...]"""

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from test_gpu_solver import SCREEN, _plan, _Scenes, _solver, traj_err  # noqa: E402

from conftest import golden  # noqa: E402


def run(name):
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    z = golden(name)
    solver = _solver(z)
    out = {}
    for prec in ("fp64", "fp32"):
        out[prec] = plan_batch(solver, _Scenes(z), max_iter=int(z["iters"]), tol=0.0,
                               spec=MetaCostSpec("cruise", v_cruise=20.0), limits=FilterLimits(),
                               precision=prec)
    P = solver.basis.P
    stable = z["screen_div"] <= SCREEN
    g = lambda r: dict(c_x=r.c_x, c_y=r.c_y, c_psi=r.c_psi)  # noqa: E731
    e64 = traj_err(P, g(out["fp64"]), z)
    e32 = traj_err(P, g(out["fp32"]), z)
    e3264 = traj_err(P, g(out["fp32"]), g(out["fp64"]))
    same = lambda a, b: [int(x if x is not None else -1) for x in a] == [int(x if x is not None else -1) for x in b]  # noqa: E731
    print(f"{name}: stable {stable.sum()}/{stable.size} | fp64 max {e64[stable].max():.2e} | "
          f"fp32 max {e32[stable].max():.2e} med {np.median(e32[stable]):.2e} "
          f"(all cols max {e32.max():.2e}) | fp32 vs fp64 max {e3264.max():.2e} | "
          f"best {out['fp32'].best_index} vs ref {list(z['cruise_best_index'])} "
          f"same {same(out['fp32'].best_index, z['cruise_best_index'])} "
          f"argmin_all same {same(out['fp32'].argmin_all, z['cruise_argmin_all'])} "
          f"feasible agree {np.mean(out['fp32'].feasible == z['cruise_feasible'].astype(bool)):.4f} "
          f"res_final max rel {np.max(np.abs(out['fp32'].res_final - z['res_final']) / np.maximum(1e-9, np.abs(z['res_final']))):.2e}",
          flush=True)


if __name__ == "__main__":
    import torch

    torch.cuda.set_device(0)
    for n in sys.argv[1:] or ["c0", "c1", "c2s", "c2f", "c3s", "c3f", "c4s", "c4f", "reverse"]:
        run(n)
