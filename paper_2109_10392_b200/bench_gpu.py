"""`bench-gpu` CLI: the reference harness's batch-size timing sweep and run log,
driven by the device MPC cycle.

    python -m paper_2109_10392_b200.bench_gpu --sizes 110 1024 4096 --cycles 30 \
        --out-dir runs/gpu

writes, in the reference's formats (harness.py:582-606, :360-399):
  timing.csv  l,n_solves,mean,min,max   (solve seconds per MPC cycle)
  run.jsonl   one record per cycle of the last size (ego, obstacles, goal lanes,
              meta costs, feasibility, best index, residuals of the chosen
              candidate, command)

Traffic here is constant-velocity (the obstacle states the planner sees are
advanced exactly as its own predictions assume); the reference's IDM /
trace-driven traffic simulation is out of scope.
"""

from __future__ import annotations

import argparse
import csv
import json
import math
from pathlib import Path

import numpy as np

from .planner import EgoState, LaneGeometry, MetaCostSpec, Planner, PlannerConfig
from .traffic import VehicleState


def _kinematics(ego: EgoState, accel: float, steering: float, dt: float, h: float) -> EgoState:
    """Unicycle update under (accel, steering) (the harness's ego model)."""
    v = math.hypot(ego.vx, ego.vy)
    psidot = math.tan(steering) * v / h if v > 1e-9 else 0.0
    v1 = max(0.0, v + accel * dt)
    psi1 = ego.psi + psidot * dt
    vx1, vy1 = v1 * math.cos(psi1), v1 * math.sin(psi1)
    return EgoState(x=ego.x + vx1 * dt, y=ego.y + vy1 * dt, psi=psi1, psidot=psidot, vx=vx1, vy=vy1,
                    ax=(vx1 - ego.vx) / dt, ay=(vy1 - ego.vy) / dt)


def _scene(rng, lanes: LaneGeometry, n_vehicles: int):
    c = lanes.centers
    ego = EgoState(x=0.0, y=float(c[rng.integers(len(c))]), vx=float(rng.uniform(15, 25)))
    veh = [VehicleState(id=i, x=float(rng.uniform(-30, 120)), y=float(c[rng.integers(len(c))]),
                        vx=float(rng.uniform(10, 25)), vy=0.0, lane=0) for i in range(n_vehicles)]
    return ego, veh


def _r(v, d=9):
    return [round(float(x), d) for x in v]


def run(size: int, cycles: int, seed: int, cfg_kw: dict, records: list | None = None) -> list[float]:
    rng = np.random.default_rng(seed)
    lanes = LaneGeometry(4, 3.5, -5.25)
    cfg = PlannerConfig(l=size, **cfg_kw)
    planner = Planner(cfg, lanes, MetaCostSpec("cruise", v_cruise=20.0))
    planner.solver._context()  # one-time constant upload, like the reference's factorisation in __init__
    ego, veh = _scene(rng, lanes, cfg_kw.get("m", 10))
    times = []
    for cycle in range(cycles):
        res = planner.mpc_cycle(ego, veh)
        times.append(res.solve_time)
        if records is not None:
            plan, hist = res.plan, res.info.residual_history
            best = plan.best_index
            rb = best if best is not None else int(np.argmin(plan.residuals.max_per_instance()))
            records.append({
                "cycle": cycle, "t": round(cycle * cfg.dt_cycle, 9),
                "ego": {k: getattr(ego, k) for k in ("x", "y", "psi", "psidot", "vx", "vy", "ax", "ay")},
                "obstacles": [{"id": v.id, "x": v.x, "y": v.y, "vx": v.vx, "vy": v.vy, "lane": v.lane}
                              for v in veh],
                "goal_lanes": [g.lane for g in plan.goals],
                "meta_costs": _r(plan.meta_cost), "feasible": [bool(f) for f in plan.feasible],
                "min_ratio": _r(plan.min_ratio), "heading_max": _r(plan.heading_max),
                "best_index": best, "fallback": res.fallback, "converged": bool(res.info.converged),
                "residual_iters": int(res.info.iterations),
                "residuals_best": {"obs": _r([h.r_obs[rb] for h in hist]),
                                   "acc": _r([h.r_acc[rb] for h in hist]),
                                   "nonhol": _r([h.r_nonhol[rb] for h in hist])},
                "command": {"accel": res.command.accel, "steering": res.command.steering},
            })
        ego = _kinematics(ego, res.command.accel, res.command.steering, cfg.dt_cycle, cfg.h)
        veh = [VehicleState(id=v.id, x=v.x + v.vx * cfg.dt_cycle, y=v.y + v.vy * cfg.dt_cycle, vx=v.vx,
                            vy=v.vy, lane=v.lane) for v in veh]
    return times


def main(argv=None) -> None:
    ap = argparse.ArgumentParser(prog="bench-gpu", description=__doc__.split("\n\n")[0])
    ap.add_argument("--sizes", type=int, nargs="+", default=[110, 1024])
    ap.add_argument("--cycles", type=int, default=30)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-iter", type=int, default=100)
    ap.add_argument("--tol", type=float, default=1e-3)
    ap.add_argument("--out-dir", default="runs/gpu")
    a = ap.parse_args(argv)
    out = Path(a.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    cfg_kw = dict(t_f=5.0, max_iter=a.max_iter, tol=a.tol, m=10, b=2.4, v_max=35.0)
    rows, records = [], []
    for i, size in enumerate(a.sizes):
        t = np.array(run(size, a.cycles, a.seed, cfg_kw, records if i == len(a.sizes) - 1 else None))
        rows.append({"l": size, "n_solves": len(t), "mean": float(t.mean()), "min": float(t.min()),
                     "max": float(t.max())})
        print(f"l={size}: {len(t)} solves, mean {t.mean() * 1e3:.3f} ms, min {t.min() * 1e3:.3f} ms")
    with open(out / "timing.csv", "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=["l", "n_solves", "mean", "min", "max"])
        w.writeheader()
        w.writerows(rows)
    with open(out / "run.jsonl", "w") as fh:
        for r in records:
            fh.write(json.dumps(r, sort_keys=True, separators=(",", ":"), allow_nan=False) + "\n")


if __name__ == "__main__":
    main()
