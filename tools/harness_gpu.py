"""The reference's OWN closed-loop harness driving this package's GPU solver
(INTEGRATION.md section 2).

Runs the reference package shipped by build() in oracle/_ref/pkg (its sources,
its compiled kernels, its TOML configs) with exactly one change: the planner's
``solver`` attribute is this package's BatchSolver built from the planner's own
basis and constant matrices -- the one-line swap INTEGRATION.md documents.  The
harness itself (IDM traffic world, goal sampling, warm starts, filtering,
ranking, control, logs) is the reference's code, unmodified.

    python tools/harness_gpu.py OUTDIR [--config cruise_idm] [--duration 5]
        [--sizes 4,11,22,44,110,1024] [--cycles 10] [--cpu]

Writes OUTDIR/{run.jsonl, times.csv, summary.json} of one run_scenario and
OUTDIR/timing.csv of bench_batch (the reference's own formats,
harness.py:425-473, :602-606); --cpu runs the same with the reference's own
solver for comparison.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "oracle" / "_ref" / "pkg"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(REF))

from threadpoolctl import threadpool_limits  # noqa: E402

import batchmpc.harness as H  # noqa: E402  (the reference's harness)

from paper_2109_10392_b200.solver import BatchSolver as GpuSolver  # noqa: E402


def gpu_planner_class(base):
    class GpuPlanner(base):
        """The reference Planner with its solver swapped for the sm_100a one."""

        def __init__(self, *a, **k):
            super().__init__(*a, **k)
            self.solver = GpuSolver(self.basis, self.mats, self.cfg.rho_xy)

    return GpuPlanner


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("out")
    ap.add_argument("--config", default="cruise_idm")
    ap.add_argument("--duration", type=float, default=5.0)
    ap.add_argument("--sizes", default="4,11,22,44,110,1024")
    ap.add_argument("--cycles", type=int, default=10)
    ap.add_argument("--cpu", action="store_true", help="keep the reference's own CPU solver")
    args = ap.parse_args()
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    threadpool_limits(1)
    if not args.cpu:
        H.Planner = gpu_planner_class(H.Planner)
    cfg = H.load_config(str(REF / "configs" / f"{args.config}.toml"))
    cfg.duration = args.duration
    t0 = time.perf_counter()
    log = H.run_scenario(cfg)
    wall = time.perf_counter() - t0
    H.write_log(log, out)  # run.jsonl, times.csv, summary.json (harness.py:429-448)
    (out / "driver.json").write_text(json.dumps({
        "wall_s": wall, "config": args.config, "duration_s": args.duration,
        "solver": "reference CPU (its own)" if args.cpu else "paper_2109_10392_b200 BatchSolver (sm_100a)"},
        indent=1))
    rows = H.bench_batch(cfg, [int(s) for s in args.sizes.split(",")], cycles=args.cycles)
    H.write_timing_csv(rows, out / "timing.csv")
    print(json.dumps({"run_wall_s": wall, "cycles": len(log.records),
                      "mean_solve_ms": 1e3 * sum(log.solve_times) / len(log.solve_times),
                      "fallbacks": sum(1 for r in log.records if r["fallback"]), "timing": rows}))


if __name__ == "__main__":
    main()
