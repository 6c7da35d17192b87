"""Find BASELINE-generator scenes whose reference solve has feasible candidates.

Runs the REFERENCE (build container only, like make_golden.py): for each seed,
the full goal batch of a config is solved with the reference's BatchSolver
(compiled kernels from oracle/_ref, 1 BLAS thread per process) and scored with
its filter_candidates/rank.  Prints, per seed, the feasible column indices and
the best index.  make_golden.py then builds the c3f/c4f fixtures from the
seeds and columns found here (columns are independent, so a fixture may hold a
subset of a scene's goal columns).

    python tests/golden/seed_search.py c3 0 32
"""

from __future__ import annotations

import json
import sys
from multiprocessing import Pool
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def _one(args):
    name, seed, l = args
    import make_golden as G  # noqa: F401  (registers the compiled backend)
    from paper_2109_10392_b200.scenes import CONFIGS, make_workload

    from batchmpc.planner import MetaCostSpec

    cfg = CONFIGS[name]
    W = make_workload(name, scenes=1, l=l, seed0=seed)
    solver = G.ref_solver(W.n, W.t_f, W.degree, W.m)
    from batchmpc.solver import ProblemBatch

    batch = ProblemBatch(l=W.l, xi_x=W.xi_x[0], xi_y=W.xi_y[0], a=W.a, b=W.b, v_min=W.v_min,
                         v_max=W.v_max, a_max=W.a_max, b_xy=W.b_xy, b_psi=W.b_psi)
    st, info = solver.solve(batch, max_iter=cfg.iters, tol=0.0)
    sc = G.score(solver, st, info, batch, MetaCostSpec("cruise", v_cruise=20.0))
    feas = [int(i) for i in (sc["feasible"] > 0).nonzero()[0]]
    return dict(seed=seed, feasible=feas, best=int(sc["best_index"]), argmin_hc=int(sc["argmin_hc"]))


def main():
    name, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    l = int(sys.argv[4]) if len(sys.argv) > 4 else None
    from paper_2109_10392_b200.scenes import CONFIGS

    l = CONFIGS[name].l if l is None else l
    with Pool(8) as p:
        for r in p.imap_unordered(_one, [(name, s, l) for s in range(lo, hi)]):
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
