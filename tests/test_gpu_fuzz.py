"""Randomised parity sweep: many seeded scenes with aggressive goals (lane
changes across all four lanes, speed changes that clip the acceleration,
obstacles spawned on the ego's path, reversing egos whose headings wrap past
+-pi) against the oracle.  Every stable column within 1e-8, every scoring
index identical.  Exercises the rare paths of the kernel: inside-ellipse
corrections, clipped-acceleration corrections and the serial unwrap."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _random_scene(rng, n, t_f, m, l):
    times = np.linspace(0.0, t_f, n)
    lanes = np.array([-5.25, -1.75, 1.75, 5.25])
    reverse = rng.random() < 0.25
    v0 = rng.uniform(-8.0, -2.0) if reverse else rng.uniform(5.0, 30.0)
    x0 = rng.uniform(-40.0, 80.0, m)
    vx = rng.uniform(-5.0, 30.0, m)
    xi_x = (x0[:, None] + vx[:, None] * times[None, :]).ravel()
    xi_y = np.repeat(rng.choice(lanes, m), n).astype(np.float64)
    y_ego = rng.choice(lanes)
    vg = rng.uniform(-10.0, 0.0, l) if reverse else rng.uniform(0.0, 40.0, l)
    b_xy = np.zeros((12, l))
    b_xy[1], b_xy[3], b_xy[4] = v0, vg * t_f, vg
    b_xy[6], b_xy[9] = y_ego, rng.uniform(-6.0, 6.0, l)
    b_xy[2] = rng.normal(0, 2.0)   # initial acceleration
    b_psi = np.zeros((4, l))
    b_psi[0] = np.pi if reverse else 0.0
    return xi_x, xi_y, b_xy, b_psi


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_parity(cuda, seed):
    import am_oracle as O

    from paper_2109_10392_b200 import ProblemBatch, make_solver
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    rng = np.random.default_rng(1000 + seed)
    n, t_f, degree, m, l, iters = 100, 5.0, 10, int(rng.integers(3, 25)), 32, 80
    xi_x, xi_y, b_xy, b_psi = _random_scene(rng, n, t_f, m, l)
    a, b, v_min, v_max, a_max = 5.6, 2.4, 0.1, 35.0, 8.0
    o = O.OracleSolver(n, t_f, degree, m)
    ref = o.solve(xi_x, xi_y, b_xy, b_psi, a, b, v_min, v_max, a_max, max_iter=iters)
    scr = o.solve(xi_x * (1 + 2.2e-16), xi_y, b_xy, b_psi, a, b, v_min, v_max, a_max, max_iter=iters)
    P = o.P
    div = np.zeros(l)
    for k in ("c_x", "c_y", "c_psi"):
        tr = P @ ref[k]
        div = np.maximum(div, np.abs(P @ scr[k] - tr).max(axis=0) / np.maximum(1.0, np.abs(tr).max(axis=0)))
    stable = div <= 1e-10

    solver = make_solver(n, t_f, degree, m)

    class Sc:
        pass

    sc = Sc()
    sc.xi_x, sc.xi_y, sc.b_xy, sc.b_psi, sc.l, sc.S = xi_x[None], xi_y[None], b_xy, b_psi, l, 1
    sc.a, sc.b, sc.v_min, sc.v_max, sc.a_max = a, b, v_min, v_max, a_max
    spec = MetaCostSpec("cruise", v_cruise=20.0)
    res = plan_batch(solver, sc, max_iter=iters, tol=0.0, spec=spec, limits=FilterLimits())
    err = np.zeros(l)
    for k in ("c_x", "c_y", "c_psi"):
        tr = P @ ref[k]
        err = np.maximum(err, np.abs(P @ getattr(res, k) - tr).max(axis=0) / np.maximum(1.0, np.abs(tr).max(axis=0)))
    print(f"seed {seed} m={m}: stable {stable.sum()}/{l}, max rel err {err[stable].max() if stable.any() else 0:.2e}")
    if stable.any():
        assert err[stable].max() <= 1e-8
    # scoring, column by column on the screen-stable columns: meta cost and the
    # feasibility flag of each, and the argmins restricted to those columns
    # (recomputed from our per-column outputs with numpy's tie rule) -- checked
    # on every seed, also when some other column is ill-posed
    sref = o.score(ref, xi_x, xi_y, a, b, kind="cruise", v_cruise=20.0)
    if stable.any():
        idx = np.flatnonzero(stable)
        np.testing.assert_allclose(res.meta_cost[idx], sref["meta_cost"][idx], rtol=1e-8, atol=1e-10)
        np.testing.assert_array_equal(res.feasible[idx], sref["feasible"][idx])
        ours = np.where(res.feasible[idx], res.meta_cost[idx], np.inf)
        theirs = np.where(sref["feasible"][idx], sref["meta_cost"][idx], np.inf)
        if np.isfinite(theirs).any():
            assert int(np.argmin(ours)) == int(np.argmin(theirs))
        assert int(np.argmin(res.meta_cost[idx])) == int(np.argmin(sref["meta_cost"][idx]))
    if stable.all():  # the indices over all columns are only well-posed when every column is
        assert (res.best_index[0] if res.best_index[0] is not None else -1) == (
            sref["best_index"] if sref["best_index"] is not None else -1)
        assert int(res.argmin_all[0]) == int(sref["argmin_all"])
