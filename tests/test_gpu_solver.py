"""Parity of the persistent sm_100a AM solver + fused scoring with the
reference, on the golden fixtures produced by running the reference itself.

Contract: fp64 trajectories x, y, psi within 1e-8
relative (max_k |gpu - ref| / max(1, max_k |ref|)) on every column the
reference's own 1-ulp self-sensitivity screen marks stable (divergence <= 1e-10);
identical best index, identical unfiltered and heading+collision argmins, and
meta costs within 1e-8 relative on stable columns.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

TRAJ_TOL = 1e-8
SCREEN = 1e-10


def _solver(z):
    from paper_2109_10392_b200 import make_solver

    return make_solver(int(z["n"]), float(z["t_f"]), int(z["degree"]), int(z["m"]))


class _Scenes:
    def __init__(self, z):
        self.xi_x, self.xi_y = np.atleast_2d(z["xi_x"]), np.atleast_2d(z["xi_y"])
        self.b_xy, self.b_psi = z["b_xy"], z["b_psi"]
        self.l, self.S = int(z["l"]), self.xi_x.shape[0]
        self.a, self.b = float(z["a"]), float(z["b"])
        self.v_min, self.v_max, self.a_max = float(z["v_min"]), float(z["v_max"]), float(z["a_max"])


def traj_err(P, got, ref):
    err = np.zeros(got["c_x"].shape[1])
    for k in ("c_x", "c_y", "c_psi"):
        tr, tg = P @ ref[k], P @ got[k]
        scale = np.maximum(1.0, np.abs(tr).max(axis=0))
        err = np.maximum(err, np.abs(tg - tr).max(axis=0) / scale)
    return err


def _plan(z, kind="cruise"):
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    solver = _solver(z)
    spec = (MetaCostSpec("cruise", v_cruise=20.0) if kind == "cruise"
            else MetaCostSpec("highspeed", v_max=25.0, y_rl=-5.25, w1=1.0, w2=0.1))
    res = plan_batch(solver, _Scenes(z), max_iter=int(z["iters"]), tol=0.0, spec=spec,
                     limits=FilterLimits())
    return solver, res


PARITY = ["c0", "c1", "c2s", "c2f", "c3s", "c3f", "c4s", "c4f", "reverse"]
# fixtures whose every scene has a feasible candidate: best_index is a real
# index on both sides (c2f / c3f / c4f, tests/golden/seed_search.py)
FEASIBLE = ["c2f", "c3f", "c4f"]


@pytest.mark.parametrize("name", PARITY)
def test_solve_and_score_parity(cuda, name):
    z = golden(name)
    solver, res = _plan(z)
    got = dict(c_x=res.c_x, c_y=res.c_y, c_psi=res.c_psi)
    err = traj_err(solver.basis.P, got, z)
    stable = z["screen_div"] <= SCREEN
    print(f"{name}: stable {stable.sum()}/{stable.size}, max rel traj err {err[stable].max():.3e}")
    assert err[stable].max() <= TRAJ_TOL
    assert res.iterations == int(z["iters"])
    np.testing.assert_allclose(res.res_final[:, stable], z["res_final"][:, stable], rtol=1e-6, atol=1e-9)
    l = int(z["l"])
    for s in range(int(z["S"])):
        assert (res.best_index[s] if res.best_index[s] is not None else -1) == int(z["cruise_best_index"][s])
        assert int(res.argmin_all[s]) == int(z["cruise_argmin_all"][s])
        assert int(res.argmin_hc[s]) == int(z["cruise_argmin_hc"][s])
    mc = z["cruise_meta_cost"]
    rel = np.abs(res.meta_cost - mc) / np.maximum(1.0, np.abs(mc))
    assert rel[stable].max() <= 1e-8
    np.testing.assert_array_equal(res.feasible[stable], z["cruise_feasible"][stable].astype(bool))
    np.testing.assert_allclose(res.min_ratio[stable], z["cruise_min_ratio"][stable], rtol=1e-8)
    np.testing.assert_allclose(res.heading_max[stable], z["cruise_heading_max"][stable], rtol=1e-7,
                               atol=1e-12)
    if name in FEASIBLE:
        assert all(b is not None for b in res.best_index), res.best_index
    del l


# fp32 mode (precision="fp32": the per-sample passes in single precision, the
# QP steps / Gram terms / multipliers in fp64): stated tolerance 5e-5 relative
# trajectory error; measured on B200 <= 1.2e-5 (c4s), <= 4.4e-6 elsewhere
# (tools/fp32_report.py).
FP32_TOL = 5e-5


@pytest.mark.parametrize("name", ["c0", "c1", "c2s", "c2f", "c3s", "c3f", "c4s", "c4f", "reverse"])
def test_fp32_mode_tolerance(cuda, name):
    """fp32 mode against the reference: the stated tolerance on stable
    columns, and the same best / unfiltered / heading+collision argmin indices
    and feasibility as the reference's fp64 solve (measured identical on every
    fixture); reported separately, not bit-compatible."""
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    z = golden(name)
    solver = _solver(z)
    res = plan_batch(solver, _Scenes(z), max_iter=int(z["iters"]), tol=0.0,
                     spec=MetaCostSpec("cruise", v_cruise=20.0), limits=FilterLimits(),
                     precision="fp32")
    err = traj_err(solver.basis.P, dict(c_x=res.c_x, c_y=res.c_y, c_psi=res.c_psi), z)
    stable = z["screen_div"] <= SCREEN
    print(f"fp32 {name}: max rel traj err {err[stable].max():.3e} median {np.median(err[stable]):.3e}")
    assert err[stable].max() <= FP32_TOL
    for s in range(int(z["S"])):
        assert (res.best_index[s] if res.best_index[s] is not None else -1) == int(z["cruise_best_index"][s])
        assert int(res.argmin_all[s]) == int(z["cruise_argmin_all"][s])
        assert int(res.argmin_hc[s]) == int(z["cruise_argmin_hc"][s])
    np.testing.assert_array_equal(res.feasible, z["cruise_feasible"].astype(bool))


@pytest.mark.parametrize("name", ["c0", "c2f", "c3s", "c3f", "c4f"])
def test_highspeed_scoring_parity(cuda, name):
    z = golden(name)
    _, res = _plan(z, "highspeed")
    if name in FEASIBLE:
        assert all(b is not None for b in res.best_index)
    for s in range(int(z["S"])):
        assert (res.best_index[s] if res.best_index[s] is not None else -1) == int(z["highspeed_best_index"][s])
        assert int(res.argmin_all[s]) == int(z["highspeed_argmin_all"][s])
    stable = z["screen_div"] <= SCREEN
    mc = z["highspeed_meta_cost"]
    assert (np.abs(res.meta_cost - mc) / np.maximum(1.0, np.abs(mc)))[stable].max() <= 1e-8


def _batch(z, cols=None, s=0):
    from paper_2109_10392_b200 import ProblemBatch

    l = int(z["l"])
    cols = cols if cols is not None else slice(s * l, (s + 1) * l)
    bx, bp = z["b_xy"][:, cols], z["b_psi"][:, cols]
    xi_x = np.atleast_2d(z["xi_x"])[s]
    xi_y = np.atleast_2d(z["xi_y"])[s]
    return ProblemBatch(l=bx.shape[1], xi_x=xi_x, xi_y=xi_y, a=float(z["a"]), b=float(z["b"]),
                        v_min=float(z["v_min"]), v_max=float(z["v_max"]), a_max=float(z["a_max"]),
                        b_xy=np.ascontiguousarray(bx), b_psi=np.ascontiguousarray(bp))


def test_demo_reference_api(cuda):
    """BatchSolver.solve through the reference-shaped API (demo batch, 80 sweeps):
    the reference's own cross-backend bars (tests/test_kernels.py:115-130) and
    the tighter 1e-8 trajectory contract."""
    z = golden("demo")
    solver = _solver(z)
    state, info = solver.solve(_batch(z), max_iter=80, tol=0.0)
    assert info.iterations == 80 and not info.converged
    scale = max(1.0, np.abs(z["c_x"]).max())
    assert np.abs(state.c_x - z["c_x"]).max() <= 1e-7 * scale
    assert np.abs(state.c_psi - z["c_psi"]).max() <= 1e-7
    err = traj_err(solver.basis.P, dict(c_x=state.c_x, c_y=state.c_y, c_psi=state.c_psi), z)
    assert err.max() <= TRAJ_TOL
    hist = np.stack([[h.r_obs, h.r_acc, h.r_nonhol] for h in info.residual_history])
    np.testing.assert_allclose(hist[-1], z["history"][-1], rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(hist, z["history"], rtol=1e-6, atol=1e-9)
    for k in ("v", "d_a", "d", "lambda_x", "lambda_y", "lambda_psi"):
        ref = z[k]
        assert np.abs(getattr(state, k) - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max()), k
    # The angles are ill-posed where their vectors vanish or sit on the branch
    # cut: alpha_a = atan2(yddot, xddot) at the pinned zero-acceleration samples,
    # alpha = atan2(a wy, b wx) at +-pi when a trajectory runs exactly along an
    # obstacle's lane (wy = +-0).  Compare the well-posed targets d*(cos, sin).
    for ang, mag in (("alpha_a", "d_a"), ("alpha", "d")):
        for f in (np.cos, np.sin):
            got = getattr(state, mag) * f(getattr(state, ang))
            ref = z[mag] * f(z[ang])
            assert np.abs(got - ref).max() <= 1e-6 * max(1.0, np.abs(ref).max()), ang
    assert state.alpha.shape == (1000, 11) and state.iteration == 80
    assert solver.kkt.n_factorizations == 2 and solver.kkt.n_solves == 2 * 80


def test_batch_vs_sequential_bitwise(cuda):
    z = golden("c0")
    solver = _solver(z)
    full, _ = solver.solve(_batch(z), max_iter=40, tol=0.0)
    for i in (0, 7, 55, 109):
        one, _ = solver.solve(_batch(z, cols=slice(i, i + 1)), max_iter=40, tol=0.0)
        for k in ("c_x", "c_y", "c_psi", "lambda_x", "lambda_y", "lambda_psi", "v"):
            np.testing.assert_array_equal(getattr(one, k)[:, 0], getattr(full, k)[:, i])


def test_permutation_and_identical_columns_bitwise(cuda, rng):
    z = golden("c0")
    solver = _solver(z)
    b = _batch(z)
    perm = rng.permutation(b.l)
    pb = _batch(z, cols=perm)
    s1, _ = solver.solve(b, max_iter=30, tol=0.0)
    s2, _ = solver.solve(pb, max_iter=30, tol=0.0)
    np.testing.assert_array_equal(s1.c_x[:, perm], s2.c_x)
    np.testing.assert_array_equal(s1.c_psi[:, perm], s2.c_psi)
    same = _batch(z, cols=np.array([3, 3, 3, 3]))
    s3, _ = solver.solve(same, max_iter=30, tol=0.0)
    assert (s3.c_x == s3.c_x[:, :1]).all() and (s3.c_y == s3.c_y[:, :1]).all()


def test_stacked_scenes_equal_single_scene(cuda):
    from paper_2109_10392_b200.planner import plan_batch

    z = golden("c3s")
    solver = _solver(z)
    stacked = plan_batch(solver, _Scenes(z), max_iter=50, tol=0.0)
    l = int(z["l"])
    for s in (1, 3):
        one = plan_batch(solver, _batch(z, s=s), max_iter=50, tol=0.0)
        np.testing.assert_array_equal(one.c_x, stacked.c_x[:, s * l:(s + 1) * l])
        np.testing.assert_array_equal(one.meta_cost, stacked.meta_cost[s * l:(s + 1) * l])


def test_record_iterates_matches_single_launch(cuda):
    z = golden("demo")
    solver = _solver(z)
    s1, i1 = solver.solve(_batch(z), max_iter=12, tol=0.0, record_iterates=True)
    s2, i2 = solver.solve(_batch(z), max_iter=12, tol=0.0)
    np.testing.assert_array_equal(s1.c_x, s2.c_x)
    np.testing.assert_array_equal(s1.lambda_psi, s2.lambda_psi)
    assert len(i1.iterates) == 12
    np.testing.assert_array_equal(i1.iterates[-1][0], s2.c_x)
    ref = z["iter_c_x"]
    for t in (0, 5, 11):
        scale = max(1.0, np.abs(ref[t]).max())
        assert np.abs(i1.iterates[t][0] - ref[t]).max() <= 1e-8 * scale


def test_tol_early_stop_semantics(cuda):
    import am_oracle as O

    z = golden("demo")
    solver = _solver(z)
    b = _batch(z)
    o = O.OracleSolver(100, 10.0, 10, 10)
    full = o.solve(b.xi_x, b.xi_y, b.b_xy, b.b_psi, b.a, b.b, b.v_min, b.v_max, b.a_max, 60)
    worst = full["history"].max(axis=(1, 2))
    t_stop = 20
    tol = float(worst[t_stop]) * (1 + 1e-6)
    expect = int(np.argmax(worst <= tol)) + 1
    state, info = solver.solve(b, max_iter=60, tol=tol)
    assert info.converged and info.iterations == expect == len(info.residual_history)
    state_exact, _ = solver.solve(b, max_iter=expect, tol=0.0)
    np.testing.assert_array_equal(state.c_x, state_exact.c_x)
    _, info2 = solver.solve(b, max_iter=5, tol=-1.0)
    assert info2.iterations == 5 and not info2.converged


@pytest.mark.parametrize("mode", ["fixed", "early", "iterates"])
def test_history_last_row_without_the_table(cuda, mode):
    """residual_history[-1] comes from the final residuals that travel with the
    coefficients; it must equal the last row of the device history table."""
    z = golden("demo")
    solver = _solver(z)
    b = _batch(z)
    tol = 0.0
    if mode == "early":  # a tolerance the 21st sweep meets
        _, full = solver.solve(b, max_iter=30, tol=0.0)
        tol = full.residual_history[20].overall_max() * (1 + 1e-6)
    kw = dict(fixed=dict(max_iter=30, tol=0.0), early=dict(max_iter=60, tol=tol),
              iterates=dict(max_iter=6, tol=0.0, record_iterates=True))[mode]
    _, info = solver.solve(b, **kw)
    hist = info.residual_history
    quick = hist[-1]
    assert hist._rows is None  # the table stayed on the device
    quick2 = hist[info.iterations - 1]
    table = hist[0:len(hist)]  # loads every row
    assert len(table) == info.iterations
    for q in (quick, quick2):
        for f in ("r_obs", "r_acc", "r_nonhol"):
            np.testing.assert_array_equal(getattr(q, f), getattr(table[-1], f))
    if mode == "early":
        assert info.converged and info.iterations <= 21 and quick.overall_max() <= tol


def test_warm_start_keep_multipliers(cuda):
    import am_oracle as O

    z = golden("demo")
    solver = _solver(z)
    b = _batch(z)
    first, _ = solver.solve(b, max_iter=25, tol=0.0)
    o = O.OracleSolver(100, 10.0, 10, 10)
    warm = {k: getattr(first, k) for k in ("c_x", "c_y", "c_psi", "alpha", "d", "alpha_a", "d_a",
                                           "v", "lambda_x", "lambda_y", "lambda_psi")}
    for keep in (False, True):
        ref = o.solve(b.xi_x, b.xi_y, b.b_xy, b.b_psi, b.a, b.b, b.v_min, b.v_max, b.a_max, 20,
                      warm=warm, keep_multipliers=keep)
        st, info = solver.solve(b, max_iter=20, tol=0.0, warm=first, keep_multipliers=keep)
        err = traj_err(solver.basis.P, dict(c_x=st.c_x, c_y=st.c_y, c_psi=st.c_psi), ref)
        assert err.max() <= TRAJ_TOL, (keep, err.max())
    init = solver.init_state(b, warm=first)
    assert (init.lambda_x == 0).all() and init.iteration == 0


def test_cold_init_state_matches_reference(cuda):
    z = golden("demo")
    solver = _solver(z)
    st = solver.init_state(_batch(z))
    import am_oracle as O

    o = O.OracleSolver(100, 10.0, 10, 10)
    b = _batch(z)
    ref = o.init_cold(b.xi_x, b.xi_y, b.b_xy, b.a, b.b, b.v_min, b.v_max, O.kernels("c"))
    np.testing.assert_array_equal(st.c_x, ref["c_x"])
    assert np.abs(st.alpha - ref["alpha"]).max() <= 1e-12
    assert np.abs(st.d - ref["d"]).max() <= 1e-12
    assert (st.lambda_x == 0).all() and st.iteration == 0


def test_solve_validation(cuda):
    z = golden("demo")
    solver = _solver(z)
    with pytest.raises(ValueError):
        solver.solve(_batch(z), max_iter=0)
    first, _ = solver.solve(_batch(z), max_iter=2, tol=0.0)
    first.c_x = first.c_x[:, :-1]
    with pytest.raises(ValueError):
        solver.solve(_batch(z), max_iter=2, warm=first)


def test_smoke_entry(cuda):
    import __graft_entry__

    __graft_entry__.smoke()


@pytest.mark.parametrize("name", ["c3s", "c4s"])
def test_fused_scoring_equals_standalone(cuda, name):
    """bmpc_plan's in-kernel scoring epilogue == bmpc_score on the solved
    coefficients, bit for bit (same shared code, csrc/score.cuh; c3s reads the
    last sweep's stored positions, c4s (n = 200) re-samples them)."""
    import ctypes

    from paper_2109_10392_b200 import _native as nat
    from paper_2109_10392_b200 import device as D
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, _spec_struct

    z = golden(name)
    solver = _solver(z)
    S = _Scenes(z)
    prob = D.DeviceProblem.from_host(int(z["n"]), S.xi_x, S.xi_y, S.b_xy, S.b_psi, S.l, S.a, S.b,
                                     S.v_min, S.v_max, S.a_max)
    spec = _spec_struct(MetaCostSpec("highspeed", v_max=25.0, y_rl=-5.25, w1=1.0, w2=0.1),
                        FilterLimits())
    lib, ctx = nat.load(), solver._context()
    sp = ctypes.c_void_p(D.stream_ptr())
    dev = prob.b_xy.device
    sol = D.alloc_solution(solver.basis.n_b, solver.basis.grid.n, prob.L, 40, False, dev)
    opts = nat.SolveOpts(max_iter=40, tol=0.0)
    fused = D.alloc_score(prob.L, prob.S, dev)
    nat.check(lib.bmpc_plan(ctx, ctypes.byref(prob.c_struct()), ctypes.byref(opts),
                            ctypes.byref(D.solution_struct(sol)), ctypes.byref(spec),
                            ctypes.byref(D.score_struct(fused)), sp))
    alone = D.alloc_score(prob.L, prob.S, dev)
    nat.check(lib.bmpc_score(ctx, ctypes.byref(prob.c_struct()), D.ptr(sol.c_x), D.ptr(sol.c_y),
                             D.ptr(sol.c_psi), D.ptr(sol.res_final), ctypes.byref(spec),
                             ctypes.byref(D.score_struct(alone)), sp))
    for k in ("meta_cost", "min_ratio", "heading_max", "flags", "best_index", "argmin_all",
              "argmin_hc", "n_feasible"):
        assert cuda.equal(getattr(fused, k), getattr(alone, k)), k


@pytest.mark.parametrize("tol_mode", ["none", "early"])
def test_async_plan_matches_sync(cuda, tol_mode):
    """bmpc_plan with status_dev (no host synchronisation; the early-stop re-run
    decided on the device) == the synchronous call, bit for bit, and the
    device status carries {iterations, converged}."""
    import ctypes

    from paper_2109_10392_b200 import _native as nat
    from paper_2109_10392_b200 import device as D
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, _spec_struct

    z = golden("c0")
    solver = _solver(z)
    S = _Scenes(z)
    prob = D.DeviceProblem.from_host(int(z["n"]), S.xi_x, S.xi_y, S.b_xy, S.b_psi, S.l, S.a, S.b,
                                     S.v_min, S.v_max, S.a_max)
    spec = _spec_struct(MetaCostSpec("cruise", v_cruise=20.0), FilterLimits())
    lib, ctx = nat.load(), solver._context()
    sp = ctypes.c_void_p(D.stream_ptr())
    dev = prob.b_xy.device
    tol = 0.0
    if tol_mode == "early":  # a tolerance first met at sweep 25 of 60
        sol = D.alloc_solution(solver.basis.n_b, solver.basis.grid.n, prob.L, 60, False, dev)
        nat.check(lib.bmpc_solve(ctx, ctypes.byref(prob.c_struct()), ctypes.byref(nat.SolveOpts(max_iter=60)),
                                 ctypes.byref(D.solution_struct(sol)), sp))
        worst = sol.history.amax(dim=(1, 2)).cpu().numpy()
        tol = float(worst[24]) * (1 + 1e-9)
    results = []
    for use_async in (False, True):
        sol = D.alloc_solution(solver.basis.n_b, solver.basis.grid.n, prob.L, 60, False, dev)
        sc = D.alloc_score(prob.L, prob.S, dev)
        status = cuda.full((2,), -5, dtype=cuda.int32, device=dev)
        opts = nat.SolveOpts(max_iter=60, tol=tol, status_dev=status.data_ptr() if use_async else None)
        out = D.solution_struct(sol)
        nat.check(lib.bmpc_plan(ctx, ctypes.byref(prob.c_struct()), ctypes.byref(opts), ctypes.byref(out),
                                ctypes.byref(spec), ctypes.byref(D.score_struct(sc)), sp))
        cuda.cuda.synchronize()
        it, conv = (out.iterations, out.converged) if not use_async else tuple(status.cpu().tolist())
        if use_async:
            assert out.iterations == -1
        results.append((it, conv, sol, sc))
    (i0, c0, s0, k0), (i1, c1, s1, k1) = results
    assert (i0, c0) == (i1, c1)
    if tol_mode == "early":
        assert i0 == int(np.argmax(worst <= tol)) + 1 and c0 == 1
    else:
        assert (i0, c0) == (60, 0)
    for k in ("c_x", "c_y", "c_psi", "res_final"):
        assert cuda.equal(getattr(s0, k), getattr(s1, k)), k
    for k in ("meta_cost", "flags", "best_index", "argmin_all", "argmin_hc"):
        assert cuda.equal(getattr(k0, k), getattr(k1, k)), k


@pytest.mark.parametrize("team", [2, 4])
@pytest.mark.parametrize("name", ["c0", "c1", "c3s", "reverse"])
def test_team_parity(cuda, name, team):
    """Teams of 2 or 4 warps per instance (the small-batch latency mode) meet
    the same contract; a fixed team size is bitwise reproducible."""
    from paper_2109_10392_b200 import device as D

    z = golden(name)
    solver = _solver(z)
    S = _Scenes(z)
    prob = D.DeviceProblem.from_host(int(z["n"]), S.xi_x, S.xi_y, S.b_xy, S.b_psi, S.l, S.a, S.b,
                                     S.v_min, S.v_max, S.a_max)
    sol = solver.solve_device(prob, max_iter=int(z["iters"]), tol=0.0, team_warps=team)
    got = {k: getattr(sol, k).cpu().numpy() for k in ("c_x", "c_y", "c_psi")}
    err = traj_err(solver.basis.P, got, z)
    stable = z["screen_div"] <= SCREEN
    print(f"team {team} {name}: max rel traj err {err[stable].max():.3e}")
    assert err[stable].max() <= TRAJ_TOL
    np.testing.assert_allclose(sol.res_final.cpu().numpy()[:, stable], z["res_final"][:, stable],
                               rtol=1e-6, atol=1e-9)
    again = solver.solve_device(prob, max_iter=int(z["iters"]), tol=0.0, team_warps=team)
    assert cuda.equal(again.c_x, sol.c_x) and cuda.equal(again.c_psi, sol.c_psi)


def test_team_validation(cuda):
    """Teams are the fp64, n <= 128 latency mode: other requests fail loudly."""
    from paper_2109_10392_b200 import device as D

    z = golden("c4s")  # n = 200
    solver = _solver(z)
    S = _Scenes(z)
    prob = D.DeviceProblem.from_host(int(z["n"]), S.xi_x, S.xi_y, S.b_xy, S.b_psi, S.l, S.a, S.b,
                                     S.v_min, S.v_max, S.a_max)
    with pytest.raises(ValueError, match="team_warps"):
        solver.solve_device(prob, max_iter=3, tol=0.0, team_warps=4)
    with pytest.raises(ValueError, match="team_warps"):
        solver.solve_device(prob, max_iter=3, tol=0.0, team_warps=3)


def test_null_space_qp_info_and_refinement(cuda, monkeypatch):
    """The persistent solve's null-space QP (capi.cu reduced_qp): well-conditioned
    shapes skip the refinement step, ill-conditioned ones (c4) keep it, and
    forcing the refinement on a well-conditioned shape changes the trajectories
    by no more than rounding."""
    from paper_2109_10392_b200 import make_solver

    info = make_solver(100, 5.0, 10, 10).qp_info()
    assert not info["refine_xy"] and not info["refine_psi"]
    assert 1.0 < info["cond_xy"] < 1e4 and 1.0 < info["cond_psi"] < 1e4
    info4 = make_solver(200, 10.0, 15, 50).qp_info()
    assert info4["refine_xy"] and info4["cond_xy"] > 1e4

    z = golden("c1")
    solver, res = _plan(z)
    monkeypatch.setenv("BMPC_QP_REFINE", "3")
    forced = _solver(z)
    assert forced.qp_info()["refine_xy"] and forced.qp_info()["refine_psi"]
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    res2 = plan_batch(forced, _Scenes(z), max_iter=int(z["iters"]), tol=0.0,
                      spec=MetaCostSpec("cruise", v_cruise=20.0), limits=FilterLimits())
    err = traj_err(solver.basis.P, {"c_x": res2.c_x, "c_y": res2.c_y, "c_psi": res2.c_psi},
                   {"c_x": res.c_x, "c_y": res.c_y, "c_psi": res.c_psi})
    assert err.max() <= 1e-11, err.max()
    assert res.best_index == res2.best_index


def test_plan_host_direct_block_equals_staged(cuda):
    """plan_batch's zero-copy result block (one pinned block at the
    bmpc_plan_host_layout offsets) and the staged path (separate pageable
    numpy outputs) return the same bits."""
    import ctypes

    from paper_2109_10392_b200 import _native as nat
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, _spec_struct, plan_batch

    z = golden("c3s")
    solver = _solver(z)
    S = _Scenes(z)
    spec, limits = MetaCostSpec("cruise", v_cruise=20.0), FilterLimits()
    res = plan_batch(solver, S, max_iter=30, tol=0.0, spec=spec, limits=limits)
    assert res.c_x.base is not None  # a view of the pinned block
    nb, L, Sn = solver.basis.n_b, S.l * S.S, S.S
    c = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    xi_x, xi_y, b_xy, b_psi = c(S.xi_x), c(S.xi_y), c(S.b_xy), c(S.b_psi)
    prob = nat.Problem(xi_x.shape[1] // solver.basis.grid.n, S.l, Sn, xi_x.ctypes.data, xi_y.ctypes.data,
                       b_xy.ctypes.data, b_psi.ctypes.data, S.a, S.b, S.v_min, S.v_max, S.a_max)
    coef, rf = np.empty((3, nb, L)), np.empty((3, L))
    out = nat.SolveOut(coef[0].ctypes.data, coef[1].ctypes.data, coef[2].ctypes.data, None, None, None,
                       None, None, rf.ctypes.data, 0, 0)
    meta, mr, hm = np.empty((3, L))
    flags = np.empty(L, dtype=np.uint8)
    idx = np.empty((4, Sn), dtype=np.int64)
    so = nat.ScoreOut(meta.ctypes.data, mr.ctypes.data, hm.ctypes.data, flags.ctypes.data,
                      idx[0].ctypes.data, idx[1].ctypes.data, idx[2].ctypes.data, idx[3].ctypes.data)
    nat.check(nat.load().bmpc_plan_host(solver._context(), ctypes.byref(prob),
                                        ctypes.byref(nat.SolveOpts(max_iter=30, tol=0.0)), ctypes.byref(out),
                                        ctypes.byref(_spec_struct(spec, limits)), ctypes.byref(so), None),
              "plan_host")
    for got, want in ((res.c_x, coef[0]), (res.c_y, coef[1]), (res.c_psi, coef[2]), (res.res_final, rf),
                      (res.meta_cost, meta), (res.min_ratio, mr), (res.heading_max, hm),
                      (res.flags, flags), (res.argmin_all, idx[1]), (res.argmin_hc, idx[2]),
                      (res.n_feasible, idx[3])):
        assert np.array_equal(got, want, equal_nan=got.dtype.kind == "f")
    assert [b if b is not None else -1 for b in res.best_index] == list(idx[0])
    assert res.iterations == out.iterations == 30


def test_plan_host_pinned_inputs_read_in_place(cuda):
    """Page-locked inputs (read in place by the kernels) and pageable inputs
    (copied in) give the same bits."""
    import torch

    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    z = golden("c3s")
    solver = _solver(z)
    S = _Scenes(z)
    P = _Scenes(z)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).pin_memory().numpy()  # noqa: E731
    P.xi_x, P.xi_y, P.b_xy, P.b_psi = pin(S.xi_x), pin(S.xi_y), pin(S.b_xy), pin(S.b_psi)
    spec, limits = MetaCostSpec("cruise", v_cruise=20.0), FilterLimits()
    a = plan_batch(solver, S, max_iter=30, tol=0.0, spec=spec, limits=limits)
    b = plan_batch(solver, P, max_iter=30, tol=0.0, spec=spec, limits=limits)
    for k in ("c_x", "c_y", "c_psi", "res_final", "meta_cost", "min_ratio", "heading_max", "flags"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert a.best_index == b.best_index


@pytest.mark.parametrize("team", [1, 4])
def test_tol_early_exit(cuda, team):
    """tol > 0: the first launch exits once some sweep is globally converged
    (BMPC_F_POLL), the re-run reproduces exactly t* sweeps (solver.py:437-439).
    Same bits as a fixed t*-sweep solve, and far cheaper than max_iter sweeps."""
    import time

    z = golden("demo")
    solver = _solver(z)
    b = _batch(z)
    prob = solver.device_problem(b)
    ref = solver.solve_device(prob, max_iter=60, tol=0.0, team_warps=team)
    worst = ref.history[:60].amax(dim=(1, 2)).cpu().numpy()
    tol = float(worst[20]) * (1 + 1e-9)
    expect = int(np.argmax(worst <= tol)) + 1
    got = solver.solve_device(prob, max_iter=3000, tol=tol, team_warps=team)
    assert got.converged and got.iterations == expect
    exact = solver.solve_device(prob, max_iter=expect, tol=0.0, team_warps=team)
    for k in ("c_x", "c_y", "c_psi", "l_x", "l_y", "l_psi", "res_final"):
        assert cuda.equal(getattr(got, k), getattr(exact, k)), k
    assert cuda.equal(got.history[:expect], exact.history[:expect])

    def timed(max_iter, t):
        cuda.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            solver.solve_device(prob, max_iter=max_iter, tol=t, team_warps=team)
        cuda.cuda.synchronize()
        return (time.perf_counter() - t0) / 3

    timed(3000, tol)
    t_tol, t_full = timed(3000, tol), timed(3000, 0.0)
    print(f"team {team}: converged at {expect}; tol solve {1e3 * t_tol:.2f} ms vs 3000 sweeps {1e3 * t_full:.2f} ms")
    assert t_tol < 0.2 * t_full


def test_solve_stacked_scenes_lazy_state(cuda):
    """BatchSolver.solve on a stacked scene batch (the c3/c4 form): v, alpha, d,
    alpha_a, d_a stay on the device until read, the history is read back on
    first access; results equal plan_batch and per-scene solves bit for bit,
    and a lazy state warm-starts the next solve without a host round trip."""
    from paper_2109_10392_b200.planner import plan_batch

    z = golden("c3s")
    solver = _solver(z)
    S = _Scenes(z)
    state, info = solver.solve(S, max_iter=50, tol=0.0)
    for k in ("v", "alpha", "d", "alpha_a", "d_a"):
        assert type(state._raw(k)).__name__ == "_Deferred", k
    assert state._raw("alpha").shape == (int(z["m"]) * int(z["n"]), S.S * S.l)
    pb = plan_batch(solver, S, max_iter=50, tol=0.0)
    np.testing.assert_array_equal(state.c_x, pb.c_x)
    np.testing.assert_array_equal(state.c_psi, pb.c_psi)
    assert len(info.residual_history) == 50
    last = info.residual_history[-1]
    np.testing.assert_array_equal(np.stack([last.r_obs, last.r_acc, last.r_nonhol]), pb.res_final)
    l = S.l
    one, _ = solver.solve(_batch(z, s=2), max_iter=50, tol=0.0)
    cols = slice(2 * l, 3 * l)
    for k in ("c_x", "lambda_y", "v", "alpha", "d", "alpha_a", "d_a"):
        np.testing.assert_array_equal(getattr(one, k), getattr(state, k)[:, cols], err_msg=k)
    # warm start from a lazy state (device fields used in place) == from host arrays
    state2, _ = solver.solve(S, max_iter=50, tol=0.0)
    w_lazy, _ = solver.solve(S, max_iter=7, tol=0.0, warm=state2, keep_multipliers=True)
    host = state2.copy()
    for k in ("v", "alpha", "d", "alpha_a", "d_a"):
        getattr(host, k)  # materialise
    w_host, _ = solver.solve(S, max_iter=7, tol=0.0, warm=host, keep_multipliers=True)
    np.testing.assert_array_equal(w_lazy.c_x, w_host.c_x)
    np.testing.assert_array_equal(w_lazy.lambda_psi, w_host.lambda_psi)
    with pytest.raises(ValueError):
        solver.solve(_batch(z, s=0), max_iter=3, warm=state2)  # L columns vs l


@pytest.mark.parametrize("name,team", [("c0", 4), ("c0", 2), ("c1", 0), ("c2f", 0), ("c4f", 0)])
def test_repeat_runs_bitwise_deterministic(cuda, name, team):
    """Race / barrier-misuse canary (compute-sanitizer is closed on this GPU
    pool): the persistent kernel's shared-memory exchanges (transpose buffer,
    team exchange slots, staged predictions, the polled early exit) would
    show up as run-to-run differences; 12 repeated solves of every kernel
    variant must agree bit for bit."""
    from paper_2109_10392_b200 import device as D

    z = golden(name)
    solver = _solver(z)
    S = _Scenes(z)
    prob = D.DeviceProblem.from_host(int(z["n"]), S.xi_x, S.xi_y, S.b_xy, S.b_psi, S.l, S.a, S.b,
                                     S.v_min, S.v_max, S.a_max)
    ref = solver.solve_device(prob, max_iter=30, tol=0.0, team_warps=team)
    tol_ref = solver.solve_device(prob, max_iter=30, tol=1e-9, team_warps=team)
    for _ in range(12):
        again = solver.solve_device(prob, max_iter=30, tol=0.0, team_warps=team)
        for k in ("c_x", "c_y", "c_psi", "l_x", "l_psi", "res_final"):
            assert cuda.equal(getattr(again, k), getattr(ref, k)), k
    again = solver.solve_device(prob, max_iter=30, tol=1e-9, team_warps=team)
    assert again.iterations == tol_ref.iterations and cuda.equal(again.c_x, tol_ref.c_x)


@pytest.mark.parametrize("name,where", [("c0", "b_xy"), ("c3f", "b_xy"), ("c0", "xi")])
def test_nan_stays_in_its_column(cuda, name, where):
    """Non-finite inputs behave as in the reference's numpy arithmetic: a NaN
    boundary value poisons exactly its own instance (coefficients NaN, never
    feasible, numpy's argmin rule picks it as the unfiltered argmin) and every
    other column keeps its bits; a NaN obstacle sample poisons its scene."""
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    z = golden(name)
    solver = _solver(z)
    spec, limits = MetaCostSpec("cruise", v_cruise=20.0), FilterLimits()
    clean = plan_batch(solver, _Scenes(z), max_iter=20, tol=0.0, spec=spec, limits=limits)
    sc = _Scenes(z)
    L = sc.l * sc.S
    if where == "b_xy":
        bad = min(5, sc.l - 1)  # an instance of scene 0
        sc.b_xy = np.array(sc.b_xy, copy=True)
        sc.b_xy[3, bad] = np.nan
        res = plan_batch(solver, sc, max_iter=20, tol=0.0, spec=spec, limits=limits)
        keep = np.arange(L) != bad
        for k in ("c_x", "c_y", "c_psi"):
            np.testing.assert_array_equal(getattr(res, k)[:, keep], getattr(clean, k)[:, keep])
        for k in ("meta_cost", "min_ratio", "heading_max", "flags"):
            np.testing.assert_array_equal(getattr(res, k)[keep], getattr(clean, k)[keep])
        # (the coefficients the boundary pins come straight from b; the free ones are NaN)
        assert np.isnan(res.c_x[:, bad]).any() and np.isnan(res.meta_cost[bad])
        assert not res.feasible[bad]
        assert int(res.argmin_all[0]) == bad  # np.argmin returns the first NaN
        # the filtered winner ignores the poisoned column
        want = clean.best_index[0]
        if want == bad:
            cost = np.where(clean.feasible[:sc.l] & (np.arange(sc.l) != bad), clean.meta_cost[:sc.l], np.inf)
            want = int(np.argmin(cost)) if np.isfinite(cost).any() else None
        assert res.best_index[0] == want
        assert res.best_index[1:] == clean.best_index[1:]
    else:
        sc.xi_x = np.array(sc.xi_x, copy=True)
        sc.xi_x[0, 17] = np.nan  # obstacle 0, sample 17 of scene 0
        res = plan_batch(solver, sc, max_iter=20, tol=0.0, spec=spec, limits=limits)
        # every instance of the scene sees the NaN term at sample 17: the reference's
        # closed forms propagate it into g and the whole column
        assert np.isnan(res.c_x[:, :sc.l]).any(axis=0).all() and not res.feasible[:sc.l].any()
        assert res.best_index[0] is None
    # The reference-shaped BatchSolver.solve keeps the reference's error: its QP
    # solves go through scipy's lu_solve (solver.py:166), whose finite check
    # raises ValueError on the first non-finite right-hand side.
    if sc.S == 1:
        from paper_2109_10392_b200 import ProblemBatch

        pb = ProblemBatch(l=sc.l, xi_x=sc.xi_x[0], xi_y=sc.xi_y[0], a=sc.a, b=sc.b, v_min=sc.v_min,
                          v_max=sc.v_max, a_max=sc.a_max, b_xy=sc.b_xy, b_psi=sc.b_psi)
        with pytest.raises(ValueError, match="infs or NaNs"):
            solver.solve(pb, max_iter=8, tol=0.0)
        with pytest.raises(ValueError, match="infs or NaNs"):
            solver.solve(pb, max_iter=8, tol=1e-3)
