"""Step-wise solver API (reference solver.py:288-410) on the device, checked
against numpy restatements of each reference step (the oracle's formulas) on
randomised states, and composed into one sweep against solve(max_iter=1)."""

import numpy as np
import pytest

import am_oracle as O
from conftest import golden

pytestmark = pytest.mark.gpu


def _setup():
    from paper_2109_10392_b200 import ProblemBatch, make_solver

    z = golden("demo")
    solver = make_solver(100, 10.0, 10, 10)
    batch = ProblemBatch(l=11, xi_x=z["xi_x"], xi_y=z["xi_y"], a=float(z["a"]), b=float(z["b"]),
                         v_min=float(z["v_min"]), v_max=float(z["v_max"]), a_max=float(z["a_max"]),
                         b_xy=z["b_xy"], b_psi=z["b_psi"])
    return solver, batch, O.OracleSolver(100, 10.0, 10, 10)


def _random_state(solver, batch, rng):
    st = solver.init_state(batch)
    nb, l = solver.basis.n_b, batch.l
    st.c_x = st.c_x + rng.normal(0, 1.0, (nb, l))
    st.c_y = st.c_y + rng.normal(0, 1.0, (nb, l))
    st.c_psi = rng.normal(0, 0.05, (nb, l))
    st.alpha = rng.uniform(-np.pi, np.pi, st.alpha.shape)
    st.d = 1.0 + rng.uniform(0, 2.0, st.d.shape)
    st.alpha_a = rng.uniform(-np.pi, np.pi, st.alpha_a.shape)
    st.d_a = rng.uniform(0, 8.0, st.d_a.shape)
    st.v = rng.uniform(0.5, 20.0, st.v.shape)
    st.lambda_x = rng.normal(0, 5.0, (nb, l))
    st.lambda_y = rng.normal(0, 5.0, (nb, l))
    st.lambda_psi = rng.normal(0, 5.0, (nb, l))
    return st


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def test_build_g_and_qp_steps(cuda, rng):
    solver, batch, o = _setup()
    st = _random_state(solver, batch, rng)
    kern = O.kernels("numpy")
    ost = {k: getattr(st, k).copy() for k in ("c_x", "c_y", "c_psi", "alpha", "d", "alpha_a", "d_a",
                                               "v", "lambda_x", "lambda_y", "lambda_psi")}
    g_x, g_y = o.g_parts(ost, batch.xi_x, batch.xi_y, batch.a, batch.b, kern)
    assert _rel(solver.build_g(st, batch), np.vstack([g_x, g_y])) <= 1e-12
    # xy QP (solver.py:302-312) through the oracle's LU + refinement
    nb, l = solver.basis.n_b, batch.l
    proj = o.F_axis.T @ np.concatenate([g_x, g_y], axis=1)
    rhs = np.vstack([proj[:, :l] + ost["lambda_x"], proj[:, l:] + ost["lambda_y"], batch.b_xy])
    sol = o._refined_solve(o.lu_xy, o.matrix_xy, rhs)
    n0 = solver.kkt.n_solves
    cx, cy = solver.step_xy(st, batch)
    assert _rel(cx, sol[:nb]) <= 1e-9 and _rel(cy, sol[nb:2 * nb]) <= 1e-9
    # psi QP (solver.py:314-328)
    th = np.unwrap(np.arctan2(o.Pdot @ st.c_y, o.Pdot @ st.c_x), axis=0)
    rp = np.vstack([o.P.T @ th + st.lambda_psi, batch.b_psi])
    ref_p = o._refined_solve(o.lu_psi, o.matrix_psi, rp)[:nb]
    assert _rel(solver.step_psi(st, batch), ref_p) <= 1e-9
    assert solver.kkt.n_solves == n0 + 2


def test_closed_form_steps(cuda, rng):
    solver, batch, o = _setup()
    st = _random_state(solver, batch, rng)
    P, Pd, Pdd = o.P, o.Pdot, o.Pddot
    kern = O.kernels("numpy")
    xd, yd = Pd @ st.c_x, Pd @ st.c_y
    np.testing.assert_allclose(solver.step_v(st, batch), kern.v_update(xd, yd, batch.v_min, batch.v_max),
                               rtol=1e-13, atol=1e-13)
    x, y = P @ st.c_x, P @ st.c_y
    al_ref, _ = kern.obstacle_update(x, y, batch.xi_x, batch.xi_y, batch.a, batch.b)
    assert np.abs(solver.step_alpha_obs(st, batch) - al_ref).max() <= 1e-12
    # d given alpha (solver.py:342-354)
    n, m = 100, 10
    wx = np.tile(x, (m, 1)) - batch.xi_x[:, None]
    wy = np.tile(y, (m, 1)) - batch.xi_y[:, None]
    ca, sa = np.cos(st.alpha), np.sin(st.alpha)
    d_ref = np.maximum(1.0, (batch.a * ca * wx + batch.b * sa * wy) /
                       ((batch.a * ca) ** 2 + (batch.b * sa) ** 2))
    assert _rel(solver.step_d_obs(st, batch), d_ref) <= 1e-12
    xdd, ydd = Pdd @ st.c_x, Pdd @ st.c_y
    assert np.abs(solver.step_alpha_acc(st, batch) - np.arctan2(ydd, xdd)).max() <= 1e-12
    np.testing.assert_allclose(solver.step_d_acc(st, batch),
                               np.minimum(np.sqrt(xdd**2 + ydd**2), batch.a_max), rtol=1e-13, atol=1e-13)
    del n


def test_multipliers_and_residuals(cuda, rng):
    solver, batch, o = _setup()
    st = _random_state(solver, batch, rng)
    P, Pd, Pdd = o.P, o.Pdot, o.Pddot
    kern = O.kernels("numpy")
    r_x, r_y = kern.residual_vectors(P @ st.c_x, P @ st.c_y, Pd @ st.c_x, Pd @ st.c_y, Pdd @ st.c_x,
                                     Pdd @ st.c_y, P @ st.c_psi, batch.xi_x, batch.xi_y, st.alpha,
                                     st.d, st.alpha_a, st.d_a, st.v, batch.a, batch.b)
    res = solver.compute_residuals(st, batch)
    mn, n = 1000, 100
    for got, lo, hi in ((res.r_obs, 0, mn), (res.r_acc, mn, mn + n), (res.r_nonhol, mn + n, mn + 2 * n)):
        ref = np.sqrt((r_x[lo:hi] ** 2).sum(axis=0) + (r_y[lo:hi] ** 2).sum(axis=0))
        np.testing.assert_allclose(got, ref, rtol=1e-11)
    lx = st.lambda_x - o.F_axis.T @ r_x
    ly = st.lambda_y - o.F_axis.T @ r_y
    th = np.unwrap(np.arctan2(Pd @ st.c_y, Pd @ st.c_x), axis=0)
    lp = st.lambda_psi - P.T @ (P @ st.c_psi - th)
    solver.update_multipliers(st, batch)
    assert _rel(st.lambda_x, lx) <= 1e-11 and _rel(st.lambda_y, ly) <= 1e-11
    assert _rel(st.lambda_psi, lp) <= 1e-11


def test_manual_sweep_equals_one_iteration(cuda):
    """The reference's step order reproduces one solve sweep
    (tests/test_solver_units.py:290-306 pins the same property)."""
    solver, batch, _ = _setup()
    st = solver.init_state(batch)
    solver.step_xy(st, batch)
    solver.step_psi(st, batch)
    solver.step_v(st, batch)
    solver.step_alpha_obs(st, batch)
    solver.step_d_obs(st, batch)
    solver.step_alpha_acc(st, batch)
    solver.step_d_acc(st, batch)
    solver.update_multipliers(st, batch)
    one, info = solver.solve(batch, max_iter=1, tol=0.0)
    for k in ("c_x", "c_y", "c_psi", "lambda_x", "lambda_y", "lambda_psi", "v", "d_a"):
        assert _rel(getattr(st, k), getattr(one, k)) <= 1e-9, k
    res = solver.compute_residuals(st, batch)
    np.testing.assert_allclose(res.r_nonhol, info.residual_history[-1].r_nonhol, rtol=1e-8, atol=1e-10)
