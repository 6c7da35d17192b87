"""CPU ORACLE for the batched AM trajectory optimizer -- TEST INFRASTRUCTURE ONLY.

This module is the checker the CUDA path is compared against, and the CPU
baseline ("port") that ``bench.py`` times.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may import it; the
product package never does.

It restates, operation for operation, the reference's numpy path
(/root/reference/pkg/src/batchmpc/, cited as file:line below), so with the
same BLAS it reproduces the reference's numbers bit for bit; the golden
fixtures under tests/golden/ (produced by running the reference itself, see
tests/golden/make_golden.py) pin that.

  basis_matrices          basis.py:30-37 (grid), :61-96 (Bernstein rows, exact derivatives)
  OracleSolver.__init__   basis.py:158-200 (F_o, F_axis, Q, A, A_psi); solver.py:131-155 (KKT
                          assembly, one LU per matrix); solver.py:182-193 (pinv(P), [P;Pdot;Pddot])
  _refined_solve          solver.py:164-168 (LU solve + one refinement step)
  init_cold               solver.py:226-252 (straight line -> pinv(P); clipped start speed;
                          obstacle_update on the line; zero multipliers)
  iterate                 solver.py:458-500 (xy QP, sampling, unwrap(atan2), psi QP,
                          tail_core, multiplier updates, residual norms)
  solve                   solver.py:414-456 (tol = global max over instances; end-of-solve
                          materialisation of alpha/d/alpha_a/d_a)
  sample_plan/score       planner.py:412-423, :219-257 (collision ratios, filters, meta cost,
                          argmin with lowest-index ties, None when nothing is feasible)

Kernel back-ends for the per-iteration elementwise work:
  "numpy" -- restatement of kernels/_numpy.py
  "c"     -- oracle/am_oracle.c (restatement of kernels/_speedups.pyx), via ctypes
  "ref"   -- the reference's own Cython kernels compiled by oracle/Makefile into oracle/_ref/
"""

from __future__ import annotations

import ctypes
import importlib.util
import math
import os
from pathlib import Path

import numpy as np
from scipy.linalg import lu_factor, lu_solve
from scipy.special import comb

HERE = Path(__file__).resolve().parent

# ----------------------------------------------------------------------------
# basis (basis.py:30-96, :158-200)
# ----------------------------------------------------------------------------


def bernstein_rows(u: np.ndarray, degree: int) -> np.ndarray:
    k = np.arange(degree + 1)
    uu = u[:, None]
    return comb(degree, k) * uu**k * (1.0 - uu) ** (degree - k)


def basis_matrices(n: int, t_f: float, degree: int, t0: float = 0.0):
    """(times, P, Pdot, Pddot) exactly as basis.build_time_grid/build_basis."""
    times = np.linspace(t0, t_f, n)
    span = t_f - t0
    u = (times - t0) / span
    P = bernstein_rows(u, degree)
    low1 = bernstein_rows(u, degree - 1)
    dP = np.zeros_like(P)
    dP[:, :-1] -= low1
    dP[:, 1:] += low1
    dP *= degree
    low2 = bernstein_rows(u, degree - 2)
    ddP = np.zeros_like(P)
    ddP[:, :-2] += low2
    ddP[:, 1:-1] -= 2.0 * low2
    ddP[:, 2:] += low2
    ddP *= degree * (degree - 1)
    return times, P, dP / span, ddP / span**2


# ----------------------------------------------------------------------------
# elementwise kernels
# ----------------------------------------------------------------------------


class _NumpyKernels:
    """Restatement of kernels/_numpy.py (the reference's spec for the compiled twin)."""

    @staticmethod
    def obstacle_update(x, y, xi_x, xi_y, a, b):  # _numpy.py:11-22
        n = x.shape[0]
        m = xi_x.shape[0] // n if n else 0
        wx = np.tile(x, (m, 1)) - xi_x[:, None]
        wy = np.tile(y, (m, 1)) - xi_y[:, None]
        alpha = np.arctan2(a * wy, b * wx)
        ca, sa = np.cos(alpha), np.sin(alpha)
        num = a * ca * wx + b * sa * wy
        den = (a * ca) ** 2 + (b * sa) ** 2
        return alpha, np.maximum(1.0, num / den)

    @staticmethod
    def accel_update(xddot, yddot, a_max):  # _numpy.py:25-29
        return np.arctan2(yddot, xddot), np.minimum(np.sqrt(xddot * xddot + yddot * yddot), a_max)

    @staticmethod
    def v_update(xdot, ydot, v_min, v_max):  # _numpy.py:32-34
        return np.clip(np.sqrt(xdot * xdot + ydot * ydot), v_min, v_max)

    @staticmethod
    def assemble_g(xi_x, xi_y, alpha, d, alpha_a, d_a, v, psi, a, b):  # _numpy.py:37-49
        mn, l = alpha.shape
        n = v.shape[0]
        g_x = np.empty((mn + 2 * n, l))
        g_y = np.empty((mn + 2 * n, l))
        g_x[:mn] = xi_x[:, None] + a * d * np.cos(alpha)
        g_y[:mn] = xi_y[:, None] + b * d * np.sin(alpha)
        g_x[mn : mn + n] = d_a * np.cos(alpha_a)
        g_y[mn : mn + n] = d_a * np.sin(alpha_a)
        g_x[mn + n :] = v * np.cos(psi)
        g_y[mn + n :] = v * np.sin(psi)
        return g_x, g_y

    @staticmethod
    def residual_vectors(x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, alpha, d,
                         alpha_a, d_a, v, a, b):  # _numpy.py:52-66
        mn = alpha.shape[0]
        n, l = x.shape
        m = mn // n if n else 0
        r_x = np.empty((mn + 2 * n, l))
        r_y = np.empty((mn + 2 * n, l))
        r_x[:mn] = np.tile(x, (m, 1)) - xi_x[:, None] - a * d * np.cos(alpha)
        r_y[:mn] = np.tile(y, (m, 1)) - xi_y[:, None] - b * d * np.sin(alpha)
        r_x[mn : mn + n] = xddot - d_a * np.cos(alpha_a)
        r_y[mn : mn + n] = yddot - d_a * np.sin(alpha_a)
        r_x[mn + n :] = xdot - v * np.cos(psi)
        r_y[mn + n :] = ydot - v * np.sin(psi)
        return r_x, r_y

    @staticmethod
    def tail_core(x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, v_min, v_max, a_max, a, b):
        # _numpy.py:69-131
        mn = xi_x.shape[0]
        n, l = x.shape
        m = mn // n if n else 0
        wx = np.tile(x, (m, 1)) - xi_x[:, None]
        wy = np.tile(y, (m, 1)) - xi_y[:, None]
        py, px = a * wy, b * wx
        r = np.sqrt(px * px + py * py)
        safe = np.where(r > 0.0, r, 1.0)
        ca = np.where(r > 0.0, px / safe, 1.0)
        sa = np.where(r > 0.0, py / safe, 0.0)
        d = np.maximum(1.0, r / (a * b))
        mag = np.sqrt(xddot * xddot + yddot * yddot)
        safe_m = np.where(mag > 0.0, mag, 1.0)
        ca_a = np.where(mag > 0.0, xddot / safe_m, 1.0)
        sa_a = np.where(mag > 0.0, yddot / safe_m, 0.0)
        d_a = np.minimum(mag, a_max)
        v = np.clip(np.sqrt(xdot * xdot + ydot * ydot), v_min, v_max)
        cp, sp = np.cos(psi), np.sin(psi)
        r_x = np.empty((mn + 2 * n, l))
        r_y = np.empty((mn + 2 * n, l))
        g_x = np.empty((mn + 2 * n, l))
        g_y = np.empty((mn + 2 * n, l))
        adca = a * d * ca
        bdsa = b * d * sa
        r_x[:mn] = wx - adca
        r_y[:mn] = wy - bdsa
        g_x[:mn] = xi_x[:, None] + adca
        g_y[:mn] = xi_y[:, None] + bdsa
        daca = d_a * ca_a
        dasa = d_a * sa_a
        r_x[mn : mn + n] = xddot - daca
        r_y[mn : mn + n] = yddot - dasa
        g_x[mn : mn + n] = daca
        g_y[mn : mn + n] = dasa
        vcp = v * cp
        vsp = v * sp
        r_x[mn + n :] = xdot - vcp
        r_y[mn + n :] = ydot - vsp
        g_x[mn + n :] = vcp
        g_y[mn + n :] = vsp
        sq_obs = np.einsum("ij,ij->j", r_x[:mn], r_x[:mn]) + np.einsum("ij,ij->j", r_y[:mn], r_y[:mn])
        sq_acc = np.einsum("ij,ij->j", r_x[mn : mn + n], r_x[mn : mn + n]) + np.einsum(
            "ij,ij->j", r_y[mn : mn + n], r_y[mn : mn + n])
        sq_nonhol = np.einsum("ij,ij->j", r_x[mn + n :], r_x[mn + n :]) + np.einsum(
            "ij,ij->j", r_y[mn + n :], r_y[mn + n :])
        return d, d_a, v, r_x, r_y, g_x, g_y, sq_obs, sq_acc, sq_nonhol


_dp = ctypes.POINTER(ctypes.c_double)
_i = ctypes.c_ssize_t
_d = ctypes.c_double


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class _CKernels:
    """ctypes front of oracle/am_oracle.c (restates kernels/_speedups.pyx)."""

    def __init__(self, path: Path):
        lib = ctypes.CDLL(str(path))
        lib.oracle_obstacle_update.argtypes = [_i, _i, _i] + [_dp] * 4 + [_d, _d] + [_dp] * 2
        lib.oracle_accel_update.argtypes = [_i, _i, _dp, _dp, _d, _dp, _dp]
        lib.oracle_v_update.argtypes = [_i, _i, _dp, _dp, _d, _d, _dp]
        lib.oracle_assemble_g.argtypes = [_i, _i, _i] + [_dp] * 8 + [_d, _d] + [_dp] * 2
        lib.oracle_tail_core.argtypes = [_i, _i, _i] + [_dp] * 9 + [_d] * 5 + [_dp] * 10
        for f in ("oracle_obstacle_update", "oracle_accel_update", "oracle_v_update",
                  "oracle_assemble_g", "oracle_tail_core"):
            getattr(lib, f).restype = None
        self.lib = lib

    def obstacle_update(self, x, y, xi_x, xi_y, a, b):
        x, y = np.ascontiguousarray(x), np.ascontiguousarray(y)
        xi_x, xi_y = np.ascontiguousarray(xi_x), np.ascontiguousarray(xi_y)
        n, l = x.shape
        mn = xi_x.shape[0]
        alpha = np.empty((mn, l))
        d = np.empty((mn, l))
        self.lib.oracle_obstacle_update(n, l, mn, _ptr(x), _ptr(y), _ptr(xi_x), _ptr(xi_y),
                                        a, b, _ptr(alpha), _ptr(d))
        return alpha, d

    def accel_update(self, xddot, yddot, a_max):
        xddot, yddot = np.ascontiguousarray(xddot), np.ascontiguousarray(yddot)
        n, l = xddot.shape
        al = np.empty((n, l))
        da = np.empty((n, l))
        self.lib.oracle_accel_update(n, l, _ptr(xddot), _ptr(yddot), a_max, _ptr(al), _ptr(da))
        return al, da

    def v_update(self, xdot, ydot, v_min, v_max):
        xdot, ydot = np.ascontiguousarray(xdot), np.ascontiguousarray(ydot)
        n, l = xdot.shape
        v = np.empty((n, l))
        self.lib.oracle_v_update(n, l, _ptr(xdot), _ptr(ydot), v_min, v_max, _ptr(v))
        return v

    def assemble_g(self, xi_x, xi_y, alpha, d, alpha_a, d_a, v, psi, a, b):
        arrs = [np.ascontiguousarray(t) for t in (xi_x, xi_y, alpha, d, alpha_a, d_a, v, psi)]
        mn, l = arrs[2].shape
        n = arrs[6].shape[0]
        g_x = np.empty((mn + 2 * n, l))
        g_y = np.empty((mn + 2 * n, l))
        self.lib.oracle_assemble_g(n, l, mn, *[_ptr(t) for t in arrs], a, b, _ptr(g_x), _ptr(g_y))
        return g_x, g_y

    def residual_vectors(self, *args):
        return _NumpyKernels.residual_vectors(*args)

    def tail_core(self, x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, v_min, v_max, a_max, a, b):
        arrs = [np.ascontiguousarray(t) for t in (x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y)]
        n, l = arrs[0].shape
        mn = arrs[7].shape[0]
        d = np.empty((mn, l))
        d_a = np.empty((n, l))
        v = np.empty((n, l))
        r_x = np.empty((mn + 2 * n, l))
        r_y = np.empty((mn + 2 * n, l))
        g_x = np.empty((mn + 2 * n, l))
        g_y = np.empty((mn + 2 * n, l))
        sq = [np.zeros(l) for _ in range(3)]
        self.lib.oracle_tail_core(n, l, mn, *[_ptr(t) for t in arrs], v_min, v_max, a_max, a, b,
                                  _ptr(d), _ptr(d_a), _ptr(v), _ptr(r_x), _ptr(r_y), _ptr(g_x),
                                  _ptr(g_y), *[_ptr(s) for s in sq])
        return d, d_a, v, r_x, r_y, g_x, g_y, sq[0], sq[1], sq[2]


def _load_ref_kernels():
    """The reference's own compiled Cython kernels (oracle/_ref), if built."""
    for p in sorted((HERE / "_ref").glob("_speedups*.so")):
        spec = importlib.util.spec_from_file_location("_speedups", p)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        return mod
    return None


_KERNEL_CACHE: dict = {}


def kernels(kind: str = "c"):
    if kind in _KERNEL_CACHE:
        return _KERNEL_CACHE[kind]
    if kind == "numpy":
        k = _NumpyKernels()
    elif kind == "c":
        so = HERE / "liboracle.so"
        if not so.exists():
            build_c()
        k = _CKernels(so)
    elif kind == "ref":
        k = _load_ref_kernels()
        if k is None:
            raise FileNotFoundError("oracle/_ref not built (make -C oracle ref)")
    else:
        raise ValueError(f"unknown oracle kernel kind {kind!r}")
    _KERNEL_CACHE[kind] = k
    return k


def build_c() -> Path:
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    return HERE / "liboracle.so"


# ----------------------------------------------------------------------------
# solver (solver.py)
# ----------------------------------------------------------------------------


class OracleSolver:
    """One problem shape: basis, constant matrices, the two LU-factored KKT systems."""

    def __init__(self, n: int, t_f: float, degree: int, m: int, rho: float = 1.0, t0: float = 0.0):
        self.n, self.m, self.degree, self.rho = n, m, degree, rho
        self.n_b = nb = degree + 1
        self.times, self.P, self.Pdot, self.Pddot = basis_matrices(n, t_f, degree, t0)
        self.t0, self.tf = t0, t_f
        P, Pd, Pdd = self.P, self.Pdot, self.Pddot
        self.F_axis = np.vstack([np.tile(P, (m, 1)), Pdd, Pd])
        self.Q = Pdd.T @ Pdd
        self.A_axis = np.array([P[0], Pd[0], Pdd[0], P[-1], Pd[-1], Pdd[-1]])
        self.A_psi = np.array([P[0], Pd[0], P[-1], Pd[-1]])
        A = np.zeros((12, 2 * nb))
        A[:6, :nb] = self.A_axis
        A[6:, nb:] = self.A_axis
        H = np.zeros((2 * nb, 2 * nb))
        H[:nb, :nb] = self.Q + rho * (self.F_axis.T @ self.F_axis)
        H[nb:, nb:] = H[:nb, :nb]
        K = np.zeros((2 * nb + 12, 2 * nb + 12))
        K[: 2 * nb, : 2 * nb] = H
        K[: 2 * nb, 2 * nb :] = A.T
        K[2 * nb :, : 2 * nb] = A
        Kp = np.zeros((nb + 4, nb + 4))
        Kp[:nb, :nb] = self.Q + rho * (P.T @ P)
        Kp[:nb, nb:] = self.A_psi.T
        Kp[nb:, :nb] = self.A_psi
        self.matrix_xy, self.matrix_psi = K, Kp
        self.lu_xy, self.lu_psi = lu_factor(K), lu_factor(Kp)
        self.pinvP = np.linalg.pinv(P)
        self.sample_all = np.vstack([P, Pd, Pdd])

    @staticmethod
    def _refined_solve(lu, K, rhs):
        sol = lu_solve(lu, rhs)
        sol += lu_solve(lu, rhs - K @ sol)
        return sol

    # -- state ---------------------------------------------------------------
    def init_cold(self, xi_x, xi_y, b_xy, a, b, v_min, v_max, kern):
        n, nb, l = self.n, self.n_b, b_xy.shape[1]
        x0, xf, y0, yf = b_xy[0], b_xy[3], b_xy[6], b_xy[9]
        vx0, vy0 = b_xy[1], b_xy[7]
        tau = (self.times - self.t0) / (self.tf - self.t0)
        x_line = x0[None, :] + tau[:, None] * (xf - x0)[None, :]
        y_line = y0[None, :] + tau[:, None] * (yf - y0)[None, :]
        st = dict(
            c_x=self.pinvP @ x_line, c_y=self.pinvP @ y_line, c_psi=np.zeros((nb, l)),
            alpha_a=np.zeros((n, l)), d_a=np.zeros((n, l)),
            lambda_x=np.zeros((nb, l)), lambda_y=np.zeros((nb, l)), lambda_psi=np.zeros((nb, l)),
        )
        speed0 = np.clip(np.sqrt(vx0 * vx0 + vy0 * vy0), v_min, v_max)
        st["v"] = np.broadcast_to(speed0, (n, l)).copy()
        st["alpha"], st["d"] = kern.obstacle_update(x_line, y_line, xi_x, xi_y, a, b)
        return st

    def g_parts(self, st, xi_x, xi_y, a, b, kern):  # solver.py:281-286
        psi = self.P @ st["c_psi"]
        return kern.assemble_g(xi_x, xi_y, st["alpha"], st["d"], st["alpha_a"], st["d_a"],
                               st["v"], psi, a, b)

    # -- one AM sweep (solver.py:458-500) -------------------------------------
    def iterate(self, st, prm, g_x, g_y, kern):
        n, nb, rho = self.n, self.n_b, prm["rho"]
        l = g_x.shape[1]
        proj = self.F_axis.T @ np.concatenate([g_x, g_y], axis=1)
        rhs = np.empty((2 * nb + 12, l))
        rhs[:nb] = rho * proj[:, :l] + st["lambda_x"]
        rhs[nb : 2 * nb] = rho * proj[:, l:] + st["lambda_y"]
        rhs[2 * nb :] = prm["b_xy"]
        sol = self._refined_solve(self.lu_xy, self.matrix_xy, rhs)
        st["c_x"] = sol[:nb].copy()
        st["c_y"] = sol[nb : 2 * nb].copy()

        s = self.sample_all @ np.concatenate([st["c_x"], st["c_y"]], axis=1)
        x, xdot, xddot = s[:n, :l], s[n : 2 * n, :l], s[2 * n :, :l]
        y, ydot, yddot = s[:n, l:], s[n : 2 * n, l:], s[2 * n :, l:]
        theta = np.unwrap(np.arctan2(ydot, xdot), axis=0)
        rhs_p = np.empty((nb + 4, l))
        rhs_p[:nb] = rho * (self.P.T @ theta) + st["lambda_psi"]
        rhs_p[nb:] = prm["b_psi"]
        st["c_psi"] = self._refined_solve(self.lu_psi, self.matrix_psi, rhs_p)[:nb].copy()
        psi = self.P @ st["c_psi"]

        (st["d"], st["d_a"], st["v"], r_x, r_y, g_x2, g_y2, sq_o, sq_a, sq_n) = kern.tail_core(
            np.ascontiguousarray(x), np.ascontiguousarray(y),
            np.ascontiguousarray(xdot), np.ascontiguousarray(ydot),
            np.ascontiguousarray(xddot), np.ascontiguousarray(yddot), psi,
            prm["xi_x"], prm["xi_y"], prm["v_min"], prm["v_max"], prm["a_max"], prm["a"], prm["b"])
        lam = self.F_axis.T @ np.concatenate([r_x, r_y], axis=1)
        st["lambda_x"] -= rho * lam[:, :l]
        st["lambda_y"] -= rho * lam[:, l:]
        st["lambda_psi"] -= rho * (self.P.T @ (psi - theta))
        res = np.stack([np.sqrt(sq_o), np.sqrt(sq_a), np.sqrt(sq_n)])
        return res, g_x2, g_y2

    # -- full solve (solver.py:414-456) ---------------------------------------
    def solve(self, xi_x, xi_y, b_xy, b_psi, a, b, v_min, v_max, a_max, max_iter=100,
              tol=0.0, rho=None, kernel="c", record_iterates=False, warm=None,
              keep_multipliers=False):
        if max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        kern = kernels(kernel)
        xi_x = np.ascontiguousarray(xi_x, dtype=np.float64)
        xi_y = np.ascontiguousarray(xi_y, dtype=np.float64)
        prm = dict(xi_x=xi_x, xi_y=xi_y, b_xy=b_xy, b_psi=b_psi, a=a, b=b, v_min=v_min,
                   v_max=v_max, a_max=a_max, rho=self.rho if rho is None else rho)
        if warm is not None:
            st = {k: np.array(v, dtype=np.float64, copy=True) for k, v in warm.items()}
            if not keep_multipliers:
                for k in ("lambda_x", "lambda_y", "lambda_psi"):
                    st[k][...] = 0.0
        else:
            st = self.init_cold(xi_x, xi_y, b_xy, a, b, v_min, v_max, kern)
        history, iterates = [], []
        g_x, g_y = self.g_parts(st, xi_x, xi_y, a, b, kern)
        converged = False
        it = 0
        for _ in range(max_iter):
            res, g_x, g_y = self.iterate(st, prm, g_x, g_y, kern)
            it += 1
            history.append(res)
            if record_iterates:
                iterates.append((st["c_x"].copy(), st["c_y"].copy(), st["c_psi"].copy()))
            if float(res.max()) <= tol:
                converged = True
                break
        x = self.P @ st["c_x"]
        y = self.P @ st["c_y"]
        st["alpha"], st["d"] = kern.obstacle_update(x, y, xi_x, xi_y, a, b)
        st["alpha_a"], st["d_a"] = kern.accel_update(self.Pddot @ st["c_x"], self.Pddot @ st["c_y"], a_max)
        st["history"] = np.stack(history)  # (iters, 3, l): r_obs, r_acc, r_nonhol
        st["iterations"] = it
        st["converged"] = converged
        if record_iterates:
            st["iterates"] = iterates
        return st

    # -- scoring (planner.py:210-257, :412-423) --------------------------------
    def sample_plan(self, st):
        P, Pd, Pdd = self.P, self.Pdot, self.Pddot
        xdot = Pd @ st["c_x"]
        ydot = Pd @ st["c_y"]
        return dict(x=P @ st["c_x"], y=P @ st["c_y"], psi=P @ st["c_psi"],
                    psidot=Pd @ st["c_psi"], v=np.sqrt(xdot**2 + ydot**2),
                    xddot=Pdd @ st["c_x"], yddot=Pdd @ st["c_y"])

    def score(self, st, xi_x, xi_y, a, b, kind="cruise", v_cruise=15.0, v_max=20.0, y_rl=0.0,
              w1=1.0, w2=1.0, heading_limit=math.radians(13.0), residual_tol=1e-3,
              collision_margin=0.01):
        plan = self.sample_plan(st)
        n = plan["x"].shape[0]
        m = xi_x.shape[0] // n if n else 0
        l = plan["x"].shape[1]
        heading_max = np.abs(plan["psi"]).max(axis=0)
        wx = (np.tile(plan["x"], (m, 1)) - xi_x[:, None]) / a
        wy = (np.tile(plan["y"], (m, 1)) - xi_y[:, None]) / b
        ratios = np.sqrt(wx * wx + wy * wy)
        min_ratio = ratios.min(axis=0) if ratios.size else np.full(l, np.inf)
        res_max = st["history"][-1].max(axis=0)
        ok_heading = heading_max <= heading_limit
        ok_coll = min_ratio >= 1.0 - collision_margin
        feasible = ok_heading & (res_max <= residual_tol) & ok_coll
        costs = []
        for i in range(l):
            v, y = plan["v"][:, i], plan["y"][:, i]
            if kind == "cruise":
                costs.append(float(np.sum((v - v_cruise) ** 2)))
            else:
                costs.append(float(np.sum(w1 * (v - v_max) ** 2 + w2 * (y - y_rl) ** 2)))
        meta = np.array(costs)
        best = int(np.argmin(np.where(feasible, meta, np.inf))) if feasible.any() else None
        hc = ok_heading & ok_coll
        best_hc = int(np.argmin(np.where(hc, meta, np.inf))) if hc.any() else None
        return dict(plan=plan, heading_max=heading_max, min_ratio=min_ratio, feasible=feasible,
                    meta_cost=meta, best_index=best, argmin_all=int(np.argmin(meta)),
                    argmin_heading_collision=best_hc, res_max=res_max)


def solve_scenes(scn, max_iter, kernel="c", tol=0.0, solver=None):
    """Loop single-scene oracle solves over a stacked SceneBatch-like object."""
    solver = solver or OracleSolver(scn.n, scn.t_f, scn.degree, scn.m, scn.rho)
    out = []
    for s in range(scn.S):
        cols = slice(s * scn.l, (s + 1) * scn.l)
        out.append(solver.solve(scn.xi_x[s], scn.xi_y[s], scn.b_xy[:, cols], scn.b_psi[:, cols],
                                scn.a, scn.b, scn.v_min, scn.v_max, scn.a_max, max_iter=max_iter,
                                tol=tol, kernel=kernel))
    return solver, out


def single_thread_blas():
    """Context manager pinning BLAS to one thread (the fair CPU baseline, SURVEY finding 5)."""
    from threadpoolctl import threadpool_limits

    return threadpool_limits(1)


if __name__ == "__main__":  # pragma: no cover
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    s = OracleSolver(100, 10.0, 10, 10)
    print("oracle ok", s.matrix_xy.shape)
