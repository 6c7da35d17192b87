"""Batched alternating-minimization solver -- drop-in for the reference's
``batchmpc.solver`` (/root/reference/pkg/src/batchmpc/solver.py).

Same classes, fields, method names, argument meanings and error behaviour as
the reference; the work runs in one persistent sm_100a kernel per solve
(csrc/am_solve_kernel.cuh) instead of per-iteration numpy/BLAS/LAPACK calls.

Differences by design (B200 formulation, SURVEY.md finding 8):
* ``KktSystem`` holds explicit inverses of the two shared KKT matrices instead
  of LU factors (the step API applies them with one refinement step, as the
  reference's LU solve does).  The persistent solve runs both QPs in
  null-space form (csrc/capi.cu reduced_qp): the boundary rows fix the end
  coefficients once per solve and each sweep applies the reduced-Hessian
  inverse, refined only where that Hessian is ill-conditioned (c4).
  ``n_factorizations`` counts the two inversions, ``n_solves`` two solves per
  AM sweep exactly as the reference's solve_xy/solve_psi calls do.
* the obstacle penalty targets are summed over obstacles before the basis
  contraction (F_o^T g = P^T sum_j g_j), in exact form (an outside term gives
  g_j = x, r_j = 0), and the line-of-sight ratios use rsqrt-and-multiply.
  Trajectories match the reference to <= 1e-8 relative on every column the
  reference's own 1-ulp sensitivity screen marks stable.
"""

from __future__ import annotations

import ctypes
import dataclasses
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .basis import BasisSet, BoundarySpec, ConstantMatrices


@dataclass
class ProblemBatch:
    """Shared scene data plus per-instance boundary vectors (solver.py:26-59)."""

    l: int
    xi_x: np.ndarray
    xi_y: np.ndarray
    a: float
    b: float
    v_min: float
    v_max: float
    a_max: float
    b_xy: np.ndarray
    b_psi: np.ndarray
    rho_xy: float = 1.0

    def __post_init__(self):
        if not 0.0 < self.v_min < self.v_max:
            raise ValueError(f"need 0 < v_min < v_max, got [{self.v_min}, {self.v_max}]")
        if self.a_max <= 0.0:
            raise ValueError(f"a_max must be positive, got {self.a_max}")
        if not self.a >= self.b > 0.0:
            raise ValueError(f"ellipse axes must satisfy a >= b > 0, got ({self.a}, {self.b})")
        if self.rho_xy <= 0.0:
            raise ValueError(f"rho_xy must be positive, got {self.rho_xy}")
        if self.xi_x.shape != self.xi_y.shape:
            raise ValueError("obstacle prediction arrays must have equal shape")
        if self.b_xy.shape[1] != self.l or self.b_psi.shape[1] != self.l:
            raise ValueError("boundary vectors must have one column per instance")


class _Deferred:
    """An AmState field that still lives on the device: materialised on the host
    the first time it is read (solver.py:440-450 builds alpha, d, alpha_a, d_a
    eagerly; at c3/c4 batch sizes those (m*n, L) arrays are gigabytes, so here
    they are only built when someone looks)."""

    __slots__ = ("shape", "_src", "_name")

    def __init__(self, src, name, shape):
        self._src, self._name, self.shape = src, name, tuple(shape)

    def device(self):
        return self._src.device(self._name)

    def host(self) -> np.ndarray:
        return self.device().cpu().numpy()


class _LazyAux:
    """Device source of the deferred AmState fields of one solve: v from the
    last sweep, and alpha, d, alpha_a, d_a re-derived from the final
    coefficients with the closed forms (obstacle_update per scene,
    accel_update), computed together on first use."""

    def __init__(self, solver, sol, prob):
        self.solver, self.sol, self.prob = solver, sol, prob
        self._t = None

    def device(self, name):
        if name == "v":
            return self.sol.v
        if self._t is None:
            import torch

            from . import kernels

            smp = self.solver.sample_device(self.sol, which=("x", "y", "xddot", "yddot"))
            p = self.prob
            n = self.solver.basis.grid.n
            alpha = torch.empty(p.m * n, p.L, dtype=torch.float64, device=p.b_xy.device)
            d = torch.empty_like(alpha)
            for sc in range(p.S):
                cols = slice(sc * p.l, (sc + 1) * p.l)
                alpha[:, cols], d[:, cols] = kernels.obstacle_update(
                    smp["x"][:, cols], smp["y"][:, cols], p.xi_x[sc], p.xi_y[sc], p.a, p.b)
            alpha_a, d_a = kernels.accel_update(smp["xddot"], smp["yddot"], p.a_max)
            self._t = dict(alpha=alpha, d=d, alpha_a=alpha_a, d_a=d_a)
        return self._t[name]


class _History(Sequence):
    """SolveInfo.residual_history: one Residuals per sweep, read from the
    device history on first access (the list the reference builds eagerly,
    solver.py:432-436)."""

    def __init__(self, dev_hist, iterations, final=None):
        # final: host copy of the last sweep's residuals (3, L), so reading
        # history[-1] -- the common case -- does not bring the whole table back
        self._dev, self._n, self._rows, self._final = dev_hist, iterations, None, final

    def _load(self):
        if self._rows is None:
            h = self._dev[: self._n].cpu().numpy()
            self._rows = [Residuals(r_obs=r[0].copy(), r_acc=r[1].copy(), r_nonhol=r[2].copy()) for r in h]
            self._dev = None
        return self._rows

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if (self._rows is None and self._final is not None and isinstance(i, (int, np.integer))
                and self._n > 0 and i in (-1, self._n - 1)):
            r = self._final
            return Residuals(r_obs=r[0].copy(), r_acc=r[1].copy(), r_nonhol=r[2].copy())
        return self._load()[i]

    def __repr__(self):
        return repr(self._load())


@dataclass
class AmState:
    """All per-instance iterates (solver.py:62-94).  Fields a solve leaves on the
    device (v, alpha, d, alpha_a, d_a) are materialised on first read."""

    c_x: np.ndarray
    c_y: np.ndarray
    c_psi: np.ndarray
    alpha: np.ndarray
    d: np.ndarray
    alpha_a: np.ndarray
    d_a: np.ndarray
    v: np.ndarray
    lambda_x: np.ndarray
    lambda_y: np.ndarray
    lambda_psi: np.ndarray
    iteration: int = 0

    def __getattribute__(self, name):
        v = object.__getattribute__(self, name)
        if type(v) is _Deferred:
            v = v.host()
            object.__setattr__(self, name, v)
        return v

    def _raw(self, name):
        """The field without materialising it (ndarray or _Deferred)."""
        return object.__getattribute__(self, name)

    def copy(self) -> "AmState":
        vals = {}
        for f in dataclasses.fields(self):
            v = self._raw(f.name)
            vals[f.name] = v.copy() if isinstance(v, np.ndarray) else v  # a _Deferred is shared
        return AmState(**vals)

    def shapes_match(self, other: "AmState") -> bool:
        for f in dataclasses.fields(self):
            v = self._raw(f.name)
            if isinstance(v, (np.ndarray, _Deferred)) and v.shape != other._raw(f.name).shape:
                return False
        return True


@dataclass
class Residuals:
    """Per-instance L2 norms of the three penalty blocks (solver.py:97-109)."""

    r_obs: np.ndarray
    r_acc: np.ndarray
    r_nonhol: np.ndarray

    def max_per_instance(self) -> np.ndarray:
        return np.maximum(self.r_obs, np.maximum(self.r_acc, self.r_nonhol))

    def overall_max(self) -> float:
        return float(self.max_per_instance().max())


@dataclass
class SolveInfo:
    residual_history: Sequence[Residuals]
    iterations: int
    converged: bool
    iterates: list[tuple[np.ndarray, np.ndarray, np.ndarray]] | None = None


def _single_scene(batch) -> bool:
    """A one-scene batch: this package's ProblemBatch or any object with its
    fields (the reference's own batchmpc.solver.ProblemBatch: 1-D predictions)."""
    return isinstance(batch, ProblemBatch) or np.ndim(batch.xi_x) == 1


def _default_boundary(spec) -> bool:
    """True when ``spec`` pins the default derivative orders.  Compared field by
    field, so a BoundarySpec of the reference's own ``batchmpc.basis`` (another
    class; dataclass equality is per class) is accepted too."""
    d = BoundarySpec()
    keys = ("start_orders", "end_orders", "psi_start_orders", "psi_end_orders")
    try:
        return all(tuple(getattr(spec, k)) == getattr(d, k) for k in keys)
    except AttributeError:
        return False


def _precision_code(precision: str) -> int:
    """"fp64": everything in double (the reference's arithmetic); "fp32": the
    per-sample passes in single precision -- sampling, heading atan2 / unwrap,
    sin/cos, the acceleration, non-holonomic and obstacle blocks and their
    residual contractions -- while the QP steps, the Gram terms of G and the
    multipliers stay fp64 (tolerance in DESIGN.md, tests/test_gpu_solver.py)."""
    codes = {"fp64": 0, "fp32": 1}
    if precision not in codes:
        raise ValueError(f"precision must be one of {sorted(codes)}, got {precision!r}")
    return codes[precision]


def _inverse_ext(K: np.ndarray) -> np.ndarray:
    """Gauss-Jordan inverse with partial pivoting in x87 extended precision,
    rounded once to float64 (the KKT blocks are at most 22 x 22)."""
    n = K.shape[0]
    M = np.concatenate([K.astype(np.longdouble), np.eye(n, dtype=np.longdouble)], axis=1)
    for col in range(n):
        piv = col + int(np.argmax(np.abs(M[col:, col])))
        if M[piv, col] == 0:
            raise np.linalg.LinAlgError("KKT factorization failed: singular matrix")
        if piv != col:
            M[[col, piv]] = M[[piv, col]]
        M[col] /= M[col, col]
        others = np.arange(n) != col
        M[others] -= M[others, col:col + 1] * M[col]
    inv = M[:, n:].astype(np.float64)
    if not np.isfinite(inv).all():
        raise np.linalg.LinAlgError("KKT factorization failed: non-finite inverse")
    return inv


class KktSystem:
    """The two shared KKT matrices (solver.py:120-176), kept as explicit inverses.

    ``matrix_xy``/``matrix_psi`` are assembled exactly as the reference does
    (bitwise); the device applies rows 0..n_b-1 of the per-axis inverse (the
    x and y blocks of matrix_xy are identical and uncoupled) and of the heading
    inverse.  ``solve_xy``/``solve_psi`` are host conveniences with the
    reference's signatures.
    """

    def __init__(self, mats: ConstantMatrices, rho_xy: float):
        nb = mats.basis.n_b
        P = mats.basis.P
        r_xy = mats.A.shape[0]
        r_psi = mats.A_psi.shape[0]
        H = np.zeros((2 * nb, 2 * nb))
        H[:nb, :nb] = mats.Q + rho_xy * (mats.F_axis.T @ mats.F_axis)
        H[nb:, nb:] = H[:nb, :nb]
        K = np.zeros((2 * nb + r_xy, 2 * nb + r_xy))
        K[: 2 * nb, : 2 * nb] = H
        K[: 2 * nb, 2 * nb:] = mats.A.T
        K[2 * nb:, : 2 * nb] = mats.A
        Kp = np.zeros((nb + r_psi, nb + r_psi))
        Kp[:nb, :nb] = mats.Q + rho_xy * (P.T @ P)
        Kp[:nb, nb:] = mats.A_psi.T
        Kp[nb:, :nb] = mats.A_psi
        self.matrix_xy, self.matrix_psi = K, Kp
        self.n_factorizations = 0
        self.n_solves = 0
        ra = mats.A_axis.shape[0]
        axis = np.r_[0:nb, 2 * nb:2 * nb + ra]
        self.matrix_axis = K[np.ix_(axis, axis)]
        self.ftf_axis = mats.F_axis.T @ mats.F_axis
        self.inv_xy = self._invert(K)
        self.inv_axis = self._invert_quiet(self.matrix_axis)
        self.inv_psi = self._invert(Kp)
        self.kinv_axis = np.ascontiguousarray(self.inv_axis[:nb])   # (nb, nb + 6)
        self.kinv_psi = np.ascontiguousarray(self.inv_psi[:nb])     # (nb, nb + 4)
        self.matrix_xy.setflags(write=False)
        self.matrix_psi.setflags(write=False)

    def _invert(self, K):
        self.n_factorizations += 1
        return _inverse_ext(K)

    @staticmethod
    def _invert_quiet(K):
        return _inverse_ext(K)

    def solve_xy(self, rhs: np.ndarray) -> np.ndarray:
        self.n_solves += 1
        return self.inv_xy @ rhs

    def solve_psi(self, rhs: np.ndarray) -> np.ndarray:
        self.n_solves += 1
        return self.inv_psi @ rhs


class BatchSolver:
    """Algorithm driver (solver.py:179-500) on one B200.

    The device context (constants in HBM) is created lazily on first use, so
    the solver can be built and inspected on a host without a GPU.
    """

    def __init__(self, basis: BasisSet, mats: ConstantMatrices, rho_xy: float = 1.0):
        if mats.basis is not basis:
            raise ValueError("constant matrices were built from a different basis")
        if not _default_boundary(mats.boundary):
            raise ValueError("the device path supports the default BoundarySpec only")
        if not 6 <= basis.n_b <= 16:
            raise ValueError(f"basis size {basis.n_b} outside the supported 6..16")
        if not 2 <= basis.grid.n <= 256:
            raise ValueError(f"horizon samples {basis.grid.n} outside the supported 2..256")
        self.basis = basis
        self.mats = mats
        self.rho_xy = rho_xy
        self.kkt = KktSystem(mats, rho_xy)
        self._P_pinv = np.linalg.pinv(basis.P)
        self._sample_all = np.vstack([basis.P, basis.Pdot, basis.Pddot])
        g = basis.grid
        self._tau = np.ascontiguousarray((g.times - g.t0) / (g.tf - g.t0))
        self._ctxs = {}  # device index -> bmpc_ctx (constants uploaded once per device)

    # -- device context ------------------------------------------------------
    def _context(self):
        """The C-ABI context of the current CUDA device (created on first use)."""
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("BatchSolver needs a CUDA device (sm_100a); there is no CPU fallback")
        dev = torch._C._cuda_getDevice()
        c = self._ctxs.get(dev)
        if c is not None:
            return c
        lib = nat.load()
        c = ctypes.c_void_p()
        b = self.basis
        arrs = [np.ascontiguousarray(a, dtype=np.float64)
                for a in (b.P, b.Pdot, b.Pddot, self._tau, self.kkt.inv_axis, self.kkt.matrix_axis,
                          self.kkt.inv_psi, self.kkt.matrix_psi, self.kkt.ftf_axis)]
        nat.check(lib.bmpc_ctx_create(b.grid.n, b.n_b, float(self.rho_xy),
                                      *[nat.c_double_ptr(a) for a in arrs], ctypes.byref(c)),
                  "bmpc_ctx_create")
        self._ctxs[dev] = c
        return c

    def qp_info(self) -> dict:
        """Null-space QP form of the device solve: the 1-norm condition numbers
        of the reduced xy / psi Hessians and whether each QP step refines."""
        c = self._context()
        cx, cp, rf = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
        nat.check(nat.load().bmpc_ctx_qp_info(c, ctypes.byref(cx), ctypes.byref(cp), ctypes.byref(rf)),
                  "bmpc_ctx_qp_info")
        return {"cond_xy": cx.value, "cond_psi": cp.value, "refine_xy": bool(rf.value & 1),
                "refine_psi": bool(rf.value & 2)}

    def __del__(self):
        try:
            lib = nat.load()
            for c in self.__dict__.get("_ctxs", {}).values():
                lib.bmpc_ctx_destroy(c)
        except Exception:
            pass

    @staticmethod
    def _on_current_device(t, what="problem"):
        import torch

        cur = torch._C._cuda_getDevice()
        if t.device.type != "cuda" or t.device.index != cur:
            raise ValueError(f"the {what} lives on {t.device} but the current device is cuda:{cur}; "
                             "select it with torch.cuda.set_device / torch.cuda.device first")

    # -- validation ---------------------------------------------------------
    def _check_batch(self, batch: ProblemBatch):
        mn = self.mats.rows_obs
        if batch.xi_x.shape != (mn,):
            raise ValueError(f"expected obstacle predictions of shape ({mn},), got {batch.xi_x.shape}")
        if batch.b_xy.shape[0] != self.mats.A.shape[0]:
            raise ValueError(
                f"b_xy has {batch.b_xy.shape[0]} rows but the boundary matrix has {self.mats.A.shape[0]}")
        if batch.b_psi.shape[0] != self.mats.A_psi.shape[0]:
            raise ValueError(
                f"b_psi has {batch.b_psi.shape[0]} rows but the heading boundary matrix has "
                f"{self.mats.A_psi.shape[0]}")
        if batch.rho_xy != self.rho_xy:
            raise ValueError("batch.rho_xy differs from the rho the KKT inverses were built with")

    def _zero_state(self, batch: ProblemBatch) -> AmState:
        nb, l, n = self.basis.n_b, batch.l, self.basis.grid.n
        mn = batch.xi_x.shape[0]
        z = np.zeros
        return AmState(c_x=z((nb, l)), c_y=z((nb, l)), c_psi=z((nb, l)),
                       alpha=z((mn, l)), d=np.ones((mn, l)),
                       alpha_a=z((n, l)), d_a=z((n, l)), v=z((n, l)),
                       lambda_x=z((nb, l)), lambda_y=z((nb, l)), lambda_psi=z((nb, l)))

    # -- device plumbing ------------------------------------------------------
    def device_problem(self, batch: ProblemBatch, non_blocking: bool = False):
        from .device import DeviceProblem

        return DeviceProblem.from_host(self.basis.grid.n, batch.xi_x[None, :], batch.xi_y[None, :],
                                       batch.b_xy, batch.b_psi, batch.l, batch.a, batch.b,
                                       batch.v_min, batch.v_max, batch.a_max,
                                       non_blocking=non_blocking)

    def solve_device(self, prob, max_iter: int = 150, tol: float = 1e-3, warm: dict | None = None,
                     keep_multipliers: bool = False, want_v: bool = True, warps_per_block: int = 0,
                     precision: str = "fp64", warm_mask=None, team_warps: int = 0):
        """Solve a DeviceProblem (one or many scenes) with every buffer in HBM.

        ``warm`` maps AmState field names to device tensors; ``warm_mask`` (L
        uint8 device tensor, optional) limits the warm start to the instances
        it marks, the others start cold.  Returns a device.DeviceSolution;
        blocks only to learn the sweep count.
        """
        import torch

        from . import device as D

        if max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {max_iter}")
        self._on_current_device(prob.b_xy)
        ctx = self._context()
        dev = prob.b_xy.device
        sol = D.alloc_solution(self.basis.n_b, self.basis.grid.n, prob.L, max_iter, want_v, dev)
        opts = nat.SolveOpts(max_iter=int(max_iter), tol=float(tol),
                             keep_multipliers=int(bool(keep_multipliers)),
                             warps_per_block=int(warps_per_block), want_v=int(bool(want_v)),
                             precision=_precision_code(precision), team_warps=int(team_warps))
        if warm is not None:
            for fld, key in (("w_alpha", "alpha"), ("w_d", "d"), ("w_alpha_a", "alpha_a"),
                             ("w_d_a", "d_a"), ("w_v", "v"), ("w_c_psi", "c_psi"),
                             ("w_l_x", "lambda_x"), ("w_l_y", "lambda_y"), ("w_l_psi", "lambda_psi")):
                setattr(opts, fld, warm[key].data_ptr())
            if warm_mask is not None:
                opts.w_mask = warm_mask.data_ptr()
        out = D.solution_struct(sol)
        nat.check(nat.load().bmpc_solve(ctx, ctypes.byref(prob.c_struct()), ctypes.byref(opts),
                                        ctypes.byref(out), ctypes.c_void_p(D.stream_ptr())), "solve")
        sol.iterations, sol.converged = out.iterations, bool(out.converged)
        self.kkt.n_solves += 2 * sol.iterations
        del torch
        return sol

    def sample_device(self, sol, which=("x", "y", "xdot", "ydot", "xddot", "yddot", "psi",
                                        "psidot", "v")):
        """(n, L) samples of the solved coefficients on the device."""
        import torch

        from . import device as D

        ctx = self._context()
        L = sol.c_x.shape[1]
        n = self.basis.grid.n
        out = {k: torch.empty(n, L, dtype=torch.float64, device=sol.c_x.device) for k in which}
        names = ("x", "y", "xdot", "ydot", "xddot", "yddot", "psi", "psidot", "v")
        args = [D.ptr(out.get(k)) for k in names]
        nat.check(nat.load().bmpc_sample(ctx, L, D.ptr(sol.c_x), D.ptr(sol.c_y), D.ptr(sol.c_psi),
                                         *args, ctypes.c_void_p(D.stream_ptr())), "sample")
        return out

    # -- reference API ----------------------------------------------------------
    def init_state(self, batch: ProblemBatch, warm: AmState | None = None,
                   keep_multipliers: bool = False) -> AmState:
        """Cold start from straight start->goal lines, or a copy of a warm state
        (solver.py:197-252)."""
        self._check_batch(batch)
        if warm is not None:
            if not warm.shapes_match(self._zero_state(batch)):
                raise ValueError("warm state shapes do not match the batch")
            state = warm.copy()
            if not keep_multipliers:
                for lam in (state.lambda_x, state.lambda_y, state.lambda_psi):
                    lam.fill(0.0)
            state.iteration = 0
            return state
        from . import kernels

        n, l = self.basis.grid.n, batch.l
        bnd = self.mats.boundary
        rpa = bnd.rows_per_axis
        i0, i1, iv = bnd.row_index("t0", 0), bnd.row_index("tf", 0), bnd.row_index("t0", 1)
        x0, xf = batch.b_xy[i0], batch.b_xy[i1]
        y0, yf = batch.b_xy[rpa + i0], batch.b_xy[rpa + i1]
        vx0, vy0 = batch.b_xy[iv], batch.b_xy[rpa + iv]
        tau = self._tau
        x_line = x0[None, :] + tau[:, None] * (xf - x0)[None, :]
        y_line = y0[None, :] + tau[:, None] * (yf - y0)[None, :]
        state = self._zero_state(batch)
        state.c_x = self._P_pinv @ x_line
        state.c_y = self._P_pinv @ y_line
        speed0 = np.clip(np.sqrt(vx0 * vx0 + vy0 * vy0), batch.v_min, batch.v_max)
        state.v = np.broadcast_to(speed0, (n, l)).copy()
        state.alpha, state.d = kernels.obstacle_update(x_line, y_line, batch.xi_x, batch.xi_y,
                                                       batch.a, batch.b)
        return state

    def solve(self, batch: ProblemBatch, max_iter: int = 150, tol: float = 1e-3,
              warm: AmState | None = None, record_iterates: bool = False,
              keep_multipliers: bool = False) -> tuple[AmState, SolveInfo]:
        """Run the alternating minimization until every instance's worst residual
        is <= tol or max_iter sweeps ran (solver.py:414-456).  Host arrays in,
        host arrays out.

        ``batch`` is a ProblemBatch (one scene, as in the reference) or a stacked
        scene batch (scenes.SceneBatch: xi_x/xi_y (S, m*n), b_xy (12, S*l),
        b_psi (4, S*l); instance s*l + i is goal i of scene s).  The returned
        AmState's coefficients and multipliers are host arrays; v, alpha, d,
        alpha_a and d_a stay on the device until first read (the reference
        materialises them at the end of every solve, solver.py:440-450), and the
        residual history is read back on first access."""
        import torch

        if max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {max_iter}")
        prob = self._problem(batch)
        dev = prob.b_xy.device
        wd = None
        if warm is not None:
            if not warm.shapes_match(self._zero_shapes(prob)):
                raise ValueError("warm state shapes do not match the batch")
            wd = {}
            for k in ("alpha", "d", "alpha_a", "d_a", "v", "c_psi", "lambda_x", "lambda_y", "lambda_psi"):
                raw = warm._raw(k)
                wd[k] = (raw.device().contiguous() if isinstance(raw, _Deferred) else
                         torch.from_numpy(np.ascontiguousarray(raw, dtype=np.float64)).to(dev))
        iterates = None
        if record_iterates:
            sol, iterates = self._solve_stepwise(prob, max_iter, tol, wd, keep_multipliers)
        else:
            sol = self.solve_device(prob, max_iter, tol, wd, keep_multipliers)
        aux = _LazyAux(self, sol, prob)
        n, L, mn = self.basis.grid.n, prob.L, prob.m * self.basis.grid.n
        nb = self.basis.n_b
        # c_x, c_y, c_psi, l_x, l_y, l_psi and the final residuals in one copy into
        # page-locked memory (torch caches the block; pageable copies run at a
        # tenth of the link rate); the arrays returned are views of it
        blk = torch.empty(sol.block.shape, dtype=torch.float64, pin_memory=True).copy_(sol.block).numpy()
        coef, final = blk[: 6 * nb].reshape(6, nb, L), blk[6 * nb:]
        # The reference's QP solves run through scipy's lu_solve (solver.py:166),
        # whose finite check raises on the first non-finite right-hand side.  A
        # non-finite right-hand side poisons its instance for good (NaN
        # coefficients, samples and residuals), so the final residuals tell: the
        # same error, raised after the solve (3 L values to look at, not the inputs).
        if not np.isfinite(final).all():
            raise ValueError("array must not contain infs or NaNs")
        state = AmState(c_x=coef[0], c_y=coef[1], c_psi=coef[2],
                        alpha=_Deferred(aux, "alpha", (mn, L)), d=_Deferred(aux, "d", (mn, L)),
                        alpha_a=_Deferred(aux, "alpha_a", (n, L)), d_a=_Deferred(aux, "d_a", (n, L)),
                        v=_Deferred(aux, "v", (n, L)), lambda_x=coef[3], lambda_y=coef[4],
                        lambda_psi=coef[5], iteration=sol.iterations)
        return state, SolveInfo(residual_history=_History(sol.history, sol.iterations, final),
                                iterations=sol.iterations, converged=sol.converged, iterates=iterates)

    def check_scenes(self, batch):
        """Validate a ProblemBatch or a stacked scene batch against this solver's
        shapes (the reference's checks, solver.py:47-59, :266-277, applied per
        scene); returns (xi_x (S, m*n), xi_y, S, l)."""
        if _single_scene(batch):
            self._check_batch(batch)
            return np.asarray(batch.xi_x)[None, :], np.asarray(batch.xi_y)[None, :], 1, batch.l
        mn = self.mats.rows_obs
        S, l = int(batch.S), int(batch.l)
        xi_x, xi_y = np.atleast_2d(batch.xi_x), np.atleast_2d(batch.xi_y)
        if S < 1 or l < 0:
            raise ValueError(f"need S >= 1 scenes and l >= 0 goals, got S={S}, l={l}")
        if xi_x.shape != (S, mn) or xi_y.shape != (S, mn):
            raise ValueError(f"expected obstacle predictions of shape ({S}, {mn}), got {xi_x.shape} "
                             f"and {xi_y.shape}")
        if np.shape(batch.b_xy) != (self.mats.A.shape[0], S * l):
            raise ValueError(f"b_xy must have shape ({self.mats.A.shape[0]}, {S * l}), got "
                             f"{np.shape(batch.b_xy)}")
        if np.shape(batch.b_psi) != (self.mats.A_psi.shape[0], S * l):
            raise ValueError(f"b_psi must have shape ({self.mats.A_psi.shape[0]}, {S * l}), got "
                             f"{np.shape(batch.b_psi)}")
        rho = getattr(batch, "rho", getattr(batch, "rho_xy", self.rho_xy))
        if rho != self.rho_xy:
            raise ValueError("batch rho differs from the rho the KKT inverses were built with")
        ProblemBatch(l=S * l, xi_x=xi_x[0], xi_y=xi_y[0], a=batch.a, b=batch.b, v_min=batch.v_min,
                     v_max=batch.v_max, a_max=batch.a_max, b_xy=np.asarray(batch.b_xy),
                     b_psi=np.asarray(batch.b_psi))  # scalar checks
        return xi_x, xi_y, S, l

    def _problem(self, batch):
        """Validated DeviceProblem of a ProblemBatch or a stacked scene batch."""
        if _single_scene(batch):
            self._check_batch(batch)
            return self.device_problem(batch)
        from .device import DeviceProblem

        xi_x, xi_y, S, l = self.check_scenes(batch)
        return DeviceProblem.from_host(self.basis.grid.n, xi_x, xi_y, batch.b_xy, batch.b_psi, l, batch.a,
                                       batch.b, batch.v_min, batch.v_max, batch.a_max)

    def _zero_shapes(self, prob) -> AmState:
        """Shape-only AmState of a problem (no allocation)."""
        nb, n, L, mn = self.basis.n_b, self.basis.grid.n, prob.L, prob.m * self.basis.grid.n
        z = lambda *sh: _Deferred(None, "", sh)  # noqa: E731
        return AmState(c_x=z(nb, L), c_y=z(nb, L), c_psi=z(nb, L), alpha=z(mn, L), d=z(mn, L),
                       alpha_a=z(n, L), d_a=z(n, L), v=z(n, L), lambda_x=z(nb, L), lambda_y=z(nb, L),
                       lambda_psi=z(nb, L))

    def _solve_stepwise(self, prob, max_iter, tol, wd, keep_multipliers):
        """One launch per sweep through the carried-state API, so every
        iterate can be recorded; numerically identical to a single launch."""
        import torch

        from . import device as D

        ctx = self._context()
        nb, n, L = self.basis.n_b, self.basis.grid.n, prob.L
        dev = prob.b_xy.device
        sol = D.alloc_solution(nb, n, L, max_iter, True, dev)
        carry = torch.empty(L, nat.load().bmpc_carry_doubles(ctx), dtype=torch.float64, device=dev)
        opts = nat.SolveOpts(max_iter=int(max_iter), tol=float(tol),
                             keep_multipliers=int(bool(keep_multipliers)), want_v=1)
        if wd is not None:
            for fld, key in (("w_alpha", "alpha"), ("w_d", "d"), ("w_alpha_a", "alpha_a"),
                             ("w_d_a", "d_a"), ("w_v", "v"), ("w_c_psi", "c_psi"),
                             ("w_l_x", "lambda_x"), ("w_l_y", "lambda_y"), ("w_l_psi", "lambda_psi")):
                setattr(opts, fld, wd[key].data_ptr())
        out = D.solution_struct(sol)
        lib = nat.load()
        iterates = []
        converged = False
        it = 0
        for t in range(max_iter):
            nat.check(lib.bmpc_sweeps(ctx, ctypes.byref(prob.c_struct()), ctypes.byref(opts), 1,
                                      int(t > 0), t, ctypes.c_void_p(carry.data_ptr()), 1,
                                      ctypes.byref(out), ctypes.c_void_p(D.stream_ptr())), "sweeps")
            it += 1
            iterates.append((sol.c_x.cpu().numpy().copy(), sol.c_y.cpu().numpy().copy(),
                             sol.c_psi.cpu().numpy().copy()))
            if float(sol.history[t].max()) <= tol:
                converged = True
                break
        sol.iterations, sol.converged = it, converged
        self.kkt.n_solves += 2 * it
        return sol, iterates

    # -- step-wise API (solver.py:288-410) --------------------------------------
    # The same math as the fused sweep, one reference step at a time, on host
    # AmState arrays; every step runs on the device (csrc/steps.cu, csrc/ops.cu).
    def _dev(self, a):
        import torch

        self._context()
        return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()

    def _samples(self, state: AmState, which):
        from .device import DeviceSolution

        d = self._dev
        sol = DeviceSolution(d(state.c_x), d(state.c_y), d(state.c_psi), None, None, None, None,
                             None, None, 0, False)
        return self.sample_device(sol, which=which)

    def _project(self, g, mode: int, m: int):
        import torch

        from .device import stream_ptr

        g = self._dev(g) if isinstance(g, np.ndarray) else g.contiguous()
        L = g.shape[1]
        out = torch.empty(self.basis.n_b, L, dtype=torch.float64, device=g.device)
        nat.check(nat.load().bmpc_project(self._context(), mode, m, L, g.data_ptr(), out.data_ptr(),
                                          ctypes.c_void_p(stream_ptr())), "project")
        return out

    def _heading(self, c_x, c_y):
        import torch

        from .device import stream_ptr

        L = c_x.shape[1]
        th = torch.empty(self.basis.grid.n, L, dtype=torch.float64, device=c_x.device)
        nat.check(nat.load().bmpc_heading(self._context(), L, c_x.data_ptr(), c_y.data_ptr(),
                                          th.data_ptr(), ctypes.c_void_p(stream_ptr())), "heading")
        return th

    def _g_parts(self, state: AmState, batch: ProblemBatch):
        """Penalty targets of a state (solver.py:281-286)."""
        from . import kernels

        psi = self._samples(state, ("psi",))["psi"]
        d = self._dev
        return kernels.assemble_g(d(batch.xi_x), d(batch.xi_y), d(state.alpha), d(state.d),
                                  d(state.alpha_a), d(state.d_a), d(state.v), psi, batch.a, batch.b)

    def build_g(self, state: AmState, batch: ProblemBatch) -> np.ndarray:
        g_x, g_y = self._g_parts(state, batch)
        return np.vstack([g_x.cpu().numpy(), g_y.cpu().numpy()])

    def step_xy(self, state: AmState, batch: ProblemBatch):
        """Equality-constrained QP update of c_x, c_y (solver.py:295-312)."""
        g_x, g_y = self._g_parts(state, batch)
        self._apply_xy(state, batch, g_x, g_y)
        return state.c_x, state.c_y

    def _apply_xy(self, state, batch, g_x, g_y):
        import torch

        from .device import stream_ptr

        nb, l, m = self.basis.n_b, batch.l, self.mats.m
        rho = batch.rho_xy
        rhs = torch.empty(2 * nb + 12, l, dtype=torch.float64, device="cuda")
        rhs[:nb] = rho * self._project(g_x, 0, m) + self._dev(state.lambda_x)
        rhs[nb:2 * nb] = rho * self._project(g_y, 0, m) + self._dev(state.lambda_y)
        rhs[2 * nb:] = self._dev(batch.b_xy)
        cx = torch.empty(nb, l, dtype=torch.float64, device="cuda")
        cy = torch.empty_like(cx)
        nat.check(nat.load().bmpc_kkt_apply(self._context(), 0, l, rhs.data_ptr(), cx.data_ptr(),
                                            cy.data_ptr(), ctypes.c_void_p(stream_ptr())), "kkt")
        self.kkt.n_solves += 1
        state.c_x, state.c_y = cx.cpu().numpy(), cy.cpu().numpy()

    def step_psi(self, state: AmState, batch: ProblemBatch) -> np.ndarray:
        """Heading QP on the unwrapped velocity angle (solver.py:314-328)."""
        th = self._heading(self._dev(state.c_x), self._dev(state.c_y))
        self._apply_psi(state, batch, th)
        return state.c_psi

    def _apply_psi(self, state, batch, theta):
        import torch

        from .device import stream_ptr

        nb, l = self.basis.n_b, batch.l
        theta = self._dev(theta) if isinstance(theta, np.ndarray) else theta
        rhs = torch.empty(nb + 4, l, dtype=torch.float64, device="cuda")
        rhs[:nb] = batch.rho_xy * self._project(theta, 1, 0) + self._dev(state.lambda_psi)
        rhs[nb:] = self._dev(batch.b_psi)
        cp = torch.empty(nb, l, dtype=torch.float64, device="cuda")
        nat.check(nat.load().bmpc_kkt_apply(self._context(), 1, l, rhs.data_ptr(), cp.data_ptr(),
                                            None, ctypes.c_void_p(stream_ptr())), "kkt")
        self.kkt.n_solves += 1
        state.c_psi = cp.cpu().numpy()

    def step_v(self, state: AmState, batch: ProblemBatch) -> np.ndarray:
        from . import kernels

        s = self._samples(state, ("xdot", "ydot"))
        state.v = kernels.v_update(s["xdot"], s["ydot"], batch.v_min, batch.v_max).cpu().numpy()
        return state.v

    def step_alpha_obs(self, state: AmState, batch: ProblemBatch) -> np.ndarray:
        from . import kernels

        s = self._samples(state, ("x", "y"))
        alpha, _ = kernels.obstacle_update(s["x"], s["y"], self._dev(batch.xi_x), self._dev(batch.xi_y),
                                           batch.a, batch.b)
        state.alpha = alpha.cpu().numpy()
        return state.alpha

    def step_d_obs(self, state: AmState, batch: ProblemBatch) -> np.ndarray:
        """1-D bound-constrained QP over each separation ratio, given alpha."""
        import torch

        from .device import stream_ptr

        s = self._samples(state, ("x", "y"))
        n, l = s["x"].shape
        mn = batch.xi_x.shape[0]
        al = self._dev(state.alpha)
        d = torch.empty(mn, l, dtype=torch.float64, device="cuda")
        xi_x, xi_y = self._dev(batch.xi_x), self._dev(batch.xi_y)
        nat.check(nat.load().bmpc_op_d_obs(n, l, mn, s["x"].data_ptr(), s["y"].data_ptr(),
                                           xi_x.data_ptr(), xi_y.data_ptr(), al.data_ptr(),
                                           float(batch.a), float(batch.b), d.data_ptr(),
                                           ctypes.c_void_p(stream_ptr())), "d_obs")
        state.d = d.cpu().numpy()
        return state.d

    def step_alpha_acc(self, state: AmState, batch: ProblemBatch) -> np.ndarray:
        from . import kernels

        s = self._samples(state, ("xddot", "yddot"))
        state.alpha_a = kernels.accel_update(s["xddot"], s["yddot"], batch.a_max)[0].cpu().numpy()
        return state.alpha_a

    def step_d_acc(self, state: AmState, batch: ProblemBatch) -> np.ndarray:
        from . import kernels

        s = self._samples(state, ("xddot", "yddot"))
        state.d_a = kernels.accel_update(s["xddot"], s["yddot"], batch.a_max)[1].cpu().numpy()
        return state.d_a

    def _residual_parts(self, state: AmState, batch: ProblemBatch):
        from . import kernels

        s = self._samples(state, ("x", "y", "xdot", "ydot", "xddot", "yddot", "psi"))
        d = self._dev
        return kernels.residual_vectors(s["x"], s["y"], s["xdot"], s["ydot"], s["xddot"], s["yddot"],
                                        s["psi"], d(batch.xi_x), d(batch.xi_y), d(state.alpha),
                                        d(state.d), d(state.alpha_a), d(state.d_a), d(state.v),
                                        batch.a, batch.b)

    def update_multipliers(self, state: AmState, batch: ProblemBatch) -> None:
        """Gradient-style multiplier update on the current residuals (solver.py:368-378)."""
        r_x, r_y = self._residual_parts(state, batch)
        m, rho = self.mats.m, batch.rho_xy
        state.lambda_x = state.lambda_x - rho * self._project(r_x, 0, m).cpu().numpy()
        state.lambda_y = state.lambda_y - rho * self._project(r_y, 0, m).cpu().numpy()
        dc = self._dev
        th = self._heading(dc(state.c_x), dc(state.c_y))
        psi = self._samples(state, ("psi",))["psi"]
        state.lambda_psi = state.lambda_psi - rho * self._project(psi - th, 1, 0).cpu().numpy()

    def _iterate(self, state: AmState, batch: ProblemBatch, g_x, g_y):
        """One full sweep on a host AmState through the device step operators
        (solver.py:458-500): xy QP, sampling, unwrap(atan2) heading target, psi
        QP, the fused tail (d, d_a, v, residual vectors, next targets) and the
        multiplier steps.  ``g_x``/``g_y`` are the incoming targets (as
        ``_g_parts`` returns them, device arrays); returns (Residuals, next
        g_x, next g_y).  The persistent kernel fuses all of this for solve()."""
        from . import kernels

        self._apply_xy(state, batch, g_x, g_y)
        d = self._dev
        cx, cy = d(state.c_x), d(state.c_y)
        s = self._samples(state, ("x", "y", "xdot", "ydot", "xddot", "yddot"))
        theta = self._heading(cx, cy)
        self._apply_psi(state, batch, theta)
        psi = self._samples(state, ("psi",))["psi"]
        (dd, d_a, v, r_x, r_y, g_x2, g_y2, sq_obs, sq_acc, sq_nonhol) = kernels.tail_core(
            s["x"], s["y"], s["xdot"], s["ydot"], s["xddot"], s["yddot"], psi, d(batch.xi_x),
            d(batch.xi_y), batch.v_min, batch.v_max, batch.a_max, batch.a, batch.b)
        state.d, state.d_a, state.v = dd.cpu().numpy(), d_a.cpu().numpy(), v.cpu().numpy()
        m, rho = self.mats.m, batch.rho_xy
        state.lambda_x = state.lambda_x - rho * self._project(r_x, 0, m).cpu().numpy()
        state.lambda_y = state.lambda_y - rho * self._project(r_y, 0, m).cpu().numpy()
        state.lambda_psi = state.lambda_psi - rho * self._project(psi - theta, 1, 0).cpu().numpy()
        state.iteration += 1
        h = lambda t: np.sqrt(t.cpu().numpy())  # noqa: E731
        return Residuals(r_obs=h(sq_obs), r_acc=h(sq_acc), r_nonhol=h(sq_nonhol)), g_x2, g_y2

    def compute_residuals(self, state: AmState, batch: ProblemBatch) -> Residuals:
        """Block L2 norms of the residual vectors (solver.py:392-410)."""
        import torch

        from .device import stream_ptr

        r_x, r_y = self._residual_parts(state, batch)
        n, l = self.basis.grid.n, batch.l
        mn = batch.xi_x.shape[0]
        out = torch.empty(3, l, dtype=torch.float64, device=r_x.device)
        nat.check(nat.load().bmpc_block_norms(n, l, mn, r_x.data_ptr(), r_y.data_ptr(),
                                              out.data_ptr(), ctypes.c_void_p(stream_ptr())), "norms")
        o = out.cpu().numpy()
        return Residuals(r_obs=o[0], r_acc=o[1], r_nonhol=o[2])
