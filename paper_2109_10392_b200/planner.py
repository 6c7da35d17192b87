"""Planner-level API: goal batch in, ranked trajectories + meta costs out.

Mirrors the scoring half of the reference planner
(/root/reference/pkg/src/batchmpc/planner.py): ``MetaCostSpec``,
``FilterLimits``, ``RankedPlan``, ``meta_cost``, ``collision_ratios``,
``filter_candidates``, ``rank``, ``Planner.build_batch``/``boundary_vectors``/
``sample_plan``.  Sampling, the collision/heading/residual filters, meta costs
and the argmin (ties -> lowest index, ``None`` when nothing is feasible) run in
the fused sm_100a scoring kernel (csrc/ops.cu: k_score, k_argmin).

``plan_batch`` is the one-call hot path used by the benchmark: host arrays in,
solve + score through the C ABI (``bmpc_plan_host``), host results out.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .basis import BoundarySpec, build_basis, build_constant_matrices, build_time_grid
from .solver import AmState, BatchSolver, ProblemBatch, Residuals, SolveInfo, _precision_code
from .traffic import VehicleState, predict_constant_velocity, select_nearest


@dataclass
class EgoState:
    x: float
    y: float
    psi: float = 0.0
    psidot: float = 0.0
    vx: float = 0.0
    vy: float = 0.0
    ax: float = 0.0
    ay: float = 0.0

    @property
    def speed(self) -> float:
        return math.hypot(self.vx, self.vy)


@dataclass
class Goal:
    x: float
    y: float
    vx: float
    vy: float
    ax: float
    ay: float
    lane: int


@dataclass(frozen=True)
class MetaCostSpec:
    """Task-level scoring (planner.py:78-93)."""

    kind: str
    v_cruise: float = 15.0
    v_max: float = 20.0
    y_rl: float = 0.0
    w1: float = 1.0
    w2: float = 1.0

    def __post_init__(self):
        if self.kind not in ("cruise", "highspeed"):
            raise ValueError(f"unknown meta-cost kind {self.kind!r}")
        if self.w1 < 0 or self.w2 < 0:
            raise ValueError("meta-cost weights must be nonnegative")


@dataclass(frozen=True)
class FilterLimits:
    heading_limit: float = math.radians(13.0)
    residual_tol: float = 1e-3
    collision_margin: float = 0.01


@dataclass
class Candidate:
    x: np.ndarray
    y: np.ndarray
    psi: np.ndarray
    psidot: np.ndarray
    v: np.ndarray
    xddot: np.ndarray
    yddot: np.ndarray


@dataclass
class RankedPlan:
    """Sampled candidates, filter results, costs and the selection (planner.py:162-194)."""

    goals: list
    x: np.ndarray
    y: np.ndarray
    psi: np.ndarray
    psidot: np.ndarray
    v: np.ndarray
    xddot: np.ndarray
    yddot: np.ndarray
    residuals: Residuals
    min_ratio: np.ndarray = field(default=None)
    heading_max: np.ndarray = field(default=None)
    feasible: np.ndarray = field(default=None)
    meta_cost: np.ndarray = field(default=None)
    best_index: int | None = None
    _dev: dict = field(default=None, repr=False)  # device coefficients for the fused kernels

    @property
    def l(self) -> int:
        return self.x.shape[1]

    def candidate(self, i: int) -> Candidate:
        return Candidate(x=self.x[:, i], y=self.y[:, i], psi=self.psi[:, i],
                         psidot=self.psidot[:, i], v=self.v[:, i], xddot=self.xddot[:, i],
                         yddot=self.yddot[:, i])

    def best(self) -> Candidate:
        if self.best_index is None:
            raise ValueError("no feasible candidate was selected")
        return self.candidate(self.best_index)


def _spec_struct(spec: MetaCostSpec | None, limits: FilterLimits) -> nat.ScoreSpec:
    spec = spec or MetaCostSpec("cruise")
    return nat.ScoreSpec(0 if spec.kind == "cruise" else 1, spec.v_cruise, spec.v_max, spec.y_rl,
                         spec.w1, spec.w2, limits.heading_limit, limits.residual_tol,
                         limits.collision_margin)


def meta_cost(traj: Candidate, spec: MetaCostSpec) -> float:
    """Scalar meta cost of one candidate (planner.py:210-216).  Per-candidate
    helper only; batched scoring runs in the fused kernel (``rank``)."""
    if spec.kind == "cruise":
        return float(np.sum((traj.v - spec.v_cruise) ** 2))
    return float(np.sum(spec.w1 * (traj.v - spec.v_max) ** 2 + spec.w2 * (traj.y - spec.y_rl) ** 2))


def collision_ratios(x, y, xi_x, xi_y, a, b):
    """(m*n, l) ellipse separation ratios recomputed from positions (planner.py:219-230)."""
    import torch

    from .device import stream_ptr

    A = [torch.as_tensor(np.asarray(t, dtype=np.float64) if not isinstance(t, torch.Tensor) else t)
         for t in (x, y, xi_x, xi_y)]
    host = not A[0].is_cuda
    dev = torch.device("cuda", torch.cuda.current_device())
    x, y, xi_x, xi_y = (t.to(dev, dtype=torch.float64).contiguous() for t in A)
    n, l = x.shape
    m = xi_x.shape[0] // n if n else 0
    r = torch.empty(m * n, l, dtype=torch.float64, device=dev)
    if n:
        nat.check(nat.load().bmpc_op_collision_ratios(n, l, m * n, x.data_ptr(), y.data_ptr(),
                                                      xi_x.data_ptr(), xi_y.data_ptr(), float(a), float(b),
                                                      r.data_ptr(), ctypes.c_void_p(stream_ptr())),
                  "collision_ratios")
    return r.cpu().numpy() if host else r


def _score_fused(plan: RankedPlan, batch: ProblemBatch, limits: FilterLimits,
                 spec: MetaCostSpec | None):
    """Scoring straight from the device coefficients a Planner solve left in
    ``plan._dev`` (bmpc_score: the fused sampling + filters + meta cost)."""
    from . import device as D

    dv = plan._dev
    solver: BatchSolver = dv["solver"]
    ctx = solver._context()
    prob = dv.get("prob")
    if prob is None:
        prob = solver.device_problem(batch)
        dv["prob"] = prob
    sc = D.alloc_score(prob.L, prob.S, prob.b_xy.device)
    nat.check(nat.load().bmpc_score(ctx, ctypes.byref(prob.c_struct()), D.ptr(dv["c_x"]),
                                    D.ptr(dv["c_y"]), D.ptr(dv["c_psi"]), D.ptr(dv["res"]),
                                    ctypes.byref(_spec_struct(spec, limits)), ctypes.byref(D.score_struct(sc)),
                                    ctypes.c_void_p(D.stream_ptr())), "score")
    return sc


def _score_samples(plan: RankedPlan, xi_x, xi_y, a: float, b: float, limits: FilterLimits,
                   spec: MetaCostSpec | None, with_residuals: bool):
    """Scoring of the plan's OWN sampled arrays (x, y, psi, v and, for the
    filters, plan.residuals) on the device (bmpc_score_samples): whatever the
    caller put in the RankedPlan is what gets filtered and ranked, as in the
    reference (planner.py:219-257)."""
    import torch

    from . import device as D

    dev = torch.device("cuda", torch.cuda.current_device())
    up = lambda t: torch.from_numpy(np.ascontiguousarray(t, dtype=np.float64)).to(dev)  # noqa: E731
    n, l = plan.x.shape
    xi_x, xi_y = np.asarray(xi_x, dtype=np.float64).ravel(), np.asarray(xi_y, dtype=np.float64).ravel()
    if xi_x.size % n or xi_x.shape != xi_y.shape:
        raise ValueError("obstacle predictions must have m*n entries")
    gx, gy = up(xi_x), up(xi_y)
    res = None
    if with_residuals:
        r = plan.residuals
        res = up(np.stack([np.asarray(r.r_obs), np.asarray(r.r_acc), np.asarray(r.r_nonhol)]))
    arrs = [up(t) for t in (plan.x, plan.y, plan.psi, plan.v)]
    sc = D.alloc_score(l, 1, dev)
    prob = nat.Problem(xi_x.size // n, l, 1, gx.data_ptr(), gy.data_ptr(), None, None, float(a), float(b),
                       0.0, 0.0, 0.0)
    nat.check(nat.load().bmpc_score_samples(ctypes.byref(prob), n, *[t.data_ptr() for t in arrs],
                                            D.ptr(res), ctypes.byref(_spec_struct(spec, limits)),
                                            ctypes.byref(D.score_struct(sc)),
                                            ctypes.c_void_p(D.stream_ptr())), "score_samples")
    return sc


def filter_candidates(plan: RankedPlan, batch: ProblemBatch, limits: FilterLimits) -> np.ndarray:
    """Heading, residual and recomputed-collision filters (planner.py:233-245),
    evaluated on the plan's own x, y, psi and residuals."""
    sc = _score_samples(plan, batch.xi_x, batch.xi_y, batch.a, batch.b, limits, None, True)
    plan.heading_max = sc.heading_max.cpu().numpy()
    plan.min_ratio = sc.min_ratio.cpu().numpy() if batch.xi_x.size else np.full(plan.l, np.inf)
    plan.feasible = sc.flags.cpu().numpy() == 7
    return plan.feasible


def _select(feasible, meta_cost) -> int | None:
    """The reference's selection rule (planner.py:252-256): argmin of the meta
    cost over the feasible candidates, lowest index on ties, None when nothing
    is feasible (numpy argmin: a NaN cost wins)."""
    if feasible is None:
        return None
    feasible = np.asarray(feasible, dtype=bool)
    if not feasible.any():
        return None
    return int(np.argmin(np.where(feasible, meta_cost, np.inf)))


def rank(plan: RankedPlan, spec: MetaCostSpec) -> RankedPlan:
    """Meta cost of every candidate from the plan's own v and y (planner.py:
    210-216, on the device) and the cheapest candidate plan.feasible marks
    (planner.py:248-257)."""
    n, l = plan.x.shape
    sc = _score_samples(plan, np.zeros(0), np.zeros(0), 1.0, 1.0, FilterLimits(), spec, False)
    plan.meta_cost = sc.meta_cost.cpu().numpy()
    plan.best_index = _select(plan.feasible, plan.meta_cost)
    return plan


def _filter_and_rank_fused(plan: RankedPlan, batch: ProblemBatch, limits: FilterLimits,
                           spec: MetaCostSpec) -> None:
    """filter_candidates + rank for a plan this package just sampled from its
    own device solve (the MPC cycle): one fused scoring launch on the device
    coefficients, the same bits as the two reference-API calls on the sampled
    arrays."""
    sc = _score_fused(plan, batch, limits, spec)
    plan.heading_max = sc.heading_max.cpu().numpy()
    plan.min_ratio = sc.min_ratio.cpu().numpy() if batch.xi_x.size else np.full(plan.l, np.inf)
    plan.feasible = sc.flags.cpu().numpy() == 7
    plan.meta_cost = sc.meta_cost.cpu().numpy()
    plan.best_index = _select(plan.feasible, plan.meta_cost)


@dataclass(frozen=True)
class LaneGeometry:
    """Straight road with equally spaced lanes; lane 0 is the right lane (planner.py:43-64)."""

    n_lanes: int
    width: float
    y0: float = 0.0

    def __post_init__(self):
        if self.n_lanes < 1 or self.width <= 0:
            raise ValueError("need at least one lane of positive width")

    @property
    def centers(self) -> np.ndarray:
        return self.y0 + self.width * np.arange(self.n_lanes)

    @property
    def y_right(self) -> float:
        return self.y0

    def lane_of(self, y: float) -> int:
        return int(np.argmin(np.abs(self.centers - y)))


def sample_goals_cruise(ego: EgoState, lanes: LaneGeometry, spec: MetaCostSpec, l: int,
                        t_f: float) -> list[Goal]:
    """Round-robin lanes, all at the cruise distance (planner.py:96-110)."""
    c = lanes.centers
    return [Goal(x=ego.x + spec.v_cruise * t_f, y=float(c[i % lanes.n_lanes]), vx=spec.v_cruise,
                 vy=0.0, ax=0.0, ay=0.0, lane=i % lanes.n_lanes) for i in range(l)]


def sample_goals_highspeed(ego: EgoState, lanes: LaneGeometry, spec: MetaCostSpec, l: int,
                           t_f: float) -> list[Goal]:
    """~60% of the goals staggered on the right lane, the rest wide (planner.py:113-138)."""
    if l < 2:
        raise ValueError("high-speed sampling needs at least 2 goals")
    n_right = math.ceil(0.6 * l)
    c = lanes.centers
    reach = spec.v_max * t_f
    goals = [Goal(x=ego.x + dist, y=float(c[0]), vx=spec.v_max, vy=0.0, ax=0.0, ay=0.0, lane=0)
             for dist in np.linspace(0.5 * reach, reach, n_right)]
    other = list(range(1, lanes.n_lanes)) or [0]
    for i in range(l - n_right):
        lane = other[i % len(other)]
        goals.append(Goal(x=ego.x + reach, y=float(c[lane]), vx=spec.v_max, vy=0.0, ax=0.0, ay=0.0,
                          lane=lane))
    return goals


def sample_goals(ego: EgoState, lanes: LaneGeometry, spec: MetaCostSpec, l: int,
                 t_f: float) -> list[Goal]:
    if spec.kind == "cruise":
        return sample_goals_cruise(ego, lanes, spec, l, t_f)
    return sample_goals_highspeed(ego, lanes, spec, l, t_f)


@dataclass
class ControlCommand:
    accel: float
    steering: float


def extract_control(traj: Candidate, h: float, dt_grid: float, dt_ctrl: float | None = None
                    ) -> ControlCommand:
    """Finite-difference accel and bicycle steering, read one control period
    ahead (planner.py:260-274)."""
    k = 1 if dt_ctrl is None else max(1, int(round(dt_ctrl / dt_grid)))
    k = min(k, len(traj.v) - 1)
    accel = (traj.v[k] - traj.v[k - 1]) / dt_grid
    steering = math.atan(traj.psidot[k] * h / max(traj.v[k], 1e-6))
    return ControlCommand(accel=accel, steering=steering)


@dataclass
class CycleResult:
    command: ControlCommand
    plan: RankedPlan
    solve_time: float
    info: object
    fallback: bool


def sample_goals_uniform(rng: np.random.Generator, ego: EgoState, l: int, t_f: float,
                         y_range=(-5.25, 5.25), v_range=(10.0, 30.0)) -> list[Goal]:
    """The BASELINE c1-c4 goal sampler: lateral target and terminal speed uniform."""
    ys = rng.uniform(*y_range, l)
    vs = rng.uniform(*v_range, l)
    return [Goal(x=ego.x + v * t_f, y=float(y), vx=float(v), vy=0.0, ax=0.0, ay=0.0, lane=-1)
            for y, v in zip(ys, vs)]


@dataclass(frozen=True)
class PlannerConfig:
    l: int = 11
    n: int = 100
    t_f: float = 10.0
    degree: int = 10
    rho_xy: float = 1.0
    max_iter: int = 100
    tol: float = 1e-3
    m: int = 10
    a: float = 5.6
    b: float = 3.1
    v_min: float = 0.1
    v_max: float = 20.0
    a_max: float = 8.0
    h: float = 2.5
    dt_cycle: float = 0.1
    warm_start: bool = True
    warm_residual_cap: float = 0.2
    limits: FilterLimits = FilterLimits()
    # warps per instance in the MPC solve: 0 = auto (a team of 4 when the batch
    # is small enough to leave SMs idle, l <= 148 with n <= 128; else 1)
    team_warps: int = 0


class Planner:
    """Owns the shared constants; builds goal batches and scores solutions
    (planner.py:308-423)."""

    def __init__(self, cfg: PlannerConfig, lanes=None, meta: MetaCostSpec | None = None):
        self.cfg = cfg
        self.lanes = lanes
        self.meta = meta or MetaCostSpec("cruise")
        grid = build_time_grid(0.0, cfg.t_f, cfg.n)
        self.basis = build_basis(grid, cfg.degree)
        self.mats = build_constant_matrices(self.basis, cfg.m, BoundarySpec())
        self.solver = BatchSolver(self.basis, self.mats, cfg.rho_xy)
        self._prev = None        # (device solution, residuals) of the last cycle
        self._shift_dev = None
        self._prev_steering = 0.0
        # exact time-shift map in coefficient space (planner.py:326-334): the
        # basis evaluated one control period later, projected back
        from .basis import bernstein

        span = grid.tf - grid.t0
        u = (grid.times + cfg.dt_cycle - grid.t0) / span
        self._shift_map = np.linalg.pinv(self.basis.P) @ bernstein(u, cfg.degree)

    def boundary_vectors(self, ego: EgoState, goals: list[Goal]) -> tuple[np.ndarray, np.ndarray]:
        """Per-instance boundary right-hand sides (planner.py:336-347), column i
        = [ego x, vx, ax, goal x, vx, ax, ego y, vy, ay, goal y, vy, ay]."""
        l = len(goals)
        g = np.array([(q.x, q.vx, q.ax, q.y, q.vy, q.ay) for q in goals], dtype=np.float64).reshape(l, 6)
        b_xy = np.empty((12, l))
        b_xy[[0, 1, 2, 6, 7, 8]] = np.array([ego.x, ego.vx, ego.ax, ego.y, ego.vy, ego.ay])[:, None]
        b_xy[[3, 4, 5, 9, 10, 11]] = g.T
        b_psi = np.zeros((4, l))
        b_psi[0], b_psi[1] = ego.psi, ego.psidot
        return b_xy, b_psi

    def build_batch(self, ego: EgoState, vehicles: list[VehicleState], goals: list[Goal]
                    ) -> ProblemBatch:
        nearest = select_nearest(vehicles, ego.x, ego.y, self.cfg.m)
        xi_x, xi_y = predict_constant_velocity(nearest, self.basis.grid.times)
        b_xy, b_psi = self.boundary_vectors(ego, goals)
        c = self.cfg
        return ProblemBatch(l=len(goals), xi_x=xi_x, xi_y=xi_y, a=c.a, b=c.b, v_min=c.v_min,
                            v_max=c.v_max, a_max=c.a_max, b_xy=b_xy, b_psi=b_psi, rho_xy=c.rho_xy)

    def _warm_device(self, prob, batch: ProblemBatch):
        """Warm start of the next solve, built and kept on the device
        (planner.py:362-410): the previous solution's near-converged columns
        (worst residual <= warm_residual_cap) shifted one cycle by the exact
        coefficient map, their closed-form alpha/d/alpha_a/d_a/v on the
        shifted trajectories, multipliers carried.  Returns (warm dict,
        eligibility mask) -- the kernel starts the other columns cold -- or
        (None, None)."""
        import torch

        from . import kernels
        from .device import DeviceSolution

        if self._prev is None:
            return None, None
        prev, prev_res = self._prev
        if prev.c_x.shape[1] != batch.l:
            return None, None
        eligible = prev_res.max_per_instance() <= self.cfg.warm_residual_cap
        if not eligible.any():
            return None, None
        dev = prev.c_x.device
        if self._shift_dev is None:
            self._shift_dev = torch.from_numpy(np.ascontiguousarray(self._shift_map)).to(dev)
        S = self._shift_dev
        cx, cy, cp = (S @ t for t in (prev.c_x, prev.c_y, prev.c_psi))
        smp = self.solver.sample_device(
            DeviceSolution(cx, cy, cp, None, None, None, None, None, None, 0, False),
            which=("x", "y", "xdot", "ydot", "xddot", "yddot"))
        alpha, d = kernels.obstacle_update(smp["x"], smp["y"], prob.xi_x[0], prob.xi_y[0],
                                           batch.a, batch.b)
        alpha_a, d_a = kernels.accel_update(smp["xddot"], smp["yddot"], batch.a_max)
        v = kernels.v_update(smp["xdot"], smp["ydot"], batch.v_min, batch.v_max)
        warm = dict(alpha=alpha, d=d, alpha_a=alpha_a, d_a=d_a, v=v, c_psi=cp, c_x=cx, c_y=cy,
                    lambda_x=prev.l_x, lambda_y=prev.l_y, lambda_psi=prev.l_psi)
        mask = torch.from_numpy(eligible.astype(np.uint8)).to(dev)
        return warm, mask

    def _warm_state(self, batch: ProblemBatch) -> AmState | None:
        """The reference-shaped warm AmState (host arrays): cold state with the
        eligible columns replaced by the device warm start."""
        warm, mask = self._warm_device(self.solver.device_problem(batch), batch)
        if warm is None:
            return None
        state = self.solver.init_state(batch)
        idx = np.where(mask.cpu().numpy() != 0)[0]
        for k in ("c_x", "c_y", "c_psi", "v", "alpha", "d", "alpha_a", "d_a", "lambda_x", "lambda_y",
                  "lambda_psi"):
            getattr(state, k)[:, idx] = warm[k].cpu().numpy()[:, idx]
        return state

    def sample_plan(self, state: AmState, goals: list, residuals: Residuals,
                    batch: ProblemBatch | None = None) -> RankedPlan:
        """x, y, psi, psidot, v = |(xdot, ydot)| (unclipped), xddot, yddot
        (planner.py:412-423), sampled on the device."""
        import torch

        dev = torch.device("cuda", torch.cuda.current_device())
        up = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
        return self._sample_plan_device(up(state.c_x), up(state.c_y), up(state.c_psi), goals,
                                        residuals, batch)

    def _sample_plan_device(self, cx, cy, cp, goals: list, residuals: Residuals,
                            batch: ProblemBatch | None = None) -> RankedPlan:
        import torch

        from .device import DeviceSolution

        dev = cx.device
        res = torch.from_numpy(np.stack([residuals.r_obs, residuals.r_acc, residuals.r_nonhol])).to(dev)
        sol = DeviceSolution(cx, cy, cp, None, None, None, None, res, None, 0, False)
        smp = self.solver.sample_device(sol, which=("x", "y", "psi", "psidot", "v", "xddot", "yddot"))
        h = {k: v.cpu().numpy() for k, v in smp.items()}
        return RankedPlan(goals=goals, x=h["x"], y=h["y"], psi=h["psi"], psidot=h["psidot"], v=h["v"],
                          xddot=h["xddot"], yddot=h["yddot"], residuals=residuals,
                          _dev=dict(solver=self.solver, c_x=cx, c_y=cy, c_psi=cp, res=res, batch=batch))

    def fallback_command(self, ego: EgoState) -> ControlCommand:
        """Hold steering, bleed speed toward v_min over the horizon (planner.py:425-430)."""
        accel = max(-self.cfg.a_max, (self.cfg.v_min - ego.speed) / self.cfg.t_f)
        return ControlCommand(accel=float(min(accel, self.cfg.a_max)), steering=self._prev_steering)

    def mpc_cycle(self, ego: EgoState, vehicles: list[VehicleState]) -> CycleResult:
        """One receding-horizon cycle (planner.py:432-462): goals, batch, warm
        start, device solve with carried multipliers, fused scoring, control."""
        import time

        c = self.cfg
        goals = sample_goals(ego, self.lanes, self.meta, c.l, c.t_f)
        batch = self.build_batch(ego, vehicles, goals)
        prob = self.solver.device_problem(batch)
        warm, mask = self._warm_device(prob, batch) if c.warm_start else (None, None)
        start = time.perf_counter()
        team = c.team_warps or (4 if batch.l <= 148 and c.n <= 128 else 1)
        sol = self.solver.solve_device(prob, max_iter=c.max_iter, tol=c.tol, warm=warm,
                                       keep_multipliers=True, want_v=False, warm_mask=mask,
                                       team_warps=team)
        hist = sol.history[: sol.iterations].cpu().numpy()
        solve_time = time.perf_counter() - start
        history = [Residuals(r_obs=h[0].copy(), r_acc=h[1].copy(), r_nonhol=h[2].copy()) for h in hist]
        info = SolveInfo(residual_history=history, iterations=sol.iterations, converged=sol.converged)
        plan = self._sample_plan_device(sol.c_x, sol.c_y, sol.c_psi, goals, history[-1], batch)
        _filter_and_rank_fused(plan, batch, c.limits, self.meta)
        self._prev = (sol, plan.residuals)
        if plan.best_index is None:
            command, fallback = self.fallback_command(ego), True
        else:
            command = extract_control(plan.candidate(plan.best_index), c.h, self.basis.grid.dt,
                                      c.dt_cycle)
            command.accel = float(np.clip(command.accel, -c.a_max, c.a_max))
            fallback = False
            self._prev_steering = command.steering
        return CycleResult(command=command, plan=plan, solve_time=solve_time, info=info,
                           fallback=fallback)


@dataclass
class PlanResult:
    """Output of plan_batch for S stacked scenes x l goals (host arrays)."""

    c_x: np.ndarray
    c_y: np.ndarray
    c_psi: np.ndarray
    res_final: np.ndarray      # (3, L)
    meta_cost: np.ndarray      # (L,)
    min_ratio: np.ndarray
    heading_max: np.ndarray
    flags: np.ndarray          # uint8 bit0 heading, bit1 residual, bit2 collision
    best_index: list           # per scene, None when nothing is feasible
    argmin_all: np.ndarray
    argmin_hc: np.ndarray      # -1 = None
    n_feasible: np.ndarray
    iterations: int
    converged: bool

    @property
    def feasible(self) -> np.ndarray:
        return self.flags == 7


_LAYOUT_CACHE: dict = {}


def _results_block(solver: BatchSolver, ctx, S: int, l: int) -> dict:
    """Fresh numpy views (caller-owned) into one pinned host block with the
    offsets of bmpc_plan_host_layout."""
    import torch

    key = (ctx.value, S, l)
    lay = _LAYOUT_CACHE.get(key)
    if lay is None:
        o = (ctypes.c_longlong * 9)()
        nat.check(nat.load().bmpc_plan_host_layout(ctx, S, l, 1, o, 9), "bmpc_plan_host_layout")
        nb, L = solver.basis.n_b, S * l
        f8, i8, u1 = np.float64, np.int64, np.uint8
        lay = (int(o[8]), [("coef", o[0], 3 * nb * L, f8), ("rf", o[1], 3 * L, f8),
                           ("meta", o[2], L, f8), ("mr", o[3], L, f8), ("hm", o[4], L, f8),
                           ("best", o[5], 4 * S, i8), ("fl", o[6], L, u1)])
        _LAYOUT_CACHE[key] = lay
    total, fields = lay
    raw = torch.empty(total, dtype=torch.uint8, pin_memory=True).numpy()
    return {name: raw[off:off + cnt * np.dtype(dt).itemsize].view(dt) for name, off, cnt, dt in fields}


def plan_batch(solver: BatchSolver, scenes, max_iter: int = 100, tol: float = 0.0,
               spec: MetaCostSpec | None = None, limits: FilterLimits | None = None,
               stream=None, precision: str = "fp64") -> PlanResult:
    """Solve + score S stacked scenes in one C-ABI call from host buffers
    (``bmpc_plan_host``): the end-to-end path the benchmark times.

    ``scenes`` is a ProblemBatch (one scene) or any object with the SceneBatch
    fields (xi_x/xi_y (S, m*n), b_xy (12, S*l), b_psi (4, S*l), l, S, scalars).
    """
    from .device import stream_ptr

    limits = limits or FilterLimits()
    # every shape is checked before the C ABI reads (or copies) the host buffers
    xi_x, xi_y, S, l = solver.check_scenes(scenes)
    L = S * l
    nb, n = solver.basis.n_b, solver.basis.grid.n
    c = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    xi_x, xi_y, b_xy, b_psi = c(xi_x), c(xi_y), c(scenes.b_xy), c(scenes.b_psi)
    ctx = solver._context()
    prob = nat.Problem(xi_x.shape[1] // n, l, S, xi_x.ctypes.data, xi_y.ctypes.data,
                       b_xy.ctypes.data, b_psi.ctypes.data, scenes.a, scenes.b, scenes.v_min,
                       scenes.v_max, scenes.a_max)
    opts = nat.SolveOpts(max_iter=int(max_iter), tol=float(tol), precision=_precision_code(precision))
    # every output is a view of one page-locked block laid out like the
    # device results block, so they come back with one copy straight into
    # place; the block returns to torch's pinned caching allocator when the
    # last view is dropped
    blk = _results_block(solver, ctx, S, l)
    coef = blk["coef"].reshape(3, nb, L)
    res = blk["rf"].reshape(3, L)
    out = nat.SolveOut(coef[0].ctypes.data, coef[1].ctypes.data, coef[2].ctypes.data, None, None,
                       None, None, None, res.ctypes.data, 0, 0)
    meta, mr, hm, flags = blk["meta"], blk["mr"], blk["hm"], blk["fl"]
    best, amin, ahc, nf = blk["best"].reshape(4, S)
    so = nat.ScoreOut(meta.ctypes.data, mr.ctypes.data, hm.ctypes.data, flags.ctypes.data,
                      best.ctypes.data, amin.ctypes.data, ahc.ctypes.data, nf.ctypes.data)
    nat.check(nat.load().bmpc_plan_host(ctx, ctypes.byref(prob), ctypes.byref(opts), ctypes.byref(out),
                                        ctypes.byref(_spec_struct(spec, limits)), ctypes.byref(so),
                                        ctypes.c_void_p(stream_ptr(stream))), "plan")
    solver.kkt.n_solves += 2 * out.iterations
    return PlanResult(c_x=coef[0], c_y=coef[1], c_psi=coef[2], res_final=res, meta_cost=meta,
                      min_ratio=mr, heading_max=hm, flags=flags,
                      best_index=[int(b) if b >= 0 else None for b in best], argmin_all=amin,
                      argmin_hc=ahc, n_feasible=nf, iterations=out.iterations,
                      converged=bool(out.converged))


def plan_states(solver: BatchSolver, egos, vehicles, goals, cfg: "PlannerConfig | None" = None,
                max_iter: int | None = None, tol: float = 0.0, spec: MetaCostSpec | None = None,
                limits: FilterLimits | None = None, precision: str = "fp64",
                stream=None) -> PlanResult:
    """Plan S scenes straight from their ego / vehicle / goal states: the scene
    assembly (select_nearest, constant-velocity prediction, boundary vectors)
    runs on the device (`bmpc_assemble`), then solve + fused scoring + argmin
    (`bmpc_plan`).  Only the small state arrays cross the host link -- not the
    (S, m*n) prediction tables the host build_batch path uploads.
    """
    from . import device as D

    cfg = cfg or PlannerConfig()
    limits = limits or FilterLimits()
    spec = spec or MetaCostSpec("cruise", v_cruise=20.0)
    max_iter = int(max_iter if max_iter is not None else cfg.max_iter)
    prob = D.assemble_scenes(solver, egos, vehicles, goals, cfg.m, cfg.a, cfg.b, cfg.v_min,
                             cfg.v_max, cfg.a_max, stream=stream)
    dev = prob.b_xy.device
    nb, n = solver.basis.n_b, solver.basis.grid.n
    sol = D.alloc_solution(nb, n, prob.L, max_iter, False, dev)
    sc = D.alloc_score(prob.L, prob.S, dev)
    out = D.solution_struct(sol)
    out.history = None
    opts = nat.SolveOpts(max_iter=max_iter, tol=float(tol), precision=_precision_code(precision))
    nat.check(nat.load().bmpc_plan(solver._context(), ctypes.byref(prob.c_struct()), ctypes.byref(opts),
                                   ctypes.byref(out), ctypes.byref(_spec_struct(spec, limits)),
                                   ctypes.byref(D.score_struct(sc)), ctypes.c_void_p(D.stream_ptr(stream))),
              "plan_states")
    solver.kkt.n_solves += 2 * out.iterations
    h = lambda t: t.cpu().numpy()  # noqa: E731
    best = h(sc.best_index)
    return PlanResult(c_x=h(sol.c_x), c_y=h(sol.c_y), c_psi=h(sol.c_psi), res_final=h(sol.res_final),
                      meta_cost=h(sc.meta_cost), min_ratio=h(sc.min_ratio),
                      heading_max=h(sc.heading_max), flags=h(sc.flags),
                      best_index=[int(x) if x >= 0 else None for x in best],
                      argmin_all=h(sc.argmin_all), argmin_hc=h(sc.argmin_hc),
                      n_feasible=h(sc.n_feasible), iterations=out.iterations,
                      converged=bool(out.converged))
