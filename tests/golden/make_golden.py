"""Generate the golden fixtures by running the REFERENCE itself.

Runs only in the build container (it imports /root/reference, which does not
exist on the GPU box); the .npz outputs are committed.  The reference's
compiled backend is the Cython extension built from the reference's own
sources by oracle/Makefile (target `ref`), registered into the reference's
kernel registry for the duration of this script.

    python tests/golden/make_golden.py

Fixtures (float64 unless noted):
  tail_case.npz   inputs + outputs of every reference kernel (compiled and numpy
                  back-ends) on the sample data shape of the reference's
                  tests/test_kernels.py (n=50, m=4, l=7, rng seed 12345)
  demo.npz        oracles.make_demo_batch(l=11, seed=0) on the canonical solver
                  (n=100, m=10, degree 10, t_f=10), 80 sweeps, tol=0
  c0.npz, c1.npz  BASELINE configs 0 and 1 (scenes.make_workload), 100 sweeps,
                  plus the 1-ulp self-sensitivity screen and planner scoring
  c3s.npz         4 scenes x 64 goals of the c3 generator (m=20), 100 sweeps
  c4s.npz         2 scenes x 32 goals of the c4 generator (n=200, n_b=16, m=50), 100 sweeps
  reverse.npz     goals behind a reversing ego: headings cross +-pi so the
                  np.unwrap corrections are non-zero (40 sweeps)
  c2s.npz         1 scene x 256 goals of the c2 generator (m=30, x~U(-50,200)),
                  200 sweeps -- the one BASELINE config at 200 sweeps
  c2f.npz, c3f.npz, c4f.npz  scenes of the c3 / c4 generators with FEASIBLE candidates,
                  so best_index is a real index on both sides (seeds found by
                  tests/golden/seed_search.py); each holds every feasible column
                  of its scene (c2f: of a 1024-goal batch) plus the lowest-index
                  other columns up to l
  mpc_kat.npz     also stores, per cycle, the set of best indices the reference
                  itself picks when the same solve (same batch, same warm state)
                  is re-run with its columns permuted or one column at a time:
                  the evidence that the reference's pick inside a tie class is
                  a column-position (BLAS rounding) artefact
"""

from __future__ import annotations

import math
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

from threadpoolctl import threadpool_limits  # noqa: E402

threadpool_limits(1)

import am_oracle  # noqa: E402
import batchmpc  # noqa: E402
from batchmpc import build_basis, build_constant_matrices, build_time_grid  # noqa: E402
from batchmpc import kernels as rk  # noqa: E402
from batchmpc.kernels import _numpy as rnp  # noqa: E402
from batchmpc.oracles import demo_solver, make_demo_batch  # noqa: E402
from batchmpc.planner import (FilterLimits, MetaCostSpec, RankedPlan,  # noqa: E402
                              filter_candidates, rank)
from batchmpc.solver import BatchSolver, ProblemBatch  # noqa: E402

from paper_2109_10392_b200.scenes import make_workload  # noqa: E402

REF = am_oracle._load_ref_kernels()
if REF is None:
    raise SystemExit("build the reference kernels first: make -C oracle ref")
rk._BACKENDS["compiled"] = REF
rk.set_backend("compiled")


def ref_solver(n, t_f, degree, m):
    grid = build_time_grid(0.0, t_f, n)
    basis = build_basis(grid, degree)
    return BatchSolver(basis, build_constant_matrices(basis, m), 1.0)


def trajectories(solver, st):
    P = solver.basis.P
    return [P @ st.c_x, P @ st.c_y, P @ st.c_psi]


def rel_div(solver, a, b):
    out = np.zeros(a.c_x.shape[1])
    for ta, tb in zip(trajectories(solver, a), trajectories(solver, b)):
        scale = np.maximum(1.0, np.abs(ta).max(axis=0))
        out = np.maximum(out, np.abs(ta - tb).max(axis=0) / scale)
    return out


def score(solver, st, info, batch, spec):
    P, Pd, Pdd = solver.basis.P, solver.basis.Pdot, solver.basis.Pddot
    xd, yd = Pd @ st.c_x, Pd @ st.c_y
    plan = RankedPlan(goals=[None] * batch.l, x=P @ st.c_x, y=P @ st.c_y, psi=P @ st.c_psi,
                      psidot=Pd @ st.c_psi, v=np.sqrt(xd**2 + yd**2), xddot=Pdd @ st.c_x,
                      yddot=Pdd @ st.c_y, residuals=info.residual_history[-1])
    limits = FilterLimits()
    filter_candidates(plan, batch, limits)
    rank(plan, spec)
    hc = (plan.heading_max <= limits.heading_limit) & (plan.min_ratio >= 1.0 - limits.collision_margin)
    best_hc = int(np.argmin(np.where(hc, plan.meta_cost, np.inf))) if hc.any() else -1
    return dict(meta_cost=plan.meta_cost, feasible=plan.feasible.astype(np.uint8),
                min_ratio=plan.min_ratio, heading_max=plan.heading_max,
                best_index=np.int64(-1 if plan.best_index is None else plan.best_index),
                argmin_all=np.int64(np.argmin(plan.meta_cost)), argmin_hc=np.int64(best_hc))


def solve_scene(solver, xi_x, xi_y, b_xy, b_psi, W, iters, screen):
    batch = ProblemBatch(l=b_xy.shape[1], xi_x=xi_x, xi_y=xi_y, a=W.a, b=W.b, v_min=W.v_min,
                         v_max=W.v_max, a_max=W.a_max, b_xy=b_xy, b_psi=b_psi)
    st, info = solver.solve(batch, max_iter=iters, tol=0.0)
    out = dict(c_x=st.c_x, c_y=st.c_y, c_psi=st.c_psi, lambda_x=st.lambda_x, lambda_y=st.lambda_y,
               lambda_psi=st.lambda_psi,
               res_final=np.stack([info.residual_history[-1].r_obs, info.residual_history[-1].r_acc,
                                   info.residual_history[-1].r_nonhol]))
    if screen:
        pb = ProblemBatch(l=batch.l, xi_x=xi_x * (1.0 + 2.2e-16), xi_y=xi_y, a=W.a, b=W.b,
                          v_min=W.v_min, v_max=W.v_max, a_max=W.a_max, b_xy=b_xy, b_psi=b_psi)
        st2, _ = solver.solve(pb, max_iter=iters, tol=0.0)
        out["screen_div"] = rel_div(solver, st, st2)
    for kind, spec in (("cruise", MetaCostSpec("cruise", v_cruise=20.0)),
                       ("highspeed", MetaCostSpec("highspeed", v_max=25.0, y_rl=-5.25, w1=1.0, w2=0.1))):
        for k, v in score(solver, st, info, batch, spec).items():
            out[f"{kind}_{k}"] = v
    return st, info, out


def workload_fixture(name, W, iters, screen=True, extra=None):
    solver = ref_solver(W.n, W.t_f, W.degree, W.m)
    outs = []
    for s in range(W.S):
        cols = slice(s * W.l, (s + 1) * W.l)
        _, info, o = solve_scene(solver, W.xi_x[s], W.xi_y[s], W.b_xy[:, cols], W.b_psi[:, cols], W,
                                 iters, screen)
        if extra is not None:
            extra(o, info)
        outs.append(o)
    data = dict(n=W.n, t_f=W.t_f, degree=W.degree, m=W.m, l=W.l, S=W.S, iters=iters,
                a=W.a, b=W.b, v_min=W.v_min, v_max=W.v_max, a_max=W.a_max,
                xi_x=W.xi_x, xi_y=W.xi_y, b_xy=W.b_xy, b_psi=W.b_psi)
    for k in outs[0]:
        vals = [o[k] for o in outs]
        if np.ndim(vals[0]) == 0:
            data[k] = np.array(vals)
        elif k in ("c_x", "c_y", "c_psi", "lambda_x", "lambda_y", "lambda_psi", "res_final", "history"):
            data[k] = np.concatenate(vals, axis=-1)
        else:
            data[k] = np.concatenate(vals, axis=0)
    np.savez_compressed(HERE / f"{name}.npz", **data)
    print(name, {k: np.shape(v) for k, v in data.items() if np.ndim(v)})


def tail_case():
    rng = np.random.default_rng(12345)
    n, m, l = 50, 4, 7
    mn = m * n
    s = dict(
        x=rng.normal(75, 40, (n, l)), y=rng.normal(6, 3, (n, l)),
        xdot=rng.normal(15, 2, (n, l)), ydot=rng.normal(0, 1, (n, l)),
        xddot=rng.normal(0, 2, (n, l)), yddot=rng.normal(0, 2, (n, l)),
        psi=rng.normal(0, 0.1, (n, l)),
        xi_x=rng.normal(75, 50, mn), xi_y=rng.normal(6, 4, mn),
        alpha=rng.uniform(-np.pi, np.pi, (mn, l)), d=1 + rng.uniform(0, 2, (mn, l)),
        alpha_a=rng.uniform(-np.pi, np.pi, (n, l)), d_a=rng.uniform(0, 8, (n, l)),
        v=rng.uniform(5, 20, (n, l)),
    )
    # exact zero-length cases for the (1, 0) fallbacks
    s["xddot"][3, 2] = s["yddot"][3, 2] = 0.0
    s["x"][5, 1] = s["xi_x"][5]
    s["y"][5, 1] = s["xi_y"][5]
    out = dict(s)
    args = (s["x"], s["y"], s["xdot"], s["ydot"], s["xddot"], s["yddot"], s["psi"],
            s["xi_x"], s["xi_y"], 0.1, 20.0, 8.0, 5.6, 3.1)
    for tag, mod in (("ref", REF), ("np", rnp)):
        for name, val in zip(("d", "d_a", "v", "r_x", "r_y", "g_x", "g_y", "sq_obs", "sq_acc", "sq_nonhol"),
                             mod.tail_core(*args)):
            out[f"{tag}_core_{name}"] = np.asarray(val)
        for name, val in zip(("alpha", "d", "alpha_a", "d_a", "v", "r_x", "r_y", "g_x", "g_y"),
                             mod.tail_update(*args)):
            out[f"{tag}_upd_{name}"] = np.asarray(val)
        al, d = mod.obstacle_update(s["x"], s["y"], s["xi_x"], s["xi_y"], 5.6, 3.1)
        out[f"{tag}_obs_alpha"], out[f"{tag}_obs_d"] = al, d
        al, da = mod.accel_update(s["xddot"], s["yddot"], 8.0)
        out[f"{tag}_acc_alpha_a"], out[f"{tag}_acc_d_a"] = al, da
        out[f"{tag}_v"] = mod.v_update(s["xdot"], s["ydot"], 0.1, 20.0)
        gx, gy = mod.assemble_g(s["xi_x"], s["xi_y"], s["alpha"], s["d"], s["alpha_a"], s["d_a"],
                                s["v"], s["psi"], 5.6, 3.1)
        out[f"{tag}_g_x"], out[f"{tag}_g_y"] = gx, gy
        rx, ry = mod.residual_vectors(s["x"], s["y"], s["xdot"], s["ydot"], s["xddot"], s["yddot"],
                                      s["psi"], s["xi_x"], s["xi_y"], s["alpha"], s["d"],
                                      s["alpha_a"], s["d_a"], s["v"], 5.6, 3.1)
        out[f"{tag}_r_x"], out[f"{tag}_r_y"] = rx, ry
    np.savez_compressed(HERE / "tail_case.npz", **out)
    print("tail_case", len(out))


def demo():
    solver = demo_solver()
    batch = make_demo_batch(solver, l=11, seed=0)
    st, info = solver.solve(batch, max_iter=80, tol=0.0, record_iterates=True)
    it = info.iterates
    np.savez_compressed(
        HERE / "demo.npz",
        n=100, t_f=10.0, degree=10, m=10, l=11, iters=80,
        xi_x=batch.xi_x, xi_y=batch.xi_y, b_xy=batch.b_xy, b_psi=batch.b_psi,
        a=batch.a, b=batch.b, v_min=batch.v_min, v_max=batch.v_max, a_max=batch.a_max,
        c_x=st.c_x, c_y=st.c_y, c_psi=st.c_psi, lambda_x=st.lambda_x, lambda_y=st.lambda_y,
        lambda_psi=st.lambda_psi, v=st.v, d_a=st.d_a, alpha_a=st.alpha_a, d=st.d, alpha=st.alpha,
        history=np.stack([[h.r_obs, h.r_acc, h.r_nonhol] for h in info.residual_history]),
        iter_c_x=np.stack([c[0] for c in it]), iter_c_psi=np.stack([c[2] for c in it]),
        g0_x=solver._g_parts(solver.init_state(batch), batch)[0],
    )
    print("demo")


def reverse_case():
    """Reversing ego with goals behind it: heading targets straddle +-pi."""
    from paper_2109_10392_b200.scenes import CONFIGS

    cfg = CONFIGS["c0"]
    W = make_workload("c0", l=24)
    l = 24
    rng = np.random.default_rng(99)
    b_xy = np.zeros((12, l))
    b_xy[1] = -6.0                       # reversing start speed
    vg = rng.uniform(-12.0, -4.0, l)
    b_xy[3] = vg * cfg.t_f
    b_xy[4] = vg
    b_xy[6] = 0.0
    b_xy[7] = rng.uniform(-0.5, 0.5, l)  # lateral start velocity: signs of ydot vary
    b_xy[9] = rng.uniform(-4.0, 4.0, l)
    W.b_xy, W.l = b_xy, l
    W.b_psi = np.zeros((4, l))
    W.xi_x = W.xi_x + 200.0              # obstacles far ahead: pure heading dynamics
    workload_fixture("reverse", W, 40, screen=True)


def _permuted(obj, perm):
    """Copy of a reference ProblemBatch / AmState with its columns permuted."""
    import dataclasses

    vals = {}
    for f in dataclasses.fields(obj):
        v = getattr(obj, f.name)
        vals[f.name] = np.ascontiguousarray(v[:, perm]) if isinstance(v, np.ndarray) and v.ndim == 2 else v
    if "l" in vals:
        vals["l"] = len(perm)
    return type(obj)(**vals)


def _ref_best(planner, batch, warm, perm, max_iter, tol):
    """The reference's own solve + sample_plan/filter/rank on the permuted
    columns; returns the best index in the ORIGINAL column numbering."""
    st, info = planner.solver.solve(_permuted(batch, perm), max_iter=max_iter, tol=tol,
                                    warm=None if warm is None else _permuted(warm, perm),
                                    keep_multipliers=True)
    plan = planner.sample_plan(st, [None] * len(perm), info.residual_history[-1])
    filter_candidates(plan, _permuted(batch, perm), planner.cfg.limits)
    rank(plan, planner.meta)
    return None if plan.best_index is None else int(np.asarray(perm)[plan.best_index])


def _ref_best_sequential(planner, batch, warm, max_iter, tol):
    """Column-at-a-time reference solves (l = 1 batches) under the batch's
    global tol rule: all columns run the same sweep count as the batch solve
    would, so each is solved for that count with tol disabled."""
    from batchmpc.solver import Residuals

    full_st, full_info = planner.solver.solve(batch, max_iter=max_iter, tol=tol, warm=warm,
                                              keep_multipliers=True)
    iters = full_info.iterations
    cols = []
    for i in range(batch.l):
        st, info = planner.solver.solve(_permuted(batch, [i]), max_iter=iters, tol=-1.0,
                                        warm=None if warm is None else _permuted(warm, [i]),
                                        keep_multipliers=True)
        cols.append((st, info.residual_history[-1]))
    cat = lambda k: np.concatenate([getattr(c[0], k) for c in cols], axis=1)  # noqa: E731
    st = full_st
    st.c_x, st.c_y, st.c_psi = cat("c_x"), cat("c_y"), cat("c_psi")
    res = Residuals(*(np.concatenate([getattr(c[1], k) for c in cols]) for k in ("r_obs", "r_acc", "r_nonhol")))
    plan = planner.sample_plan(st, [None] * batch.l, res)
    filter_candidates(plan, batch, planner.cfg.limits)
    rank(plan, planner.meta)
    return None if plan.best_index is None else int(plan.best_index)


class SequentialSolver:
    """The reference's BatchSolver run one column at a time (l = 1 batches, the
    reference's own batch-vs-sequential oracle, oracles.py:270-293), keeping the
    batch's global tol rule: every column is solved with tol disabled, the first
    sweep t at which the max over all columns is <= tol is found from the
    per-column histories, and the columns are re-solved for exactly t sweeps.
    Column arithmetic then never depends on a column's position in the batch."""

    def __init__(self, ref):
        self.ref = ref
        self.basis, self.mats, self.kkt = ref.basis, ref.mats, ref.kkt

    def __getattr__(self, k):
        return getattr(self.ref, k)

    def solve(self, batch, max_iter=150, tol=1e-3, warm=None, record_iterates=False,
              keep_multipliers=False):
        from batchmpc.solver import Residuals, SolveInfo

        def run(i, iters):
            return self.ref.solve(_permuted(batch, [i]), max_iter=iters, tol=-1.0,
                                  warm=None if warm is None else _permuted(warm, [i]),
                                  keep_multipliers=keep_multipliers)

        cols = [run(i, max_iter) for i in range(batch.l)]
        worst = np.max([[h.max_per_instance()[0] for h in info.residual_history] for _, info in cols], axis=0)
        hit = np.nonzero(worst <= tol)[0]
        iters = int(hit[0]) + 1 if hit.size else max_iter
        if iters != max_iter:
            cols = [run(i, iters) for i in range(batch.l)]
        st = cols[0][0].copy()
        for f in ("c_x", "c_y", "c_psi", "alpha", "d", "alpha_a", "d_a", "v", "lambda_x", "lambda_y",
                  "lambda_psi"):
            setattr(st, f, np.concatenate([getattr(c[0], f) for c in cols], axis=1))
        hist = [Residuals(*(np.concatenate([getattr(c[1].residual_history[t], k) for c in cols])
                            for k in ("r_obs", "r_acc", "r_nonhol"))) for t in range(iters)]
        return st, SolveInfo(residual_history=hist, iterations=iters, converged=bool(hit.size))


def mpc_kat(cycles: int = 3):
    """Closed-loop cruise_idm replay (seed 7, l=11, warm starts, tol=1e-3,
    200 sweeps) through the reference's own harness objects, full precision.
    Cross-checked against the reference's recorded testdata/run.jsonl."""
    import json

    from batchmpc import harness as H
    from batchmpc.planner import EgoState, Planner
    from batchmpc.traffic import VehicleState

    cfg = H.load_config("/root/reference/pkg/configs/cruise_idm.toml")
    rng = np.random.default_rng(cfg.seed)
    lanes = cfg.lane_geometry
    world = H.build_traffic(cfg, rng)
    pc = cfg.planner_config
    planner = Planner(pc, lanes, cfg.meta_spec)
    ego = EgoState(x=cfg.ego_x, y=float(lanes.centers[cfg.ego_lane]), psi=0.0, psidot=0.0,
                   vx=cfg.ego_v, vy=0.0, ax=0.0, ay=0.0)
    kat = [json.loads(s) for s in open("/root/reference/pkg/frontend/testdata/run.jsonl")][1:]
    seen = {}
    solve0 = planner.solver.solve

    def spy(batch, max_iter=150, tol=1e-3, warm=None, record_iterates=False, keep_multipliers=False):
        seen["batch"] = batch
        seen["warm"] = None if warm is None else warm.copy()
        return solve0(batch, max_iter=max_iter, tol=tol, warm=warm, record_iterates=record_iterates,
                      keep_multipliers=keep_multipliers)

    planner.solver.solve = spy
    seq_planner = Planner(pc, lanes, cfg.meta_spec)
    seq_planner.solver = SequentialSolver(seq_planner.solver)
    out = dict(l=pc.l, n=pc.n, t_f=pc.t_f, degree=pc.degree, rho=pc.rho_xy, max_iter=pc.max_iter,
               tol=pc.tol, m=pc.m, a=pc.a, b=pc.b, v_min=pc.v_min, v_max=pc.v_max, a_max=pc.a_max,
               h=pc.h, dt_cycle=pc.dt_cycle, warm_residual_cap=pc.warm_residual_cap,
               heading_limit=pc.limits.heading_limit, residual_tol=pc.limits.residual_tol,
               collision_margin=pc.limits.collision_margin, n_lanes=lanes.n_lanes,
               lane_width=lanes.width, lane_y0=lanes.y0, v_cruise=cfg.meta_spec.v_cruise,
               meta_v_max=cfg.meta_spec.v_max, y_rl=cfg.meta_spec.y_rl, w1=cfg.meta_spec.w1,
               w2=cfg.meta_spec.w2, cycles=cycles)
    for c in range(cycles):
        states = world.states()
        res = planner.mpc_cycle(ego, states)
        plan = res.plan
        sres = seq_planner.mpc_cycle(ego, states)
        hist = np.stack([[r.r_obs, r.r_acc, r.r_nonhol] for r in res.info.residual_history])
        # the reference's own recorded run (rounded by its log writer) must agree
        rec = kat[c]
        assert rec["best_index"] == plan.best_index
        assert np.allclose(rec["meta_costs"], plan.meta_cost, atol=1e-9, rtol=0)
        assert rec["command"]["accel"] == res.command.accel
        p = f"c{c}_"
        out[p + "ego"] = np.array([ego.x, ego.y, ego.psi, ego.psidot, ego.vx, ego.vy, ego.ax, ego.ay])
        out[p + "obstacles"] = np.array([[s.id, s.x, s.y, s.vx, s.vy, s.lane] for s in states])
        out[p + "meta_cost"] = plan.meta_cost
        out[p + "feasible"] = plan.feasible.astype(np.uint8)
        out[p + "min_ratio"] = plan.min_ratio
        out[p + "heading_max"] = plan.heading_max
        out[p + "best_index"] = np.int64(-1 if plan.best_index is None else plan.best_index)
        out[p + "command"] = np.array([res.command.accel, res.command.steering])
        out[p + "fallback"] = np.int64(res.fallback)
        out[p + "iterations"] = np.int64(res.info.iterations)
        out[p + "converged"] = np.int64(res.info.converged)
        out[p + "history"] = hist
        # the same closed loop with column-independent reference arithmetic
        out[p + "seq_best_index"] = np.int64(-1 if sres.plan.best_index is None else sres.plan.best_index)
        out[p + "seq_meta_cost"] = sres.plan.meta_cost
        out[p + "seq_feasible"] = sres.plan.feasible.astype(np.uint8)
        out[p + "seq_iterations"] = np.int64(sres.info.iterations)
        out[p + "seq_command"] = np.array([sres.command.accel, sres.command.steering])
        print(f"cycle {c}: sequential-arithmetic reference best {sres.plan.best_index}")
        # the reference's pick under column permutations / sequential solves
        planner.solver.solve = solve0
        b, w, l = seen["batch"], seen["warm"], seen["batch"].l
        prng = np.random.default_rng(100 + c)
        perms = [np.arange(l), np.arange(l)[::-1]] + [np.roll(np.arange(l), k) for k in range(1, l)]
        perms += [prng.permutation(l) for _ in range(8)]
        picks = {_ref_best(planner, b, w, pm, pc.max_iter, pc.tol) for pm in perms}
        picks.add(_ref_best_sequential(planner, b, w, pc.max_iter, pc.tol))
        assert plan.best_index in picks
        out[p + "ref_best_set"] = np.array(sorted(-1 if q is None else q for q in picks), dtype=np.int64)
        print(f"cycle {c}: reference best {plan.best_index}, picks under permutation {sorted(picks, key=str)}")
        planner.solver.solve = spy
        for k in ("x", "y", "psi", "psidot", "v"):
            out[p + k] = getattr(plan, k)
        ego = H._apply_command(ego, res.command, cfg.dt, cfg.h)
        world.step(cfg.dt, ego=VehicleState(id=-100, x=ego.x, y=ego.y, vx=ego.vx, vy=ego.vy,
                                            lane=lanes.lane_of(ego.y)))
    np.savez_compressed(HERE / "mpc_kat.npz", **out)
    print("mpc_kat", cycles, "cycles; matches testdata/run.jsonl")


def subset_fixture(name, cfg_name, seeds, l, iters, l_full=None):
    """Scenes with feasible candidates: each seed's full goal batch is solved by
    the reference, then the fixture keeps every feasible column plus the
    lowest-index others up to l and is re-solved (and screened) on that subset."""
    from paper_2109_10392_b200.scenes import CONFIGS, make_workload

    cfg = CONFIGS[cfg_name]
    parts = []
    for seed in seeds:
        Wf = make_workload(cfg_name, scenes=1, l=l_full, seed0=seed)
        solver = ref_solver(Wf.n, Wf.t_f, Wf.degree, Wf.m)
        batch = ProblemBatch(l=Wf.l, xi_x=Wf.xi_x[0], xi_y=Wf.xi_y[0], a=Wf.a, b=Wf.b, v_min=Wf.v_min,
                             v_max=Wf.v_max, a_max=Wf.a_max, b_xy=Wf.b_xy, b_psi=Wf.b_psi)
        st, info = solver.solve(batch, max_iter=cfg.iters, tol=0.0)
        sc = score(solver, st, info, batch, MetaCostSpec("cruise", v_cruise=20.0))
        feas = list(np.nonzero(sc["feasible"])[0])
        assert feas, f"{cfg_name} seed {seed} has no feasible candidate"
        others = [i for i in range(Wf.l) if i not in feas][: max(0, l - len(feas))]
        cols = np.array(sorted(feas[:l] + others))
        parts.append((Wf, cols))
    W = make_workload(cfg_name, scenes=len(seeds), l=l, seed0=0)
    for s, (Wf, cols) in enumerate(parts):
        W.xi_x[s], W.xi_y[s] = Wf.xi_x[0], Wf.xi_y[0]
        W.b_xy[:, s * l:(s + 1) * l] = Wf.b_xy[:, cols]
        W.b_psi[:, s * l:(s + 1) * l] = Wf.b_psi[:, cols]

    def check(o, info):
        assert o["cruise_best_index"] >= 0

    workload_fixture(name, W, iters, extra=check)


def main():
    t = time.time()
    only = set(sys.argv[1:])
    if only:
        for f in only:
            FIXTURES[f]()
        print(f"done in {time.time() - t:.1f}s")
        return
    mpc_kat()
    tail_case()
    demo()
    workload_fixture("c0", make_workload("c0"), 100)
    workload_fixture("c1", make_workload("c1"), 100)
    workload_fixture("c3s", make_workload("c3", scenes=4, l=64), 100)
    workload_fixture("c4s", make_workload("c4", scenes=2, l=32), 100)
    reverse_case()
    for f in ("c2s", "c2f", "c3f", "c4f"):
        FIXTURES[f]()
    print(f"done in {time.time() - t:.1f}s; reference version {batchmpc.__version__}")


FIXTURES = {
    "mpc_kat": mpc_kat,
    "tail_case": tail_case,
    "demo": demo,
    "reverse": reverse_case,
    "c2s": lambda: workload_fixture("c2s", make_workload("c2", l=256), 200),
    "c2f": lambda: subset_fixture("c2f", "c2", [4], 256, 200, l_full=1024),
    # seeds and l chosen from tests/golden/seed_search.py output
    "c3f": lambda: subset_fixture("c3f", "c3", [2, 4, 6, 10], 64, 100),
    "c4f": lambda: subset_fixture("c4f", "c4", C4F_SEEDS, 32, 100),
}
C4F_SEEDS = [2, 10]

if __name__ == "__main__":
    main()
