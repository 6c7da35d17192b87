"""Receding-horizon MPC cycle on the device against the reference's own
closed-loop run (cruise_idm, seed 7, l=11, warm starts with carried
multipliers, tol=1e-3, 200 sweeps): tests/golden/mpc_kat.npz was produced by
the reference planner + harness and cross-checked against its recorded
pkg/frontend/testdata/run.jsonl (tests/golden/make_golden.py::mpc_kat).
Ego and obstacle states per cycle come from that run, so the replay needs no
traffic simulation."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_mpc_cycles_match_reference_run(cuda):
    from paper_2109_10392_b200.planner import (EgoState, FilterLimits, LaneGeometry, MetaCostSpec,
                                               Planner, PlannerConfig)
    from paper_2109_10392_b200.traffic import VehicleState

    z = golden("mpc_kat")
    f = lambda k: float(z[k])  # noqa: E731
    i = lambda k: int(z[k])  # noqa: E731
    cfg = PlannerConfig(l=i("l"), n=i("n"), t_f=f("t_f"), degree=i("degree"), rho_xy=f("rho"),
                        max_iter=i("max_iter"), tol=f("tol"), m=i("m"), a=f("a"), b=f("b"),
                        v_min=f("v_min"), v_max=f("v_max"), a_max=f("a_max"), h=f("h"),
                        dt_cycle=f("dt_cycle"), warm_start=True,
                        warm_residual_cap=f("warm_residual_cap"),
                        limits=FilterLimits(f("heading_limit"), f("residual_tol"),
                                            f("collision_margin")))
    lanes = LaneGeometry(i("n_lanes"), f("lane_width"), f("lane_y0"))
    meta = MetaCostSpec("cruise", v_cruise=f("v_cruise"), v_max=f("meta_v_max"), y_rl=f("y_rl"),
                        w1=f("w1"), w2=f("w2"))
    planner = Planner(cfg, lanes, meta)
    for c in range(i("cycles")):
        p = f"c{c}_"
        e = z[p + "ego"]
        ego = EgoState(x=e[0], y=e[1], psi=e[2], psidot=e[3], vx=e[4], vy=e[5], ax=e[6], ay=e[7])
        vehicles = [VehicleState(id=int(r[0]), x=r[1], y=r[2], vx=r[3], vy=r[4], lane=int(r[5]))
                    for r in z[p + "obstacles"]]
        res = planner.mpc_cycle(ego, vehicles)
        plan = res.plan
        best = -1 if plan.best_index is None else plan.best_index
        ref_best = int(z[p + "best_index"])
        # Round-robin goals repeat every 4 columns (planner.py:96-110) and the
        # lanes either side of the ego mirror each other, so several candidates
        # tie to ~1e-11.  The batch reference's pick among them depends on the
        # column's position in its BLAS calls: make_golden.py re-ran each
        # cycle's solve with permuted columns (ref_best_set: cycle 0 picks any
        # of {0,2,4,6,8,10}) and replayed the whole closed loop with the
        # reference solving one column at a time (its own batch-vs-sequential
        # oracle, oracles.py:270-293).  That column-independent reference run
        # is what this solver's arithmetic corresponds to, so its pick must be
        # ours exactly; against the batch run we require the same tie class.
        seq_best = int(z[p + "seq_best_index"])
        assert best == seq_best, (c, best, seq_best)
        np.testing.assert_array_equal(plan.feasible, z[p + "seq_feasible"].astype(bool))
        np.testing.assert_allclose(plan.meta_cost, z[p + "seq_meta_cost"], rtol=1e-8, atol=1e-10)
        assert res.info.iterations == int(z[p + "seq_iterations"])
        ref_cost, ref_feas = z[p + "meta_cost"], z[p + "feasible"].astype(bool)
        if ref_best < 0:
            assert best == -1
        else:
            assert best >= 0 and ref_feas[best], c
            assert abs(ref_cost[best] - ref_cost[ref_best]) <= 1e-9 * ref_cost[ref_best], c
        if c == 0:  # no warm start yet: the permutation set is the whole tie class
            assert best in set(z[p + "ref_best_set"].tolist()), (best, z[p + "ref_best_set"])
        assert res.fallback == bool(z[p + "fallback"])
        assert res.info.iterations == int(z[p + "iterations"])
        assert res.info.converged == bool(z[p + "converged"])
        np.testing.assert_array_equal(plan.feasible, z[p + "feasible"].astype(bool))
        # costs are sums of (v - v_cruise)^2 with v ~ v_cruise: the cancellation
        # turns ~1e-12 trajectory differences into ~1e-11 absolute; the
        # reference's own log keeps 9 decimals (harness.py:366)
        np.testing.assert_allclose(plan.meta_cost, z[p + "meta_cost"], rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(plan.min_ratio, z[p + "min_ratio"], rtol=1e-8)
        np.testing.assert_allclose(plan.heading_max, z[p + "heading_max"], rtol=1e-6, atol=1e-12)
        for k in ("x", "y", "psi", "psidot", "v"):
            ref = z[p + k]
            err = np.abs(getattr(plan, k) - ref).max(axis=0) / np.maximum(1.0, np.abs(ref).max(axis=0))
            assert err.max() <= 1e-8, (c, k, err.max())
        if best >= 0:
            # the control the reference extracts from the candidate we picked
            from paper_2109_10392_b200.planner import Candidate, extract_control

            cand = Candidate(x=z[p + "x"][:, best], y=z[p + "y"][:, best], psi=z[p + "psi"][:, best],
                             psidot=z[p + "psidot"][:, best], v=z[p + "v"][:, best], xddot=None,
                             yddot=None)
            ref_cmd = extract_control(cand, cfg.h, planner.basis.grid.dt, cfg.dt_cycle)
            ref_accel = float(np.clip(ref_cmd.accel, -cfg.a_max, cfg.a_max))
            np.testing.assert_allclose(res.command.accel, ref_accel, rtol=1e-6, atol=1e-10)
            np.testing.assert_allclose(res.command.steering, ref_cmd.steering, rtol=1e-6, atol=1e-10)
            if best == ref_best:
                np.testing.assert_allclose([res.command.accel, res.command.steering],
                                           z[p + "command"], rtol=1e-6, atol=1e-10)
            np.testing.assert_allclose([res.command.accel, res.command.steering],
                                       z[p + "seq_command"], rtol=1e-6, atol=1e-10)
        hist = np.stack([[r.r_obs, r.r_acc, r.r_nonhol] for r in res.info.residual_history])
        np.testing.assert_allclose(hist, z[p + "history"], rtol=1e-6, atol=1e-9)
        print(f"cycle {c}: best {best}, accel {res.command.accel:.6e} "
              f"(ref {z[p + 'command'][0]:.6e}), solve {1e3 * res.solve_time:.2f} ms")
