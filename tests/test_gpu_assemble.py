"""Device-side scene assembly (bmpc_assemble) == the host build_batch path
(select_nearest, predict_constant_velocity, boundary_vectors; planner.py:336-360,
traffic.py:199-233), bit for bit, including distance ties, scenes with fewer
vehicles than m (virtual padding) and scenes with none."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_assemble_matches_host(cuda):
    from paper_2109_10392_b200 import make_solver
    from paper_2109_10392_b200.device import assemble_scenes
    from paper_2109_10392_b200.planner import EgoState, Goal
    from paper_2109_10392_b200.traffic import VehicleState, predict_constant_velocity, select_nearest

    rng = np.random.default_rng(7)
    solver = make_solver(100, 5.0, 10, 10)
    m, l = 10, 7
    egos, vehs, goals = [], [], []
    for s in range(6):
        ego = EgoState(x=float(rng.uniform(-50, 50)), y=float(rng.choice([-5.25, -1.75, 1.75, 5.25])),
                       psi=float(rng.normal(0, 0.05)), psidot=float(rng.normal(0, 0.01)),
                       vx=float(rng.uniform(10, 25)), vy=float(rng.normal(0, 0.3)),
                       ax=float(rng.normal(0, 0.5)), ay=float(rng.normal(0, 0.1)))
        nv = [25, 3, 0, 10, 40, 12][s]
        vs = [VehicleState(id=i, x=float(ego.x + rng.uniform(-60, 150)),
                           y=float(rng.choice([-5.25, -1.75, 1.75, 5.25])),
                           vx=float(rng.uniform(5, 30)), vy=0.0, lane=0) for i in range(nv)]
        if nv >= 4:  # exact distance ties: mirrored about the ego
            vs[1] = VehicleState(id=1, x=2 * ego.x - vs[0].x, y=2 * ego.y - vs[0].y, vx=1.0, vy=0.0, lane=0)
            vs[3] = VehicleState(id=3, x=vs[2].x, y=vs[2].y, vx=2.0, vy=0.5, lane=0)
        egos.append(ego)
        vehs.append(vs)
        goals.append([Goal(x=float(ego.x + rng.uniform(50, 150)), y=float(rng.uniform(-5, 5)),
                           vx=float(rng.uniform(10, 30)), vy=0.0, ax=0.0, ay=0.0, lane=-1)
                      for _ in range(l)])
    prob = assemble_scenes(solver, egos, vehs, goals, m, 5.6, 2.4, 0.1, 35.0, 8.0)
    times = solver.basis.grid.times
    for s in range(6):
        near = select_nearest(vehs[s], egos[s].x, egos[s].y, m)
        xx, yy = predict_constant_velocity(near, times)
        np.testing.assert_array_equal(prob.xi_x[s].cpu().numpy(), xx)
        np.testing.assert_array_equal(prob.xi_y[s].cpu().numpy(), yy)
        e = egos[s]
        for i, g in enumerate(goals[s]):
            c = s * l + i
            np.testing.assert_array_equal(
                prob.b_xy[:, c].cpu().numpy(),
                [e.x, e.vx, e.ax, g.x, g.vx, g.ax, e.y, e.vy, e.ay, g.y, g.vy, g.ay])
            np.testing.assert_array_equal(prob.b_psi[:, c].cpu().numpy(), [e.psi, e.psidot, 0.0, 0.0])


def test_plan_states_equals_host_path(cuda):
    """plan_states (device assembly) == plan_batch over the host-assembled
    scenes, bit for bit."""
    from paper_2109_10392_b200 import make_solver
    from paper_2109_10392_b200.planner import (EgoState, FilterLimits, MetaCostSpec, PlannerConfig,
                                               plan_batch, plan_states, sample_goals_uniform)
    from paper_2109_10392_b200.traffic import VehicleState, predict_constant_velocity, select_nearest

    rng = np.random.default_rng(3)
    cfg = PlannerConfig(m=10, t_f=5.0, v_max=35.0, b=2.4)
    solver = make_solver(cfg.n, cfg.t_f, cfg.degree, cfg.m)
    egos, vehs, goals = [], [], []
    for s in range(3):
        ego = EgoState(x=0.0, y=float(rng.choice([-5.25, -1.75, 1.75, 5.25])), vx=float(rng.uniform(15, 25)))
        vs = [VehicleState(id=i, x=float(rng.uniform(-30, 120)), y=float(rng.choice([-5.25, -1.75, 1.75, 5.25])),
                           vx=float(rng.uniform(10, 25)), vy=0.0, lane=0) for i in range(14)]
        egos.append(ego)
        vehs.append(vs)
        goals.append(sample_goals_uniform(rng, ego, 64, cfg.t_f))
    spec, limits = MetaCostSpec("cruise", v_cruise=20.0), FilterLimits()
    dev = plan_states(solver, egos, vehs, goals, cfg, max_iter=40, tol=0.0, spec=spec, limits=limits)

    class Scenes:
        pass

    sc = Scenes()
    xs, ys = zip(*(predict_constant_velocity(select_nearest(v, e.x, e.y, cfg.m), solver.basis.grid.times)
                   for e, v in zip(egos, vehs)))
    sc.xi_x, sc.xi_y = np.stack(xs), np.stack(ys)
    cols = [(e, g) for e, gs in zip(egos, goals) for g in gs]
    sc.b_xy = np.array([[e.x, e.vx, e.ax, g.x, g.vx, g.ax, e.y, e.vy, e.ay, g.y, g.vy, g.ay]
                        for e, g in cols]).T.copy()
    sc.b_psi = np.array([[e.psi, e.psidot, 0.0, 0.0] for e, _ in cols]).T.copy()
    sc.l, sc.S = 64, 3
    sc.a, sc.b, sc.v_min, sc.v_max, sc.a_max = cfg.a, cfg.b, cfg.v_min, cfg.v_max, cfg.a_max
    host = plan_batch(solver, sc, max_iter=40, tol=0.0, spec=spec, limits=limits)
    for k in ("c_x", "c_y", "c_psi", "res_final", "meta_cost", "flags", "argmin_all", "argmin_hc"):
        np.testing.assert_array_equal(getattr(dev, k), getattr(host, k), err_msg=k)
    assert dev.best_index == host.best_index and dev.iterations == host.iterations == 40
