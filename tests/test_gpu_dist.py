"""plan_sharded across 2 ranks sharing cuda:0 (gloo for the collectives: the
GPU boxes here have one GPU) against the single-rank plan_batch, bit for bit.

Covers both partitions of SURVEY.md section 8e -- goal columns of one scene
(c1, c3f scene 0) and scene blocks (c3s, c3f) -- and the global early-stop rule
across shards (solver.py:437-439) with ranks whose local solves converge at
different sweeps.  Ranks on one device do not wait on each other inside a
kernel, so sharing the GPU is safe (the collectives are host-side gloo)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _Scenes:
    def __init__(self, z, s_lo=0, s_hi=None):
        S = np.atleast_2d(z["xi_x"]).shape[0]
        s_hi = S if s_hi is None else s_hi
        l = int(z["l"])
        self.xi_x = np.atleast_2d(z["xi_x"])[s_lo:s_hi]
        self.xi_y = np.atleast_2d(z["xi_y"])[s_lo:s_hi]
        self.b_xy = np.ascontiguousarray(z["b_xy"][:, s_lo * l:s_hi * l])
        self.b_psi = np.ascontiguousarray(z["b_psi"][:, s_lo * l:s_hi * l])
        self.l, self.S = l, s_hi - s_lo
        self.a, self.b = float(z["a"]), float(z["b"])
        self.v_min, self.v_max, self.a_max = float(z["v_min"]), float(z["v_max"]), float(z["a_max"])
        self.rho = 1.0


def _run(name, s_hi, iters, tol):
    from paper_2109_10392_b200 import make_solver
    from paper_2109_10392_b200.dist import plan_sharded
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec

    z = golden(name)
    solver = make_solver(int(z["n"]), float(z["t_f"]), int(z["degree"]), int(z["m"]))
    r = plan_sharded(solver, _Scenes(z, 0, s_hi), max_iter=iters, tol=tol,
                     spec=MetaCostSpec("cruise", v_cruise=20.0), limits=FilterLimits())
    return dict(best=[-1 if b is None else b for b in r.best_index], amin=r.argmin_all.tolist(),
                ahc=r.argmin_hc.tolist(), nf=r.n_feasible.tolist(), cost=r.best_cost.tolist(),
                coef=[None if c is None else c.tolist() for c in r.best_coef],
                iters=r.iterations, conv=r.converged, mode=r.mode)


def _worker(rank, world, port, cases, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = [_run(*c) for c in cases]
    finally:
        dist.destroy_process_group()


CASES = [("c3s", None, 40, 0.0), ("c3f", None, 100, 0.0), ("c3f", 1, 100, 0.0), ("c1", None, 30, 0.0)]


def test_plan_sharded_world2_equals_single(cuda):
    mgr = mp.Manager()
    out = mgr.dict()
    single = [_run(*c) for c in CASES]  # no process group: world 1
    mp.spawn(_worker, args=(2, _free_port(), CASES, out), nprocs=2, join=True)
    for r in (0, 1):
        for got, want, case in zip(out[r], single, CASES):
            assert got == want, (r, case)
    modes = [s["mode"] for s in single]
    assert modes == ["scenes", "scenes", "goals", "goals"]
    assert all(b >= 0 for b in single[1]["best"]) and single[2]["best"][0] >= 0


def test_plan_sharded_single_matches_plan_batch(cuda):
    """world 1: plan_sharded's reductions reproduce plan_batch's own argmins."""
    from paper_2109_10392_b200 import make_solver
    from paper_2109_10392_b200.planner import FilterLimits, MetaCostSpec, plan_batch

    z = golden("c3f")
    solver = make_solver(int(z["n"]), float(z["t_f"]), int(z["degree"]), int(z["m"]))
    pb = plan_batch(solver, _Scenes(z), max_iter=100, tol=0.0, spec=MetaCostSpec("cruise", v_cruise=20.0),
                    limits=FilterLimits())
    got = _run("c3f", None, 100, 0.0)
    assert got["best"] == [-1 if b is None else b for b in pb.best_index]
    assert got["amin"] == pb.argmin_all.tolist() and got["ahc"] == pb.argmin_hc.tolist()
    l = int(z["l"])
    for s, b in enumerate(got["best"]):
        g = s * l + b
        np.testing.assert_array_equal(np.array(got["coef"][s]),
                                      np.stack([pb.c_x[:, g], pb.c_y[:, g], pb.c_psi[:, g]]))
        assert got["cost"][s] == pb.meta_cost[g]
    one = _run("c3f", 1, 100, 0.0)  # one scene: the goal-column reductions
    assert one["best"][0] == got["best"][0] and one["amin"][0] == got["amin"][0]


# demo columns reordered so the two shards differ: classes 1/2 (low residuals)
# on rank 0, classes 0/3 on rank 1 (the demo's goals repeat every 4 columns)
TOL_COLS = [1, 2, 5, 6, 0, 3, 4, 7]


def _demo_batch():
    from paper_2109_10392_b200 import ProblemBatch

    z = golden("demo")
    c = TOL_COLS
    return ProblemBatch(l=len(c), xi_x=z["xi_x"], xi_y=z["xi_y"], a=float(z["a"]), b=float(z["b"]),
                        v_min=float(z["v_min"]), v_max=float(z["v_max"]), a_max=float(z["a_max"]),
                        b_xy=np.ascontiguousarray(z["b_xy"][:, c]), b_psi=np.ascontiguousarray(z["b_psi"][:, c]))


def _worker_tol(rank, world, port, tol, out):
    import torch
    import torch.distributed as dist

    from paper_2109_10392_b200 import make_solver
    from paper_2109_10392_b200.dist import plan_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        solver = make_solver(100, 10.0, 10, 10)
        r = plan_sharded(solver, _demo_batch(), max_iter=60, tol=tol)
        out[rank] = (r.iterations, r.converged, r.local.iterations, r.local.c_x.tolist())
    finally:
        dist.destroy_process_group()


def test_plan_sharded_global_early_stop(cuda):
    """Two shards whose local solves first meet tol at different sweeps: both
    ranks stop at the single-GPU sweep count (solver.py:437-439) and their
    columns equal the single-GPU solve's."""
    from paper_2109_10392_b200 import make_solver

    solver = make_solver(100, 10.0, 10, 10)
    b = _demo_batch()
    sol = solver.solve_device(solver.device_problem(b), max_iter=60, tol=-1.0)
    h = sol.history[:60].cpu().numpy()  # (60, 3, 8)
    w0, w1 = h[:, :, :4].max(axis=(1, 2)), h[:, :, 4:].max(axis=(1, 2))
    g = np.maximum(w0, w1)

    def first(w, tol):
        ok = np.nonzero(w <= tol)[0]
        return int(ok[0]) + 1 if ok.size else None

    tol = None
    for t in range(10, 60):  # a tol rank 0 meets strictly before the whole batch does
        cand = float(g[t]) * (1 + 1e-9)
        f0, fg = first(w0, cand), first(g, cand)
        if f0 is not None and fg is not None and f0 < fg:
            tol = cand
            break
    assert tol is not None, (w0, w1)
    expect = (first(g, tol), True)
    single, info = solver.solve(b, max_iter=60, tol=tol)
    assert (info.iterations, info.converged) == expect
    print(f"tol {tol:.3e}: rank 0 alone stops at {first(w0, tol)}, rank 1 at {first(w1, tol)}, "
          f"globally {expect[0]}")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_tol, args=(2, _free_port(), tol, out), nprocs=2, join=True)
    for r, cols in ((0, slice(0, 4)), (1, slice(4, 8))):
        it, conv, lit, cx = out[r]
        assert (it, conv) == expect and lit == expect[0]
        np.testing.assert_array_equal(np.array(cx), single.c_x[:, cols])
