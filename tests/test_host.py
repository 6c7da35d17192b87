"""Host-side logic: constants, KKT inverses, validation, the scene generator,
and that the sm_100a library loads and exports its C ABI.  CPU only."""

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

import am_oracle as O
from paper_2109_10392_b200 import (BatchSolver, ProblemBatch, build_basis, build_constant_matrices,
                                   build_time_grid, make_solver)
from paper_2109_10392_b200 import _native
from paper_2109_10392_b200.basis import BoundarySpec
from paper_2109_10392_b200.scenes import CONFIGS, ELLIPSE_A, ELLIPSE_B, LANES, make_workload
from paper_2109_10392_b200.solver import KktSystem, _inverse_ext
from paper_2109_10392_b200.dist import local_winner, merge_winners, shard_range

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("n,t_f,deg,m", [(100, 5.0, 10, 10), (200, 10.0, 15, 50), (50, 10.0, 10, 4)])
def test_constants_bitwise_equal_oracle(n, t_f, deg, m):
    s = make_solver(n, t_f, deg, m)
    o = O.OracleSolver(n, t_f, deg, m)
    for a, b in ((s.basis.P, o.P), (s.basis.Pdot, o.Pdot), (s.basis.Pddot, o.Pddot),
                 (s.mats.F_axis, o.F_axis), (s.mats.Q, o.Q), (s.kkt.matrix_xy, o.matrix_xy),
                 (s.kkt.matrix_psi, o.matrix_psi)):
        np.testing.assert_array_equal(a, b)


def test_basis_properties():
    b = build_basis(build_time_grid(0.0, 10.0, 100), 10)
    np.testing.assert_allclose(b.P.sum(axis=1), 1.0, atol=1e-14)
    np.testing.assert_allclose(b.Pdot.sum(axis=1), 0.0, atol=1e-12)
    assert b.P[0, 0] == 1.0 and b.P[-1, -1] == 1.0
    with pytest.raises(ValueError):
        build_basis(build_time_grid(0.0, 1.0, 10), 2)
    with pytest.raises(ValueError):
        build_time_grid(0.0, 0.0, 10)
    with pytest.raises(ValueError):
        build_constant_matrices(b, -1)


@pytest.mark.parametrize("n,t_f,deg,m", [(100, 5.0, 10, 10), (200, 10.0, 15, 50)])
def test_kkt_inverse_matches_refined_lu(n, t_f, deg, m, rng):
    s = make_solver(n, t_f, deg, m)
    o = O.OracleSolver(n, t_f, deg, m)
    nb = s.basis.n_b
    rhs = rng.normal(0, 100.0, (2 * nb + 12, 64))
    ref = o._refined_solve(o.lu_xy, o.matrix_xy, rhs)
    got = s.kkt.solve_xy(rhs)
    assert np.abs(got - ref).max() <= 1e-7 * np.abs(ref).max()
    # the device applies only the per-axis coefficient rows
    idx = np.r_[0:nb, 2 * nb:2 * nb + 6]
    cx = s.kkt.kinv_axis @ rhs[idx]
    assert np.abs(cx - ref[:nb]).max() <= 1e-7 * max(1.0, np.abs(ref[:nb]).max())
    rp = rng.normal(0, 1.0, (nb + 4, 16))
    refp = o._refined_solve(o.lu_psi, o.matrix_psi, rp)
    assert np.abs(s.kkt.kinv_psi @ rp - refp[:nb]).max() <= 1e-9 * max(1.0, np.abs(refp).max())
    assert s.kkt.n_factorizations == 2


def test_inverse_ext_singular():
    with pytest.raises(np.linalg.LinAlgError):
        _inverse_ext(np.zeros((3, 3)))


def test_problem_batch_validation():
    z = np.zeros((12, 2))
    ok = dict(l=2, xi_x=np.zeros(10), xi_y=np.zeros(10), a=5.6, b=3.1, v_min=0.1, v_max=20.0,
              a_max=8.0, b_xy=z, b_psi=np.zeros((4, 2)))
    ProblemBatch(**ok)
    for bad in (dict(v_min=0.0), dict(v_min=30.0), dict(a_max=0.0), dict(a=1.0, b=2.0),
                dict(rho_xy=0.0), dict(xi_y=np.zeros(9)), dict(b_xy=np.zeros((12, 3)))):
        with pytest.raises(ValueError):
            ProblemBatch(**{**ok, **bad})


def test_solver_validation():
    g = build_time_grid(0.0, 5.0, 100)
    b1, b2 = build_basis(g, 10), build_basis(g, 10)
    with pytest.raises(ValueError):
        BatchSolver(b1, build_constant_matrices(b2, 10))
    with pytest.raises(ValueError):
        make_solver(100, 5.0, 17, 10)  # n_b = 18 > 16
    with pytest.raises(ValueError):
        BatchSolver(b1, build_constant_matrices(b1, 10, BoundarySpec(end_orders=(0, 1))))
    s = make_solver(100, 5.0, 10, 10)
    bad = ProblemBatch(l=1, xi_x=np.zeros(999), xi_y=np.zeros(999), a=5.6, b=3.1, v_min=0.1,
                       v_max=20.0, a_max=8.0, b_xy=np.zeros((12, 1)), b_psi=np.zeros((4, 1)))
    with pytest.raises(ValueError):
        s._check_batch(bad)


def test_scene_generator_deterministic_and_spawn_rule():
    for name in ("c0", "c1", "c3"):
        cfg = CONFIGS[name]
        W1 = make_workload(name, scenes=3)
        W2 = make_workload(name, scenes=3)
        np.testing.assert_array_equal(W1.xi_x, W2.xi_x)
        np.testing.assert_array_equal(W1.b_xy, W2.b_xy)
        assert W1.xi_x.shape == (3, cfg.m * cfg.n)
        n = cfg.n
        for s in range(3):
            y_ego = W1.b_xy[6, s * W1.l]
            x0 = W1.xi_x[s].reshape(cfg.m, n)[:, 0]
            y0 = W1.xi_y[s].reshape(cfg.m, n)[:, 0]
            ratio = np.hypot(x0 / ELLIPSE_A, (y0 - y_ego) / ELLIPSE_B)
            assert ratio.min() >= 1.5
            assert set(np.round(y0[y0 < 1e3], 2)) <= set(np.round(LANES, 2))
    W = make_workload("c0")
    assert W.L == 110 and W.b_xy[3].max() == pytest.approx(30.0 * 5.0)


def test_shard_ranges_cover():
    for total in (0, 1, 7, 1024, 16384):
        for world in (1, 2, 3, 8):
            got = [shard_range(total, r, world) for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == total
            for (a, b), (c, d) in zip(got, got[1:]):
                assert b == c


def test_merge_winners_tie_rule(rng):
    cost = rng.integers(0, 5, 64).astype(float)
    feas = rng.random(64) < 0.5
    for world in (1, 2, 4, 8):
        recs = []
        for r in range(world):
            lo, hi = shard_range(64, r, world)
            recs.append(local_winner(cost[lo:hi], feas[lo:hi], lo))
        best, nf = merge_winners(np.stack(recs))
        assert best == int(np.argmin(np.where(feas, cost, np.inf)))
        assert nf == int(feas.sum())
    assert merge_winners(np.array([[np.inf, -1, 0], [np.inf, -1, 0]])) == (None, 0)


def test_native_library_exports_every_header_symbol():
    assert _native.LIB_PATH.exists(), "build first (__graft_entry__.build())"
    header = (ROOT / "include" / "batchmpc_b200.h").read_text()
    names = set(re.findall(r"^(?:int|const char\*)\s+(bmpc_\w+)\(", header, flags=re.M))
    assert len(names) >= 15
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for nm in names:
        assert hasattr(lib, nm), nm
    assert names <= set(_native.EXPORTS)
    lib2 = _native.load()
    assert lib2.bmpc_abi_version() == 2


def test_ctypes_struct_layout_matches_c():
    """The ctypes Structures have the C sizes and field offsets (bmpc_abi_layout
    needs no GPU)."""
    lib = _native.load()
    n = lib.bmpc_abi_layout(None, 0)
    buf = (ctypes.c_longlong * n)()
    lib.bmpc_abi_layout(buf, n)
    got = list(buf)
    exp = []
    for cls, last in ((_native.Problem, "a_max"), (_native.SolveOpts, "team_warps"),
                      (_native.SolveOut, "converged"), (_native.ScoreSpec, "collision_margin"),
                      (_native.ScoreOut, "n_feasible")):
        exp += [ctypes.sizeof(cls), getattr(cls, last).offset]
    assert got == exp


def test_no_oracle_in_product_package():
    pkg = ROOT / "paper_2109_10392_b200"
    for p in pkg.rglob("*.py"):
        txt = p.read_text()
        assert "am_oracle" not in txt and "oracle/" not in txt, p


def test_ctypes_arity_matches_header():
    """Every prototype in include/batchmpc_b200.h has the argument count the
    ctypes binding declares (a mismatch would corrupt the call)."""
    header = (ROOT / "include" / "batchmpc_b200.h").read_text()
    body = re.sub(r"/\*.*?\*/", "", header, flags=re.S)
    for m in re.finditer(r"^(?:int|const char\*)\s+(bmpc_\w+)\((.*?)\);", body, flags=re.M | re.S):
        name, params = m.group(1), m.group(2).strip()
        n = 0 if params in ("", "void") else params.count(",") + 1
        assert len(_native.EXPORTS[name][0]) == n, (name, n, len(_native.EXPORTS[name][0]))


@pytest.mark.parametrize("n,t_f,deg,m", [(100, 5.0, 10, 10), (200, 10.0, 15, 50), (40, 2.0, 6, 2)])
def test_null_space_qp_matches_kkt_solve(n, t_f, deg, m, rng):
    """bmpc_reduced_qp (the persistent solve's QP form, host-only C ABI): the
    boundary rows fix the end coefficients, c = Z rhs + B b; it must reproduce
    the coefficient part of the reference's per-axis / heading KKT solves."""
    lib = _native.load()
    s = make_solver(n, t_f, deg, m)
    nb = s.basis.n_b
    conds = {}
    for name, K, rows in (("xy", s.kkt.matrix_axis, 6), ("psi", s.kkt.matrix_psi, 4)):
        K = np.ascontiguousarray(K, dtype=np.float64)
        Z, B = np.zeros((nb, nb)), np.zeros((nb, rows))
        cond = ctypes.c_double()
        assert lib.bmpc_reduced_qp(nb, rows, _native.c_double_ptr(K), _native.c_double_ptr(Z),
                                   _native.c_double_ptr(B), ctypes.byref(cond)) == 0
        conds[name] = cond.value
        rhs = rng.normal(0, 100.0, (nb, 32))
        b = rng.normal(0, 10.0, (rows, 32))
        ref = np.linalg.solve(K, np.vstack([rhs, b]))[:nb]
        got = Z @ rhs + B @ b
        tol = 1e-9 if cond.value < 1e4 else 1e-7
        assert np.abs(got - ref).max() <= tol * max(1.0, np.abs(ref).max()), name
        # boundary rows hold exactly: A c = b
        A = K[nb:, :nb]
        assert np.abs(A @ got - b).max() <= 1e-9 * max(1.0, np.abs(b).max())
    if (n, deg) == (100, 10):
        assert conds["xy"] < 1e4 and conds["psi"] < 1e4   # no refinement on c0-c3
    if (n, deg) == (200, 15):
        assert conds["xy"] > 1e4                           # c4 refines
    bad = np.zeros(((nb + 6) * (nb + 6)))
    assert lib.bmpc_reduced_qp(nb, 6, _native.c_double_ptr(bad), _native.c_double_ptr(np.zeros((nb, nb))),
                               _native.c_double_ptr(np.zeros((nb, 6))), ctypes.byref(ctypes.c_double())) != 0


REF_SRC = Path("/root/reference/pkg/src")


def test_solver_accepts_foreign_boundary_spec():
    """The solver swap of INTEGRATION.md passes the reference's own basis and
    constant-matrix objects: a BoundarySpec of another class with the default
    orders is accepted, non-default orders are refused."""
    import dataclasses

    @dataclasses.dataclass(frozen=True)
    class OtherSpec:
        start_orders: tuple = (0, 1, 2)
        end_orders: tuple = (0, 1, 2)
        psi_start_orders: tuple = (0, 1)
        psi_end_orders: tuple = (0, 1)

    b = build_basis(build_time_grid(0.0, 5.0, 100), 10)
    mats = build_constant_matrices(b, 10)
    BatchSolver(b, dataclasses.replace(mats, boundary=OtherSpec()))
    with pytest.raises(ValueError, match="BoundarySpec"):
        BatchSolver(b, dataclasses.replace(mats, boundary=OtherSpec(end_orders=(0, 1))))


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference tree not present (GPU box)")
def test_solver_from_reference_basis_and_matrices():
    """BatchSolver(ref_basis, ref_mats): built from the reference's batchmpc.basis
    objects, with KKT matrices bitwise equal to ours."""
    import sys

    sys.path.insert(0, str(REF_SRC))
    try:
        import batchmpc.basis as RB
    finally:
        sys.path.remove(str(REF_SRC))
    rb = RB.build_basis(RB.build_time_grid(0.0, 5.0, 100), 10)
    rm = RB.build_constant_matrices(rb, 10)
    s = BatchSolver(rb, rm, 1.0)
    ours = make_solver(100, 5.0, 10, 10)
    np.testing.assert_array_equal(s.kkt.matrix_xy, ours.kkt.matrix_xy)
    np.testing.assert_array_equal(s.kkt.matrix_psi, ours.kkt.matrix_psi)


def test_check_scenes_validation():
    """plan_batch / solve validate stacked scene batches before any host buffer
    is handed to the C ABI (shapes against S, l, m, n; rho; the scalars)."""
    import dataclasses

    s = make_solver(100, 5.0, 10, 20)
    W = make_workload("c3", scenes=2, l=8)
    xi_x, xi_y, S, l = s.check_scenes(W)
    assert (S, l) == (2, 8) and xi_x.shape == (2, 2000)
    bad = [dataclasses.replace(W, b_xy=W.b_xy[:, :-1]), dataclasses.replace(W, b_psi=W.b_psi[:3]),
           dataclasses.replace(W, xi_x=W.xi_x[:1]), dataclasses.replace(W, xi_y=W.xi_y[:, :-100]),
           dataclasses.replace(W, rho=2.0), dataclasses.replace(W, v_min=0.0),
           dataclasses.replace(W, S=3)]
    for b in bad:
        with pytest.raises(ValueError):
            s.check_scenes(b)
    m10 = make_workload("c1", scenes=1, l=4)  # m = 10 predictions for an m = 20 solver
    with pytest.raises(ValueError):
        s.check_scenes(m10)
