"""The CPU oracle is pinned against outputs of the reference itself (golden
fixtures made by tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

import am_oracle as O
from conftest import golden


def _args(s):
    return (s["x"], s["y"], s["xdot"], s["ydot"], s["xddot"], s["yddot"], s["psi"],
            s["xi_x"], s["xi_y"], 0.1, 20.0, 8.0, 5.6, 3.1)


@pytest.mark.parametrize("kind,tag", [("c", "ref"), ("numpy", "np")])
def test_oracle_kernels_bitwise_vs_reference(kind, tag):
    s = golden("tail_case")
    k = O.kernels(kind)
    core = k.tail_core(*_args(s))
    for name, got in zip(("d", "d_a", "v", "r_x", "r_y", "g_x", "g_y", "sq_obs", "sq_acc", "sq_nonhol"), core):
        np.testing.assert_array_equal(got, s[f"{tag}_core_{name}"], err_msg=name)
    al, d = k.obstacle_update(s["x"], s["y"], s["xi_x"], s["xi_y"], 5.6, 3.1)
    np.testing.assert_array_equal(al, s[f"{tag}_obs_alpha"])
    np.testing.assert_array_equal(d, s[f"{tag}_obs_d"])
    al, da = k.accel_update(s["xddot"], s["yddot"], 8.0)
    np.testing.assert_array_equal(al, s[f"{tag}_acc_alpha_a"])
    np.testing.assert_array_equal(da, s[f"{tag}_acc_d_a"])
    np.testing.assert_array_equal(k.v_update(s["xdot"], s["ydot"], 0.1, 20.0), s[f"{tag}_v"])
    gx, gy = k.assemble_g(s["xi_x"], s["xi_y"], s["alpha"], s["d"], s["alpha_a"], s["d_a"], s["v"],
                          s["psi"], 5.6, 3.1)
    np.testing.assert_array_equal(gx, s[f"{tag}_g_x"])
    np.testing.assert_array_equal(gy, s[f"{tag}_g_y"])


def test_reference_backends_agree_like_reference_test():
    # the reference's own cross-backend tolerance (tests/test_kernels.py:104-113)
    s = golden("tail_case")
    for name in ("d", "d_a", "v", "r_x", "r_y", "g_x", "g_y", "sq_obs", "sq_acc", "sq_nonhol"):
        assert np.abs(s[f"ref_core_{name}"] - s[f"np_core_{name}"]).max() <= 1e-10


def _oracle_solve(z, s=0, kernel="c", iters=None):
    l = int(z["l"])
    cols = slice(s * l, (s + 1) * l)
    osol = O.OracleSolver(int(z["n"]), float(z["t_f"]), int(z["degree"]), int(z["m"]))
    xi_x = z["xi_x"][s] if z["xi_x"].ndim == 2 else z["xi_x"]
    xi_y = z["xi_y"][s] if z["xi_y"].ndim == 2 else z["xi_y"]
    r = osol.solve(xi_x, xi_y, z["b_xy"][:, cols], z["b_psi"][:, cols], float(z["a"]), float(z["b"]),
                   float(z["v_min"]), float(z["v_max"]), float(z["a_max"]), int(iters or z["iters"]),
                   kernel=kernel)
    return osol, r, cols


@pytest.mark.parametrize("name", ["demo", "c0", "reverse", "c2f"])
def test_oracle_solver_matches_reference(name):
    z = golden(name)
    _, r, cols = _oracle_solve(z)
    for k in ("c_x", "c_y", "c_psi", "lambda_x", "lambda_y", "lambda_psi"):
        ref = z[k][:, cols]
        scale = max(1.0, float(np.abs(ref).max()))
        assert np.abs(r[k] - ref).max() <= 1e-12 * scale, k


@pytest.mark.parametrize("name,s", [("c0", 0), ("c3f", 0), ("c3f", 2)])
def test_oracle_scoring_matches_reference(name, s):
    """Scene s of a golden: the oracle's solve + scoring reproduce the
    reference's meta costs, feasibility and indices (c3f: real best indices)."""
    z = golden(name)
    osol, r, cols = _oracle_solve(z, s=s)
    sc = osol.score(r, z["xi_x"][s], z["xi_y"][s], float(z["a"]), float(z["b"]), kind="cruise",
                    v_cruise=20.0)
    np.testing.assert_allclose(sc["meta_cost"], z["cruise_meta_cost"][cols], rtol=1e-12)
    np.testing.assert_array_equal(sc["feasible"], z["cruise_feasible"][cols].astype(bool))
    best = int(z["cruise_best_index"][s])
    assert (sc["best_index"] if sc["best_index"] is not None else -1) == best
    assert sc["argmin_all"] == int(z["cruise_argmin_all"][s])
    if name == "c3f":
        assert best >= 0


def test_oracle_demo_history_and_aux():
    z = golden("demo")
    _, r, _ = _oracle_solve(z)
    np.testing.assert_allclose(r["history"], z["history"], rtol=1e-10, atol=1e-14)
    for k in ("v", "d_a", "alpha_a", "d", "alpha"):
        assert np.abs(r[k] - z[k]).max() <= 1e-10, k


def test_ref_kernels_equal_c_restatement():
    ref = O._load_ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    s = golden("tail_case")
    for a, b in zip(ref.tail_core(*_args(s)), O.kernels("c").tail_core(*_args(s))):
        np.testing.assert_array_equal(np.asarray(a), b)
