"""Operator-level CUDA kernels vs the reference's compiled kernels (golden
fixture) -- the reference's own backend-equivalence bars
(tests/test_kernels.py:72-113): <= 1e-12 per kernel, tail_core <= 1e-10."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def _args(s):
    return (s["x"], s["y"], s["xdot"], s["ydot"], s["xddot"], s["yddot"], s["psi"],
            s["xi_x"], s["xi_y"], 0.1, 20.0, 8.0, 5.6, 3.1)


def test_tail_core_vs_reference(cuda):
    from paper_2109_10392_b200 import kernels

    s = golden("tail_case")
    got = kernels.tail_core(*_args(s))
    names = ("d", "d_a", "v", "r_x", "r_y", "g_x", "g_y", "sq_obs", "sq_acc", "sq_nonhol")
    for name, g in zip(names, got):
        ref = s[f"ref_core_{name}"]
        assert isinstance(g, np.ndarray) and g.shape == ref.shape
        assert np.abs(g - ref).max() <= 1e-10, name
    # obstacle and accel blocks use only IEEE add/mul/div/sqrt: bit-identical
    for name in ("d", "d_a"):
        np.testing.assert_array_equal(got[names.index(name)], s[f"ref_core_{name}"])
    mn = s["xi_x"].shape[0]
    np.testing.assert_array_equal(got[3][:mn], s["ref_core_r_x"][:mn])


def test_tail_update_and_simple_kernels(cuda):
    from paper_2109_10392_b200 import kernels

    s = golden("tail_case")
    for name, g in zip(("alpha", "d", "alpha_a", "d_a", "v", "r_x", "r_y", "g_x", "g_y"),
                       kernels.tail_update(*_args(s))):
        assert np.abs(g - s[f"ref_upd_{name}"]).max() <= 1e-12, name
    al, d = kernels.obstacle_update(s["x"], s["y"], s["xi_x"], s["xi_y"], 5.6, 3.1)
    assert np.abs(al - s["ref_obs_alpha"]).max() <= 1e-12
    assert np.abs(d - s["ref_obs_d"]).max() <= 1e-12
    al, da = kernels.accel_update(s["xddot"], s["yddot"], 8.0)
    assert np.abs(al - s["ref_acc_alpha_a"]).max() <= 1e-12
    np.testing.assert_array_equal(da, s["ref_acc_d_a"])
    np.testing.assert_array_equal(kernels.v_update(s["xdot"], s["ydot"], 0.1, 20.0), s["ref_v"])
    gx, gy = kernels.assemble_g(s["xi_x"], s["xi_y"], s["alpha"], s["d"], s["alpha_a"], s["d_a"],
                                s["v"], s["psi"], 5.6, 3.1)
    assert np.abs(gx - s["ref_g_x"]).max() <= 1e-12 and np.abs(gy - s["ref_g_y"]).max() <= 1e-12
    rx, ry = kernels.residual_vectors(s["x"], s["y"], s["xdot"], s["ydot"], s["xddot"], s["yddot"],
                                      s["psi"], s["xi_x"], s["xi_y"], s["alpha"], s["d"],
                                      s["alpha_a"], s["d_a"], s["v"], 5.6, 3.1)
    assert np.abs(rx - s["ref_r_x"]).max() <= 1e-12 and np.abs(ry - s["ref_r_y"]).max() <= 1e-12


def test_zero_length_fallbacks(cuda):
    from paper_2109_10392_b200 import kernels

    s = golden("tail_case")
    d, d_a, v, r_x, r_y, g_x, g_y, *_ = kernels.tail_core(*_args(s))
    n = s["x"].shape[0]
    mn = s["xi_x"].shape[0]
    # xddot = yddot = 0 at (3, 2): (cos, sin) = (1, 0), d_a = 0 -> g_acc = 0
    assert d_a[3, 2] == 0.0 and g_x[mn + 3, 2] == 0.0 and g_y[mn + 3, 2] == 0.0
    # x == xi at obstacle row 5, column 1: r = 0 -> d = 1, (cos, sin) = (1, 0)
    assert d[5, 1] == 1.0
    assert g_x[5, 1] == s["xi_x"][5] + 5.6 and g_y[5, 1] == s["xi_y"][5]
    del n


def test_torch_in_torch_out(cuda):
    from paper_2109_10392_b200 import kernels

    s = golden("tail_case")
    t = lambda a: cuda.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    v = kernels.v_update(t(s["xdot"]), t(s["ydot"]), 0.1, 20.0)
    assert isinstance(v, cuda.Tensor) and v.is_cuda
    np.testing.assert_array_equal(v.cpu().numpy(), s["ref_v"])
    with pytest.raises(ValueError):
        kernels.set_backend("numpy")
    assert kernels.available_backends() == ("cuda",)


def test_dfma_peak_positive(cuda):
    from paper_2109_10392_b200.device import peak_fp64_tflops

    tf = peak_fp64_tflops(2)
    assert 1.0 < tf < 200.0


def test_device_math(cuda):
    """Branch-free atan2 / sincos / rsqrt / div used inside the AM kernel vs libm
    (numpy): <= 2 ulp, i.e. as good as CUDA's own (also measured here)."""
    import ctypes

    from paper_2109_10392_b200 import _native as nat
    from paper_2109_10392_b200.device import stream_ptr

    rng = np.random.default_rng(3)
    N = 1 << 20
    y = np.concatenate([rng.normal(0, 1, N // 2), rng.normal(0, 30, N // 4),
                        rng.uniform(-1e-3, 1e-3, N // 4)])
    x = np.concatenate([rng.normal(15, 10, N // 2), rng.normal(0, 1e-2, N // 4),
                        rng.uniform(-40, 40, N // 4)])
    y[:6] = [0.0, -0.0, 0.0, -0.0, 1.0, -1.0]
    x[:6] = [0.0, 0.0, -0.0, -0.0, 0.0, -0.0]
    t = lambda a: cuda.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    ty, tx = t(y), t(x)
    out, out2 = cuda.empty_like(ty), cuda.empty_like(ty)
    lib = nat.load()
    sp = ctypes.c_void_p(stream_ptr())

    def run(fn, a, b=None):
        nat.check(lib.bmpc_math_check(fn, a.numel(), a.data_ptr(), b.data_ptr() if b is not None else None,
                                      out.data_ptr(), out2.data_ptr(), sp))
        return out.cpu().numpy().copy(), out2.cpu().numpy().copy()

    def ulps(got, ref):
        return np.abs(got - ref) / np.spacing(np.maximum(np.abs(ref), 1e-300))

    ref = np.arctan2(y, x)
    got, _ = run(0, ty, tx)
    np.testing.assert_array_equal(got[:6], ref[:6])  # signed zeros and axes exactly
    assert ulps(got, ref).max() <= 2.0
    cuda_a, _ = run(1, ty, tx)
    assert ulps(cuda_a, ref).max() <= 2.0
    th = np.concatenate([rng.normal(0, 0.3, N // 2), rng.uniform(-50, 50, N // 2)])
    s, c = run(3, t(th))
    assert ulps(s, np.sin(th)).max() <= 2.0 and ulps(c, np.cos(th)).max() <= 2.0
    r2 = rng.uniform(1e-6, 1e6, N)
    rs, _ = run(2, t(r2))
    assert ulps(rs, 1.0 / np.sqrt(r2)).max() <= 2.0
    q, _ = run(5, t(y), t(x + 50.0))
    assert ulps(q, y / (x + 50.0)).max() <= 1.0
    # the sweep's fast paths are bit-identical to the full functions on their domains
    xo = rng.uniform(1e-3, 40.0, N)
    yo = rng.uniform(-1.0, 1.0, N) * 0.41421356237309503 * xo
    yo[:4] = [0.0, -0.0, 0.41421356237309503 * xo[2], -0.41421356237309503 * xo[3]]
    fast, _ = run(6, t(yo), t(xo))
    full, _ = run(0, t(yo), t(xo))
    np.testing.assert_array_equal(fast.view(np.int64), full.view(np.int64))
    tq = rng.uniform(-0.78, 0.78, N)
    tq[:4] = [0.0, -0.0, 0.78, -0.78]
    fs, fc = run(7, t(tq))
    ns, nc = run(3, t(tq))
    np.testing.assert_array_equal(fs.view(np.int64), ns.view(np.int64))
    np.testing.assert_array_equal(fc.view(np.int64), nc.view(np.int64))


def test_collision_ratios_bitwise(cuda, rng):
    """planner.collision_ratios (its own kernel, bmpc_op_collision_ratios) equals
    the reference's numpy expression (planner.py:219-230) bit for bit, on host
    arrays and device tensors, with non-finite entries and an empty batch."""
    import torch

    from paper_2109_10392_b200.planner import collision_ratios

    n, m, l = 37, 5, 19
    x, y = rng.normal(50, 40, (n, l)), rng.normal(0, 4, (n, l))
    xi_x, xi_y = rng.normal(50, 40, m * n), rng.normal(0, 4, m * n)
    x[3, 2], y[5, 7], xi_x[11] = np.nan, np.inf, 1e4
    xi_x[40:40 + l] = x[40 % n, :l][: min(l, m * n - 40)]  # some exact zeros in wx
    a, b = 5.6, 2.4

    def ref(x, y):
        wx = (np.tile(x, (m, 1)) - xi_x[:, None]) / a
        wy = (np.tile(y, (m, 1)) - xi_y[:, None]) / b
        return np.sqrt(wx * wx + wy * wy)

    with np.errstate(all="ignore"):
        want = ref(x, y)
    got = collision_ratios(x, y, xi_x, xi_y, a, b)
    assert isinstance(got, np.ndarray) and got.shape == (m * n, l)
    np.testing.assert_array_equal(got, want)  # exact on every finite entry, NaN where numpy has NaN
    assert np.isnan(want).any() and np.isinf(want).any()
    dev = collision_ratios(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), xi_x, xi_y, a, b)
    assert dev.is_cuda
    np.testing.assert_array_equal(dev.cpu().numpy(), want)
    assert collision_ratios(x[:, :0], y[:, :0], xi_x, xi_y, a, b).shape == (m * n, 0)
