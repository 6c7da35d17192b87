"""Operator-level kernels: the reference's ``batchmpc.kernels`` plugin API
(/root/reference/pkg/src/batchmpc/kernels/__init__.py:49-86) on sm_100a.

Same function names, argument order and return tuples as the reference.
Arguments may be numpy arrays (results come back as numpy) or CUDA float64
torch tensors (results stay on the device).  There is exactly one back-end,
"cuda"; asking for any other raises ValueError like the reference's registry.
"""

from __future__ import annotations

import ctypes
from contextlib import contextmanager

import numpy as np

from . import _native as nat

_BACKENDS = ("cuda",)
_active = "cuda"


def active_backend() -> str:
    return _active


def available_backends() -> tuple[str, ...]:
    return _BACKENDS


def set_backend(name: str) -> None:
    if name not in _BACKENDS:
        raise ValueError(f"unknown backend {name!r}; available: {sorted(_BACKENDS)}")


@contextmanager
def use_backend(name: str):
    set_backend(name)
    yield


class _Args:
    """Uploads numpy inputs, tracks whether to return numpy."""

    def __init__(self):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("batchmpc-b200 kernels need a CUDA device; there is no CPU fallback")
        self.torch = torch
        self.host = False
        self.dev = None

    def __call__(self, a):
        torch = self.torch
        if isinstance(a, torch.Tensor):
            if not a.is_cuda or a.dtype != torch.float64:
                raise ValueError("tensor arguments must be CUDA float64")
            self.dev = a.device
            return a.contiguous()
        self.host = True
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
        return t.to(self.dev or torch.device("cuda", torch.cuda.current_device()))

    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64,
                                device=self.dev or self.torch.device("cuda", self.torch.cuda.current_device()))

    def out(self, *ts):
        if self.host:
            res = tuple(t.cpu().numpy() for t in ts)
        else:
            res = ts
        return res if len(res) > 1 else res[0]


def _s():
    from .device import stream_ptr

    return ctypes.c_void_p(stream_ptr())


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def obstacle_update(x, y, xi_x, xi_y, a, b):
    """alpha = atan2(a wy, b wx), d = max(1, ...) (_speedups.pyx:12-39)."""
    A = _Args()
    x, y, xi_x, xi_y = A(x), A(y), A(xi_x), A(xi_y)
    n, l = x.shape
    mn = xi_x.shape[0]
    alpha, d = A.empty(mn, l), A.empty(mn, l)
    nat.check(nat.load().bmpc_op_obstacle_update(n, l, mn, _p(x), _p(y), _p(xi_x), _p(xi_y),
                                                 float(a), float(b), _p(alpha), _p(d), _s()),
              "obstacle_update")
    return A.out(alpha, d)


def accel_update(xddot, yddot, a_max):
    A = _Args()
    xdd, ydd = A(xddot), A(yddot)
    n, l = xdd.shape
    al, da = A.empty(n, l), A.empty(n, l)
    nat.check(nat.load().bmpc_op_accel_update(n, l, _p(xdd), _p(ydd), float(a_max), _p(al), _p(da),
                                              _s()), "accel_update")
    return A.out(al, da)


def v_update(xdot, ydot, v_min, v_max):
    A = _Args()
    xd, yd = A(xdot), A(ydot)
    n, l = xd.shape
    v = A.empty(n, l)
    nat.check(nat.load().bmpc_op_v_update(n, l, _p(xd), _p(yd), float(v_min), float(v_max), _p(v),
                                          _s()), "v_update")
    return A.out(v)


def assemble_g(xi_x, xi_y, alpha, d, alpha_a, d_a, v, psi, a, b):
    A = _Args()
    ts = [A(t) for t in (xi_x, xi_y, alpha, d, alpha_a, d_a, v, psi)]
    mn, l = ts[2].shape
    n = ts[6].shape[0]
    g_x, g_y = A.empty(mn + 2 * n, l), A.empty(mn + 2 * n, l)
    nat.check(nat.load().bmpc_op_assemble_g(n, l, mn, *[_p(t) for t in ts], float(a), float(b),
                                            _p(g_x), _p(g_y), _s()), "assemble_g")
    return A.out(g_x, g_y)


def residual_vectors(x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, alpha, d, alpha_a, d_a, v,
                     a, b):
    A = _Args()
    ts = [A(t) for t in (x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, alpha, d, alpha_a, d_a, v)]
    mn = ts[9].shape[0]
    n, l = ts[0].shape
    r_x, r_y = A.empty(mn + 2 * n, l), A.empty(mn + 2 * n, l)
    nat.check(nat.load().bmpc_op_residual_vectors(n, l, mn, *[_p(t) for t in ts], float(a), float(b),
                                                  _p(r_x), _p(r_y), _s()), "residual_vectors")
    return A.out(r_x, r_y)


def _tail(with_angles, x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, v_min, v_max, a_max, a, b):
    A = _Args()
    ts = [A(t) for t in (x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y)]
    n, l = ts[0].shape
    mn = ts[7].shape[0]
    rows = mn + 2 * n
    alpha = A.empty(mn, l) if with_angles else None
    alpha_a = A.empty(n, l) if with_angles else None
    d, d_a, v = A.empty(mn, l), A.empty(n, l), A.empty(n, l)
    r_x, r_y, g_x, g_y = (A.empty(rows, l) for _ in range(4))
    sq = [None] * 3 if with_angles else [A.empty(l) for _ in range(3)]
    P = lambda t: None if t is None else _p(t)  # noqa: E731
    nat.check(nat.load().bmpc_op_tail(n, l, mn, *[_p(t) for t in ts], float(v_min), float(v_max),
                                      float(a_max), float(a), float(b), P(alpha), _p(d), P(alpha_a),
                                      _p(d_a), _p(v), _p(r_x), _p(r_y), _p(g_x), _p(g_y),
                                      *[P(s) for s in sq], _s()), "tail")
    if with_angles:
        return A.out(alpha, d, alpha_a, d_a, v, r_x, r_y, g_x, g_y)
    return A.out(d, d_a, v, r_x, r_y, g_x, g_y, *sq)


def tail_update(x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, v_min, v_max, a_max, a, b):
    """(alpha, d, alpha_a, d_a, v, r_x, r_y, g_x, g_y) (_speedups.pyx:221-318)."""
    return _tail(True, x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, v_min, v_max, a_max, a, b)


def tail_core(x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, v_min, v_max, a_max, a, b):
    """(d, d_a, v, r_x, r_y, g_x, g_y, sq_obs, sq_acc, sq_nonhol) (_speedups.pyx:114-218)."""
    return _tail(False, x, y, xdot, ydot, xddot, yddot, psi, xi_x, xi_y, v_min, v_max, a_max, a, b)
