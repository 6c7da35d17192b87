"""Device-resident solve / score on torch-allocated HBM buffers.

torch is plumbing here (allocation, streams, pinned host memory); all compute
runs in the sm_100a kernels behind the C ABI (include/batchmpc_b200.h).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat


_CUDA_OK = False


def _torch():
    global _CUDA_OK
    import torch

    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2109_10392_b200 needs a CUDA device (sm_100a); no CPU fallback")
        _CUDA_OK = True
    return torch


def stream_ptr(stream=None) -> int:
    torch = _torch()
    if stream is not None:
        return stream.cuda_stream
    # torch's current stream on the current device, without building a Stream object
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


@dataclass
class DeviceProblem:
    """Stacked scenes on the device: instance s*l + i is goal i of scene s."""

    m: int
    l: int
    S: int
    xi_x: "object"   # torch (S, m*n) float64
    xi_y: "object"
    b_xy: "object"   # (12, L)
    b_psi: "object"  # (4, L)
    a: float
    b: float
    v_min: float
    v_max: float
    a_max: float

    @property
    def L(self) -> int:
        return self.S * self.l

    def c_struct(self) -> nat.Problem:
        return nat.Problem(self.m, self.l, self.S, ptr(self.xi_x), ptr(self.xi_y), ptr(self.b_xy),
                           ptr(self.b_psi), self.a, self.b, self.v_min, self.v_max, self.a_max)

    @staticmethod
    def from_host(n, xi_x, xi_y, b_xy, b_psi, l, a, b, v_min, v_max, a_max, device=None,
                  non_blocking=False) -> "DeviceProblem":
        torch = _torch()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        xi_x = np.atleast_2d(np.asarray(xi_x, dtype=np.float64))
        xi_y = np.atleast_2d(np.asarray(xi_y, dtype=np.float64))
        S = xi_x.shape[0]
        mn = xi_x.shape[1]

        def up(a):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
            if non_blocking:
                t = t.pin_memory()
            return t.to(dev, non_blocking=non_blocking)

        if mn % n:
            raise ValueError(f"obstacle predictions of length {mn} are not a multiple of n={n}")
        b_xy = np.asarray(b_xy, dtype=np.float64)
        b_psi = np.asarray(b_psi, dtype=np.float64)
        parts = (xi_x, xi_y, b_xy, b_psi)
        if not non_blocking and sum(p.size for p in parts) <= (1 << 19):
            # small problems (planner-sized batches): one packed copy instead of
            # four, each part a 16-byte aligned view of the device block
            offs, tot = [], 0
            for p in parts:
                offs.append(tot)
                tot += (p.size + 1) & ~1
            host = np.empty(tot)
            for p, o in zip(parts, offs):
                host[o:o + p.size] = p.reshape(-1)
            blk = torch.from_numpy(host).to(dev)
            v = [blk[o:o + p.size].view(p.shape) for p, o in zip(parts, offs)]
            return DeviceProblem(m=mn // n, l=int(l), S=S, xi_x=v[0], xi_y=v[1], b_xy=v[2], b_psi=v[3],
                                 a=float(a), b=float(b), v_min=float(v_min), v_max=float(v_max),
                                 a_max=float(a_max))
        return DeviceProblem(m=mn // n, l=int(l), S=S, xi_x=up(xi_x), xi_y=up(xi_y),
                             b_xy=up(b_xy), b_psi=up(b_psi), a=float(a), b=float(b),
                             v_min=float(v_min), v_max=float(v_max), a_max=float(a_max))


@dataclass
class DeviceSolution:
    c_x: "object"
    c_y: "object"
    c_psi: "object"
    l_x: "object"
    l_y: "object"
    l_psi: "object"
    history: "object"    # (max_iter, 3, L); rows >= iterations are stale
    res_final: "object"  # (3, L)
    v: "object"          # (n, L) or None
    iterations: int
    converged: bool
    coef: "object" = None  # (6, nb, L): c_x, c_y, c_psi, l_x, l_y, l_psi are its rows
    block: "object" = None  # (6 nb + 3, L): coef then res_final, one allocation (one copy back)


@dataclass
class DeviceScore:
    meta_cost: "object"
    min_ratio: "object"
    heading_max: "object"
    flags: "object"       # uint8: bit0 heading, bit1 residual, bit2 collision
    best_index: "object"  # (S,) int64, -1 = None
    argmin_all: "object"
    argmin_hc: "object"
    n_feasible: "object"


def alloc_solution(nb: int, n: int, L: int, max_iter: int, want_v: bool, device) -> DeviceSolution:
    torch = _torch()
    z = lambda *s: torch.empty(*s, dtype=torch.float64, device=device)  # noqa: E731
    block = z(6 * nb + 3, L)
    coef = block[: 6 * nb].view(6, nb, L)
    return DeviceSolution(coef[0], coef[1], coef[2], coef[3], coef[4], coef[5],
                          z(max_iter, 3, L), block[6 * nb:], z(n, L) if want_v else None, 0, False, coef,
                          block)


def solution_struct(sol: DeviceSolution) -> nat.SolveOut:
    return nat.SolveOut(ptr(sol.c_x), ptr(sol.c_y), ptr(sol.c_psi), ptr(sol.l_x), ptr(sol.l_y),
                        ptr(sol.l_psi), ptr(sol.v), ptr(sol.history), ptr(sol.res_final), 0, 0)


def alloc_score(L: int, S: int, device) -> DeviceScore:
    torch = _torch()
    f = lambda: torch.empty(L, dtype=torch.float64, device=device)  # noqa: E731
    i = lambda: torch.empty(S, dtype=torch.int64, device=device)  # noqa: E731
    return DeviceScore(f(), f(), f(), torch.empty(L, dtype=torch.uint8, device=device),
                       i(), i(), i(), i())


def score_struct(sc: DeviceScore) -> nat.ScoreOut:
    return nat.ScoreOut(ptr(sc.meta_cost), ptr(sc.min_ratio), ptr(sc.heading_max), ptr(sc.flags),
                        ptr(sc.best_index), ptr(sc.argmin_all), ptr(sc.argmin_hc),
                        ptr(sc.n_feasible))


def peak_fp64_tflops(reps: int = 5) -> float:
    """Measured DFMA throughput of the current device (the FP64-pipe roofline)."""
    _torch()
    out = ctypes.c_double(0.0)
    nat.check(nat.load().bmpc_dfma_peak(reps, ctypes.byref(out), ctypes.c_void_p(stream_ptr())),
              "dfma_peak")
    return out.value


def assemble_scenes(solver, egos, vehicles, goals, m: int, a: float, b: float, v_min: float,
                    v_max: float, a_max: float, device=None, stream=None) -> DeviceProblem:
    """build_batch for S scenes on the device (`bmpc_assemble`): the m nearest
    vehicles of each scene, their constant-velocity predictions and the
    boundary vectors of its goals (planner.py:336-360, traffic.py:199-233).

    egos: S EgoState; vehicles: S lists of VehicleState; goals: S lists of
    Goal (the same count l each).  Host data is packed into small state
    arrays -- (S, V, 4) vehicles, (S, 8) egos, (S*l, 6) goals -- instead of the
    (S, m*n) prediction tables, which are built on the device."""
    torch = _torch()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    S = len(egos)
    if len(vehicles) != S or len(goals) != S:
        raise ValueError("one vehicle list and one goal list per ego state")
    l = len(goals[0]) if S else 0
    if any(len(g) != l for g in goals):
        raise ValueError("every scene needs the same number of goals")
    V = max([len(v) for v in vehicles] + [1])
    veh = np.zeros((S, V, 4))
    nveh = np.array([len(v) for v in vehicles], dtype=np.int32)
    for s, vs in enumerate(vehicles):
        for i, v in enumerate(vs):
            veh[s, i] = (v.x, v.y, v.vx, v.vy)
    ego = np.array([[e.x, e.vx, e.ax, e.y, e.vy, e.ay, e.psi, e.psidot] for e in egos],
                   dtype=np.float64).reshape(S, 8)
    gl = np.array([[g.x, g.vx, g.ax, g.y, g.vy, g.ay] for gs in goals for g in gs],
                  dtype=np.float64).reshape(S * l, 6)
    times = np.asarray(solver.basis.grid.times, dtype=np.float64)
    rel = times - times[0]
    n = times.shape[0]
    up = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)  # noqa: E731
    d_veh, d_nveh, d_ego, d_goals, d_rel = up(veh), up(nveh), up(ego), up(gl), up(rel)
    f64 = lambda *shape: torch.empty(*shape, dtype=torch.float64, device=dev)  # noqa: E731
    xi_x, xi_y = f64(S, m * n), f64(S, m * n)
    b_xy, b_psi = f64(12, S * l), f64(4, S * l)
    nat.check(nat.load().bmpc_assemble(solver._context(), S, V, m, l, ptr(d_veh), ptr(d_nveh),
                                       ptr(d_ego), ptr(d_goals), ptr(d_rel), ptr(xi_x), ptr(xi_y),
                                       ptr(b_xy), ptr(b_psi), ctypes.c_void_p(stream_ptr(stream))),
              "assemble")
    return DeviceProblem(m=m, l=l, S=S, xi_x=xi_x, xi_y=xi_y, b_xy=b_xy, b_psi=b_psi, a=float(a),
                         b=float(b), v_min=float(v_min), v_max=float(v_max), a_max=float(a_max))
