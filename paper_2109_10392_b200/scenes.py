"""Seeded synthetic workloads for the BASELINE configs c0-c4.

The reference publishes no dataset for this path (its NGSIM scenes are out of
scope), so the configs are generated from numpy
``default_rng(seed)`` streams with the shapes and value distributions
BASELINE.json names.  The choices BASELINE.json leaves open are frozen here
once:

* road: 4 lanes, centres y in {-5.25, -1.75, 1.75, 5.25}; ellipse a=5.6, b=2.4
* ego: x=0, lane ~ integers(4), v0 ~ U(15, 25), heading 0, accel 0
* obstacles: constant velocity along x in a random lane, drawn with the
  reference harness's spawn-rejection rule (harness.py:268-285: no spawn within
  2.5a of the ego in its lane, ego-relative ellipse ratio >= 1.5, same-lane
  spacing >= 3a; up to 100 attempts, a vehicle that never fits is dropped),
  ordered nearest-first and padded with far virtual obstacles exactly as
  traffic.select_nearest does (traffic.py:199-213)
* predictions: traffic.predict_constant_velocity layout, row j*n + k
  (traffic.py:216-233)
* goals: b_xy = [0, v0, 0, v_g*t_f, v_g, 0, y_ego, 0, 0, y_g, 0, 0], b_psi = 0
  (the "distance v*t_f" rule of planner.py:106,121; rows per planner.py:339-346)
* solver scalars: rho=1, v_min=0.1, v_max=35 (goal speeds reach 30 m/s), a_max=8
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

LANES = np.array([-5.25, -1.75, 1.75, 5.25])
ELLIPSE_A = 5.6
ELLIPSE_B = 2.4


@dataclass(frozen=True)
class WorkloadConfig:
    name: str
    n: int
    t_f: float
    degree: int
    m: int
    l: int
    scenes: int
    iters: int
    x_range: tuple[float, float]
    v_range: tuple[float, float]
    goals: str  # "grid" (11 lateral x 10 speeds) or "uniform"
    seed0: int = 0

    @property
    def n_b(self) -> int:
        return self.degree + 1

    @property
    def problems(self) -> int:
        return self.l * self.scenes


CONFIGS = {
    "c0": WorkloadConfig("c0", 100, 5.0, 10, 10, 110, 1, 100, (-30.0, 120.0), (10.0, 25.0), "grid"),
    "c1": WorkloadConfig("c1", 100, 5.0, 10, 10, 1024, 1, 100, (-30.0, 120.0), (10.0, 25.0), "uniform"),
    "c2": WorkloadConfig("c2", 100, 5.0, 10, 30, 16384, 1, 200, (-50.0, 200.0), (8.0, 28.0), "uniform"),
    "c3": WorkloadConfig("c3", 100, 5.0, 10, 20, 1024, 128, 100, (-30.0, 120.0), (10.0, 25.0), "uniform"),
    "c4": WorkloadConfig("c4", 200, 10.0, 15, 50, 1024, 1024, 100, (-50.0, 250.0), (8.0, 28.0), "uniform"),
}


@dataclass
class SceneBatch:
    """S independent scenes x l goals, stacked column-wise (instance = s*l + i).

    xi_x, xi_y: (S, m*n) obstacle predictions; b_xy: (12, S*l); b_psi: (4, S*l).
    """

    n: int
    t_f: float
    degree: int
    m: int
    l: int
    S: int
    xi_x: np.ndarray
    xi_y: np.ndarray
    b_xy: np.ndarray
    b_psi: np.ndarray
    a: float = ELLIPSE_A
    b: float = ELLIPSE_B
    v_min: float = 0.1
    v_max: float = 35.0
    a_max: float = 8.0
    rho: float = 1.0
    ego: list = field(default_factory=list)

    @property
    def L(self) -> int:
        return self.S * self.l

    def scene(self, s: int) -> "SceneBatch":
        cols = slice(s * self.l, (s + 1) * self.l)
        return SceneBatch(self.n, self.t_f, self.degree, self.m, self.l, 1,
                          self.xi_x[s : s + 1], self.xi_y[s : s + 1],
                          np.ascontiguousarray(self.b_xy[:, cols]),
                          np.ascontiguousarray(self.b_psi[:, cols]),
                          self.a, self.b, self.v_min, self.v_max, self.a_max, self.rho,
                          self.ego[s : s + 1])

    def columns(self, lo: int, hi: int) -> "SceneBatch":
        """Goal-column slice of a single-scene batch (multi-GPU sharding of c1/c2)."""
        assert self.S == 1
        return SceneBatch(self.n, self.t_f, self.degree, self.m, hi - lo, 1, self.xi_x, self.xi_y,
                          np.ascontiguousarray(self.b_xy[:, lo:hi]),
                          np.ascontiguousarray(self.b_psi[:, lo:hi]),
                          self.a, self.b, self.v_min, self.v_max, self.a_max, self.rho, self.ego)

    def scenes(self, lo: int, hi: int) -> "SceneBatch":
        cols = slice(lo * self.l, hi * self.l)
        return SceneBatch(self.n, self.t_f, self.degree, self.m, self.l, hi - lo,
                          self.xi_x[lo:hi], self.xi_y[lo:hi],
                          np.ascontiguousarray(self.b_xy[:, cols]),
                          np.ascontiguousarray(self.b_psi[:, cols]),
                          self.a, self.b, self.v_min, self.v_max, self.a_max, self.rho,
                          self.ego[lo:hi])


def _spawn_obstacles(rng, m, x_range, v_range, ego_lane, a, b):
    """harness.py:268-285 rejection rule; returns list of (x, y, vx, vy, lane)."""
    ego_x, ego_y = 0.0, LANES[ego_lane]
    placed = []
    for _ in range(m):
        for _attempt in range(100):
            lane = int(rng.integers(0, len(LANES)))
            x = float(rng.uniform(*x_range))
            v0 = float(rng.uniform(*v_range))
            if abs(x - ego_x) < 2.5 * a and lane == ego_lane:
                continue
            if math.hypot((x - ego_x) / a, (LANES[lane] - ego_y) / b) < 1.5:
                continue
            if any(o[4] == lane and abs(o[0] - x) < 3.0 * a for o in placed):
                continue
            placed.append((x, float(LANES[lane]), v0, 0.0, lane))
            break
    # select_nearest: m nearest, padded with virtual obstacles at +1e4 m
    placed.sort(key=lambda o: (o[0] - ego_x) ** 2 + (o[1] - ego_y) ** 2)
    while len(placed) < m:
        placed.append((ego_x + 1.0e4, ego_y + 1.0e4, 0.0, 0.0, 0))
    return placed[:m]


def predict_constant_velocity(obstacles, times: np.ndarray):
    """Flat (m*n,) predictions, entry j*n + k = obstacle j at sample k (traffic.py:216-233)."""
    rel = np.asarray(times, dtype=float)
    rel = rel - rel[0]
    n = rel.shape[0]
    xi_x = np.empty(len(obstacles) * n)
    xi_y = np.empty(len(obstacles) * n)
    for j, o in enumerate(obstacles):
        xi_x[j * n : (j + 1) * n] = o[0] + o[2] * rel
        xi_y[j * n : (j + 1) * n] = o[1] + o[3] * rel
    return xi_x, xi_y


def make_scene(cfg: WorkloadConfig, seed: int, l: int | None = None):
    """One scene: (xi_x, xi_y, b_xy, b_psi, ego dict)."""
    l = cfg.l if l is None else l
    rng = np.random.default_rng(seed)
    ego_lane = int(rng.integers(0, len(LANES)))
    v0 = float(rng.uniform(15.0, 25.0))
    y_ego = float(LANES[ego_lane])
    obstacles = _spawn_obstacles(rng, cfg.m, cfg.x_range, cfg.v_range, ego_lane, ELLIPSE_A, ELLIPSE_B)
    times = np.linspace(0.0, cfg.t_f, cfg.n)
    xi_x, xi_y = predict_constant_velocity(obstacles, times)
    if cfg.goals == "grid":
        ys, vs = np.meshgrid(np.linspace(-5.25, 5.25, 11), np.linspace(10.0, 30.0, 10), indexing="ij")
        y_g, v_g = ys.ravel(), vs.ravel()
        if l != y_g.size:
            reps = int(math.ceil(l / y_g.size))
            y_g, v_g = np.tile(y_g, reps)[:l], np.tile(v_g, reps)[:l]
    else:
        y_g = rng.uniform(-5.25, 5.25, l)
        v_g = rng.uniform(10.0, 30.0, l)
    b_xy = np.zeros((12, l))
    b_xy[1] = v0
    b_xy[3] = v_g * cfg.t_f
    b_xy[4] = v_g
    b_xy[6] = y_ego
    b_xy[9] = y_g
    b_psi = np.zeros((4, l))
    ego = dict(x=0.0, y=y_ego, vx=v0, vy=0.0, lane=ego_lane, obstacles=obstacles)
    return xi_x, xi_y, b_xy, b_psi, ego


def make_workload(name_or_cfg, scenes: int | None = None, l: int | None = None,
                  seed0: int | None = None) -> SceneBatch:
    """Stacked SceneBatch for a config; ``scenes``/``l`` override for bounded samples."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    S = cfg.scenes if scenes is None else scenes
    l = cfg.l if l is None else l
    s0 = cfg.seed0 if seed0 is None else seed0
    mn = cfg.m * cfg.n
    xi_x = np.empty((S, mn))
    xi_y = np.empty((S, mn))
    b_xy = np.empty((12, S * l))
    b_psi = np.empty((4, S * l))
    egos = []
    for s in range(S):
        sx, sy, bx, bp, ego = make_scene(cfg, s0 + s, l)
        xi_x[s], xi_y[s] = sx, sy
        b_xy[:, s * l : (s + 1) * l] = bx
        b_psi[:, s * l : (s + 1) * l] = bp
        egos.append(ego)
    return SceneBatch(cfg.n, cfg.t_f, cfg.degree, cfg.m, l, S, xi_x, xi_y, b_xy, b_psi, ego=egos)
