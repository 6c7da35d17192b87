"""Obstacle selection and prediction layout (reference traffic.py:199-233).

Only the pieces that define the solver's ``xi_x/xi_y`` input live here; the
closed-loop traffic simulation of the reference is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class VehicleState:
    id: int
    x: float
    y: float
    vx: float
    vy: float
    lane: int


def select_nearest(states: list[VehicleState], ego_x: float, ego_y: float, m: int
                   ) -> list[VehicleState]:
    """The m nearest vehicles, padded with virtual ones 1e4 m away so matrix
    shapes never change (traffic.py:199-213)."""
    picked = sorted(states, key=lambda s: (s.x - ego_x) ** 2 + (s.y - ego_y) ** 2)[:m]
    pad = VehicleState(id=-1, x=ego_x + 1.0e4, y=ego_y + 1.0e4, vx=0.0, vy=0.0, lane=0)
    return picked + [pad] * (m - len(picked))


def predict_constant_velocity(states: list[VehicleState], times: np.ndarray
                              ) -> tuple[np.ndarray, np.ndarray]:
    """Flat predictions, entry j*n + k = obstacle j at sample k (traffic.py:216-233)."""
    rel = np.asarray(times, dtype=float)
    rel = rel - rel[0]
    n = rel.shape[0]
    xi_x = np.empty(len(states) * n)
    xi_y = np.empty(len(states) * n)
    for j, s in enumerate(states):
        xi_x[j * n:(j + 1) * n] = s.x + s.vx * rel
        xi_y[j * n:(j + 1) * n] = s.y + s.vy * rel
    return xi_x, xi_y
