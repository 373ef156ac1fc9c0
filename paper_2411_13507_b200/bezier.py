"""Bezier constants for the device graph stage (host side).

Mirrors the curve-family descriptor ``BezierSpec`` and the two constant
matrices the hot path needs (reference bezier.py:22-44, 161-211):

* ``derivative_matrix`` H — degree-preserving derivative operator, used to
  build the reachability oracle's endpoint maps;
* ``boundary_matrix`` D = inv(M) — per-dimension map from the 2*gamma
  boundary values of an edge to its p+1 output control points.

D comes from LAPACK and carries residues such as D[0,1] = -1.85e-17 at T=1
(SURVEY.md §0 finding 2); it is always computed here on the host with the
same numpy calls and uploaded, never re-derived in closed form on device.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from functools import lru_cache

import numpy as np


@dataclass(frozen=True)
class BezierSpec:
    """m output dims, chain length gamma, degree p (default 2*gamma-1), duration T."""

    m: int
    gamma: int
    T: float
    p: int = -1

    def __post_init__(self):
        if self.p < 0:
            object.__setattr__(self, "p", 2 * self.gamma - 1)
        if self.gamma < 1 or self.p < self.gamma:
            raise ValueError("require p >= gamma >= 1")
        if self.T <= 0:
            raise ValueError("segment duration must be positive")

    @property
    def n(self) -> int:
        return self.m * self.gamma

    def with_duration(self, T: float) -> "BezierSpec":
        return replace(self, T=T)


@lru_cache(maxsize=256)
def _h_matrix(p: int, T: float) -> np.ndarray:
    # finite difference to degree p-1 (scaled by p/T) then elevation back to p
    down = np.zeros((p + 1, p))
    for j in range(p):
        down[j, j] = -p / T
        down[j + 1, j] = p / T
    up = np.zeros((p, p + 1))
    for k in range(p + 1):
        if k >= 1:
            up[k - 1, k] += k / p
        if k <= p - 1:
            up[k, k] += (p - k) / p
    H = down @ up
    H.setflags(write=False)
    return H


def derivative_matrix(spec) -> np.ndarray:
    return _h_matrix(spec.p, spec.T)


@lru_cache(maxsize=256)
def _d_matrix(p: int, gamma: int, T: float) -> np.ndarray:
    H = _h_matrix(p, T)
    M = np.zeros((2 * gamma, p + 1))
    Hk = np.eye(p + 1)
    for k in range(gamma):
        M[k] = Hk[:, 0]
        M[gamma + k] = Hk[:, p]
        Hk = Hk @ H
    D = np.linalg.inv(M)
    D.setflags(write=False)
    return D


def boundary_matrix(spec) -> np.ndarray:
    if spec.p != 2 * spec.gamma - 1:
        raise ValueError("boundary-value curves require p = 2*gamma - 1")
    return _d_matrix(spec.p, spec.gamma, spec.T)
