"""Device helpers of the replanning loop around the graph stage.

``project_on_path`` replaces the reference simulator's ``_project_on_path`` (sim.py:220-239):
the grid time along the path's Bézier chain positionally closest to the vehicle state, which
anchors the receding MPC reference window.  The reference evaluates up to (hops x T/h) points
with a Python loop over de Casteljau per replanning cycle; here one kernel evaluates them all
(bzg_project_on_path) with the reference's arithmetic, so the anchor is the same float.
``shim.install`` patches it into ``beziergraph.sim``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from .bezier import boundary_matrix


def project_on_path(path_states, spec, h: float, state, *, ctx=None) -> float:
    """Grid time tau = k*h of the path's curve chain closest (in position) to ``state``."""
    ctx = ctx or nat.default_context()
    P = np.ascontiguousarray(np.atleast_2d(np.asarray(path_states, dtype=np.float64)))
    x = np.ascontiguousarray(np.asarray(state, dtype=np.float64))
    m, g = int(spec.m), int(spec.gamma)
    if P.shape[0] and P.shape[1] != m * g:
        raise ValueError(f"path states must have dimension {m * g}")
    spt = int(round(spec.T / h))  # sim.py:231
    D = np.ascontiguousarray(boundary_matrix(spec), dtype=np.float64)
    out = C.c_double()
    nat.check(ctx.lib.bzg_project_on_path(ctx.handle, m, g, float(spec.T), nat.ptr(D), P.shape[0], nat.ptr(P),
                                          float(h), spt, nat.ptr(x), C.byref(out)))
    return out.value
