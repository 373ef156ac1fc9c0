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


class Replanner:
    """One replanning cycle of ``sim.run_closed_loop`` -- the cut with the obstacles where they
    are now (sim.py:324-330 re-cuts through ``ObstacleTrack.at``) and ``graph.find_path`` from the
    vehicle state (graph.py:302-430) -- on a fixed graph, as ONE captured CUDA graph
    (bzg_replanner).  ``rp(obstacles, start, goal)`` returns the path ``find_path(graph,
    cut_graph(graph, obstacles), start, goal, ...)`` returns, bit for bit; ``rp.mask()`` is that
    cut's CutMask.  Creating it runs the first cycle (with ``obstacles``) eagerly and captures.
    The obstacle list keeps its length; a cycle whose list changed shape (row counts, box or
    general kinds) or outgrew a work list runs eagerly and is re-captured (``eager_cycles``).

    ``dynamic`` (one flag per obstacle, default all): the obstacles flagged False are static --
    cut once, their per-obstacle outcome rows kept on the device -- and a cycle cuts only the
    dynamic ones (the ones ``ObstacleTrack.at`` moves) and rebuilds the mask in list order."""

    def __init__(self, graph, obstacles, cfg=None, position_only_snap: bool = False, require_tube_snap: bool = True,
                 dynamic=None):
        from .graph import CutConfig, _cut_cfg, _f64, _obstacle_arrays
        from .geometry import EPS_GEO

        self._graph = graph
        self._ctx = ctx = graph._ctx
        self._h = None
        self._m = graph.spec.m
        self._arrays = _obstacle_arrays
        self._cc = _cut_cfg(cfg or CutConfig())
        tube = graph.oracle.tube.error
        tlo, thi = _f64(tube.lo), _f64(tube.hi)
        obstacles = list(obstacles)
        offs, A, b, is_box, lo, hi = _obstacle_arrays(obstacles, self._m)
        self._n_obs = len(is_box)
        dyn = None
        self._dyn_idx = None
        if dynamic is not None:
            dyn = np.ascontiguousarray(np.asarray(dynamic, dtype=bool).astype(np.uint8))
            if dyn.shape != (self._n_obs,):
                raise ValueError("dynamic needs one flag per obstacle")
            if not dyn.all():
                self._dyn_idx = [int(i) for i in np.nonzero(dyn)[0]]
        self._static = [ob for i, ob in enumerate(obstacles) if dyn is not None and not dyn[i]]
        h = C.c_void_p()
        nat.check(ctx.lib.bzg_replanner_create(ctx.handle, graph._h, self._n_obs, nat.ptr(offs), nat.ptr(A), nat.ptr(b),
                                               nat.ptr(is_box), nat.ptr(lo), nat.ptr(hi), nat.ptr(dyn),
                                               C.byref(self._cc),
                                               nat.ptr(tlo), nat.ptr(thi), EPS_GEO, int(bool(position_only_snap)),
                                               int(bool(require_tube_snap)), C.byref(h)))
        self._h = h
        self._dyn_set = set(self._dyn_idx or [])
        self._path = np.empty(graph.num_vertices + 1, dtype=np.int64)
        self._plen = C.c_int64()
        self._dist = C.c_double()
        self._eager = C.c_int32()
        self.counters = np.zeros(6, dtype=np.int64)
        self.last_eager = False

    def __call__(self, obstacles, start, goal):
        obstacles = list(obstacles)
        if len(obstacles) != self._n_obs:
            raise ValueError(f"a Replanner keeps its obstacle count ({self._n_obs})")
        lst, n = obstacles, self._n_obs
        if self._dyn_idx is not None:
            static = [ob for i, ob in enumerate(obstacles) if i not in self._dyn_set]
            if all(a is b for a, b in zip(static, self._static)):  # unchanged: pass the dynamic ones alone
                lst = [obstacles[i] for i in self._dyn_idx]
                n = len(lst)
            else:
                self._static = static
        offs, A, b, is_box, lo, hi = self._arrays(lst, self._m)
        s = np.ascontiguousarray(start, dtype=np.float64)
        g = np.ascontiguousarray(goal, dtype=np.float64)
        nat.check(self._ctx.lib.bzg_replanner_run(self._h, n, nat.ptr(offs), nat.ptr(A), nat.ptr(b),
                                                  nat.ptr(is_box), nat.ptr(lo), nat.ptr(hi), nat.ptr(s), nat.ptr(g),
                                                  nat.ptr(self._path), self._path.size, C.byref(self._plen),
                                                  C.byref(self._dist), nat.ptr(self.counters), C.byref(self._eager)))
        self.last_eager = bool(self._eager.value)
        if self._plen.value < 0:
            return None
        out = [int(v) for v in self._path[: self._plen.value]]
        self._graph._cache["last_dist"] = (tuple(out), self._dist.value)
        return out

    def mask(self):
        """The last cycle's cut as a CutMask (a device copy owned by the caller)."""
        from .graph import CutMask

        h = C.c_void_p()
        nat.check(self._ctx.lib.bzg_replanner_mask(self._h, C.byref(h)))
        return CutMask(h, self._graph, self.counters.copy())

    def info(self) -> dict:
        v = np.zeros(4, dtype=np.int64)
        nat.check(self._ctx.lib.bzg_replanner_info(self._h, nat.ptr(v)))
        return {"kernels_per_cycle": int(v[0]), "cycles": int(v[1]), "eager_cycles": int(v[2]), "captures": int(v[3])}

    def close(self):
        if getattr(self, "_h", None):
            self._ctx.lib.bzg_replanner_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
