"""The whole graph stage of one scene as ONE captured CUDA graph (bzg_planner).

``Planner(N, spec, oracle, bounds, obstacles, seed, include)`` fixes the scene's shape -- the
oracle, N, the curve, the sampling bounds, the number of included vertices and of obstacles --
and captures ``build_graph -> cut_graph -> find_path`` (reference graph.py:129-430, in the
order of ``sim.plan_once``).  ``pl(seed, obstacles, start, goal, include=...)`` then returns
what ``find_path(g, cut_graph(g, obstacles), start, goal)`` returns for ``g = build_graph(N,
spec, oracle, bounds, seed, include)``, bit for bit, in one graph launch and one
synchronisation; ``pl.result()`` gives that call's graph and mask.  Calls whose sampler round
falls short, whose edge count outgrows the capacity, whose QP work lists overflow or whose
obstacle list changes shape run eagerly and re-capture (``pl.info()``).

Keep-in regions (BASELINE configs 1 and 5, ``regions.build_region_graph``): pass ``regions``
and ``per_region`` (and optionally the host constants ``rows_added`` / ``sampling`` a caller
keeps); the captured sampler draws every region in one round sized from the measured
acceptance rates.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as nat
from . import graph as G
from .geometry import EPS_GEO


class Planner:
    def __init__(self, N, spec, oracle, bounds, obstacles, seed=0, include=None, cfg=None,
                 position_only_snap: bool = False, require_tube_snap: bool = True, *, ctx=None,
                 regions=None, per_region=None, rows_added=None, sampling=None):
        self._ctx = ctx = ctx or nat.default_context()
        self._spec, self._oracle, self._bounds = spec, oracle, bounds
        self._m = spec.m
        self._R = 0
        rsam = None
        if regions is not None:
            from . import regions as RG

            rr = rows_added or RG.region_rows(oracle, RG.region_oracles(spec, oracle.Xd, oracle.U, oracle.tube,
                                                                        regions))
            smp = sampling or RG.region_sampling(per_region, spec, oracle.Xd, regions, bounds, seed)
            self._R = len(regions)
            N = smp.total
        d, keep, D = G._build_desc(N, spec, oracle, bounds, seed, include)
        if regions is not None:  # the keep-in fields of build_region_graph's descriptor
            off = np.concatenate([[0], np.cumsum([f.shape[0] for f in rr.F])]).astype(np.int32)
            RF = G._f64(np.vstack(rr.F)) if rr.F else np.zeros((0, 2 * spec.n))
            RGv = G._f64(np.concatenate(rr.G)) if rr.G else np.zeros(0)
            blo, bhi = RG.region_boxes(regions)
            keep += [off, RF, RGv, blo, bhi, smp]
            d.n_regions = self._R
            d.region_row_off, d.region_F, d.region_G = nat.ptr(off), nat.ptr(RF), nat.ptr(RGv)
            d.region_box_lo, d.region_box_hi = nat.ptr(blo), nat.ptr(bhi)
            rsam = nat.RegionSampler(self._R, nat.ptr(smp.N), nat.ptr(smp.pcg), nat.ptr(smp.lo), nat.ptr(smp.hi),
                                     nat.ptr(smp.row_off), nat.ptr(smp.A), nat.ptr(smp.b))
            self._pcg_cache = {seed: np.ascontiguousarray(smp.pcg, dtype=np.uint64)}
        self._D = D
        self._n_include = int(d.n_include)
        self._cc = G._cut_cfg(cfg or G.CutConfig())
        tube = oracle.tube.error
        tlo, thi = G._f64(tube.lo), G._f64(tube.hi)
        obstacles = list(obstacles)
        offs, A, b, is_box, lo, hi = G._obstacle_arrays(obstacles, self._m)
        self._n_obs = len(is_box)
        self._h = None
        h = C.c_void_p()
        nat.check(ctx.lib.bzg_planner_create(ctx.handle, C.byref(d), C.byref(rsam) if rsam is not None else None,
                                             self._n_obs, nat.ptr(offs), nat.ptr(A), nat.ptr(b),
                                             nat.ptr(is_box), nat.ptr(lo), nat.ptr(hi), C.byref(self._cc), nat.ptr(tlo),
                                             nat.ptr(thi), EPS_GEO, int(bool(position_only_snap)),
                                             int(bool(require_tube_snap)), C.byref(h)))
        del keep
        self._h = h
        self._V = int(N) + self._n_include
        self._path = np.empty(self._V + 1, dtype=np.int64)
        self._plen = C.c_int64()
        self._dist = C.c_double()
        self._E = C.c_int64()
        self._eager = C.c_int32()
        self._seed = None
        self.counters = np.zeros(6, dtype=np.int64)
        self.last_eager = False
        self.last_dist = None

    @property
    def num_edges(self) -> int:
        return int(self._E.value)

    def _pcg(self, seed):
        if not self._R:
            return np.array(G._pcg_words(seed), dtype=np.uint64)
        hit = self._pcg_cache.get(seed)
        if hit is None:  # default_rng([seed, r]) per region (regions.region_sampling)
            hit = np.array([G._pcg_words([seed, r]) for r in range(self._R)], dtype=np.uint64).reshape(-1)
            if len(self._pcg_cache) > 64:
                self._pcg_cache.clear()
            self._pcg_cache[seed] = hit
        return np.ascontiguousarray(hit, dtype=np.uint64)

    def __call__(self, seed, obstacles, start, goal, include=None):
        pcg = self._pcg(seed)
        inc = None
        if self._n_include:
            if include is None:
                raise ValueError(f"this planner includes {self._n_include} vertices per call")
            inc = G._f64(np.atleast_2d(np.asarray(include, dtype=np.float64)))
            if inc.shape != (self._n_include, self._spec.n):
                raise ValueError(f"include must be ({self._n_include}, {self._spec.n})")
        offs, A, b, is_box, lo, hi = G._obstacle_arrays(list(obstacles), self._m)
        if len(is_box) != self._n_obs:
            raise ValueError(f"a Planner keeps its obstacle count ({self._n_obs})")
        s = np.ascontiguousarray(start, dtype=np.float64)
        g = np.ascontiguousarray(goal, dtype=np.float64)
        nat.check(self._ctx.lib.bzg_planner_run(self._h, nat.ptr(pcg), nat.ptr(inc), self._n_obs, nat.ptr(offs),
                                                nat.ptr(A), nat.ptr(b), nat.ptr(is_box), nat.ptr(lo), nat.ptr(hi),
                                                nat.ptr(s), nat.ptr(g), nat.ptr(self._path), self._path.size,
                                                C.byref(self._plen), C.byref(self._dist), nat.ptr(self.counters),
                                                C.byref(self._E), C.byref(self._eager)))
        self.last_eager = bool(self._eager.value)
        self._seed = seed
        if self._plen.value < 0:
            self.last_dist = None
            return None
        self.last_dist = self._dist.value
        return [int(v) for v in self._path[: self._plen.value]]

    def result(self):
        """(BezierGraph, CutMask) of the last call: device copies owned by the caller."""
        gh, mh = C.c_void_p(), C.c_void_p()
        nat.check(self._ctx.lib.bzg_planner_result(self._h, C.byref(gh), C.byref(mh)))
        graph = G.BezierGraph(gh, self._ctx, self._spec, self._oracle, self._seed, self._bounds, self._D)
        return graph, G.CutMask(mh, graph, self.counters.copy())

    def info(self) -> dict:
        v = np.zeros(6, dtype=np.int64)
        nat.check(self._ctx.lib.bzg_planner_info(self._h, nat.ptr(v)))
        reasons = {0: None, 1: "obstacle-list shape", 2: "sampler round short", 3: "edge capacity", 4: "cut work lists"}
        return {"kernels_per_call": int(v[0]), "calls": int(v[1]), "eager_calls": int(v[2]), "captures": int(v[3]),
                "edge_capacity": int(v[4]), "last_eager_reason": reasons.get(int(v[5]))}

    def close(self):
        if getattr(self, "_h", None):
            self._ctx.lib.bzg_planner_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
