"""Drop-in device implementation of the reference graph stage.

Same names, signatures, return types and error behaviour as
``beziergraph.graph`` (/root/reference/pkg/src/beziergraph/graph.py):

* ``build_graph``  (graph.py:129-199)  -> bzg_build_graph   (sampling, pair test, CSR, costs)
* ``cut_graph``    (graph.py:302-350)  -> bzg_cut_graph     (box heuristic + Cut-QP + aggregation)
* ``find_path``    (graph.py:353-430)  -> bzg_find_path     (snapping + Bellman-Ford + parents)
* ``path_cost``    (graph.py:453-458), ``check_edges`` (reachability.py:139-142)

All compute runs in libbzg.so on the GPU; the returned ``BezierGraph`` and
``CutMask`` keep their arrays device-resident and materialise the reference's
numpy fields (``vertices``, ``edges``, ``costs``, ``edge_points``, ``alive``,
``provenance``) lazily on first access, read-only like the reference's frozen
arrays (graph.py:70-73).  Inputs are duck-typed: the reference's own
``BezierSpec``/``ReachOracle``/``Box``/``Polytope`` instances work as well as
this package's host mirrors.
"""

from __future__ import annotations

import ctypes as C
import functools
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native as nat
from .bezier import boundary_matrix
from .geometry import EPS_GEO, recover_box, recover_boxes  # noqa: F401

_PAIR_CHUNK = 32  # kept for API parity with the reference module (graph.py:26)


class CutVerdict(Enum):
    UNSAFE = "unsafe"
    SAFE = "safe"
    INDETERMINATE = "indeterminate"


class CutProvenance(Enum):
    HEURISTIC_UNSAFE = "heuristic_unsafe"
    HEURISTIC_SAFE = "heuristic_safe"
    QP_SAFE = "qp_safe"
    QP_UNSAFE = "qp_unsafe"


# device provenance codes (include/bzg.h) -> enum order
_PROV_CODES = ("HEURISTIC_UNSAFE", "HEURISTIC_SAFE", "QP_SAFE", "QP_UNSAFE")
# the shim swaps this for the reference's enum so masks compare equal inside its simulator
_PROV_ENUM = CutProvenance


@dataclass
class SolveConfig:
    """Subset of the reference ``qpsolver.SolveConfig`` (qpsolver.py:60-72) the cut QP uses."""

    max_iter: int = 4000
    eps_abs: float = 1e-6
    eps_rel: float = 1e-6
    rho: float = 0.1
    sigma: float = 1e-6
    alpha: float = 1.6
    eps_pinf: float = 1e-4
    polish: bool = False


@dataclass
class CutConfig:
    """Reference ``CutConfig`` (graph.py:42-49)."""

    eps_cut: float = 1e-7
    heur_margin: float = 1e-6
    eps_geo: float = EPS_GEO
    qp: SolveConfig = field(
        default_factory=lambda: SolveConfig(max_iter=500, eps_abs=1e-7, eps_rel=0.0, rho=1.0, polish=True))


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ro(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


class BezierGraph:
    """Device-resident graph with the reference ``BezierGraph`` fields (graph.py:52-88)."""

    def __init__(self, handle, ctx, spec, oracle, seed, sample_bounds, D):
        self._h = handle
        self._ctx = ctx
        self.spec = spec
        self.oracle = oracle
        self.seed = seed
        self.sample_bounds = sample_bounds
        self._D = D
        V, E, rb, re_ = (C.c_int64() for _ in range(4))
        nat.check(ctx.lib.bzg_graph_info(handle, C.byref(V), C.byref(E), C.byref(rb), C.byref(re_)))
        self._V, self._E = V.value, E.value
        self.row_block = (rb.value, re_.value)
        self._cache: dict = {}
        self._desc_fn = None  # rebuilds the bzg_build_desc this graph came from (eps_band)

    def set_cut_cache(self, max_obstacles: int) -> None:
        """Keep per-obstacle cut outcomes on the device for up to ``max_obstacles`` distinct
        obstacles (bzg_graph_set_cut_cache): a later cut_graph on this graph screens and QPs only
        the obstacles it has not seen -- the moved ones of a replanning loop -- and recombines the
        rest; the mask equals a full cut's.  0 turns it off."""
        nat.check(self._ctx.lib.bzg_graph_set_cut_cache(self._h, int(max_obstacles)))

    def eps_band(self, eps: float = 1e-11) -> dict:
        """North-star report: ordered pairs whose minimum constraint slack lies in (-eps, eps]
        (bzg_graph_eps_band), i.e. the pairs whose edge bit could flip under an eps change of
        the thresholds.  ``band`` = feasible(G+eps) - feasible(G-eps) over this graph's rows."""
        if self._desc_fn is None:
            raise ValueError("this graph was not built by build_graph / build_region_graph")
        d, keep = self._desc_fn()
        out = np.zeros(3, dtype=np.int64)
        nat.check(self._ctx.lib.bzg_graph_eps_band(self._h, C.byref(d), float(eps), nat.ptr(out)))
        del keep
        return {"eps": float(eps), "band": int(out[0]), "feasible_plus": int(out[1]), "feasible_minus": int(out[2])}

    # ---- reference fields, materialised lazily
    @property
    def vertices(self) -> np.ndarray:
        if "vertices" not in self._cache:
            out = np.empty((self._V, self.spec.m * self.spec.gamma))
            nat.check(self._ctx.lib.bzg_graph_copy_vertices(self._h, nat.ptr(out)))
            self._cache["vertices"] = _ro(out)
        return self._cache["vertices"]

    def _edges_costs(self):
        if "edges" not in self._cache:
            e = np.empty((self._E, 2), dtype=np.int64)
            c = np.empty(self._E)
            nat.check(self._ctx.lib.bzg_graph_copy_edges(self._h, nat.ptr(e), nat.ptr(c)))
            self._cache["edges"] = _ro(e)
            self._cache["costs"] = _ro(c)

    @property
    def edges(self) -> np.ndarray:
        self._edges_costs()
        return self._cache["edges"]

    @property
    def costs(self) -> np.ndarray:
        self._edges_costs()
        return self._cache["costs"]

    @property
    def edge_points(self) -> np.ndarray:
        if "edge_points" not in self._cache:
            out = np.empty((self._E, self.spec.m, self.spec.p + 1))
            nat.check(self._ctx.lib.bzg_graph_copy_points(self._h, nat.ptr(out)))
            self._cache["edge_points"] = _ro(out)
        return self._cache["edge_points"]

    def csr(self) -> tuple[np.ndarray, np.ndarray]:
        """(row_ptr (V+1,) int64, col (E,) int32): the device CSR copied to host."""
        if "csr" not in self._cache:
            rp = np.empty(self._V + 1, dtype=np.int64)
            col = np.empty(self._E, dtype=np.int32)
            nat.check(self._ctx.lib.bzg_graph_copy_csr(self._h, nat.ptr(rp), nat.ptr(col)))
            self._cache["csr"] = (_ro(rp), _ro(col))
        return self._cache["csr"]

    @property
    def num_vertices(self) -> int:
        return self._V

    @property
    def num_edges(self) -> int:
        return self._E

    def to_json(self, max_edges: int | None = None) -> dict:
        edges = [[int(i), int(j), float(c)] for (i, j), c in zip(self.edges[:max_edges], self.costs[:max_edges])]
        return {"vertices": self.vertices.tolist(), "edges": edges}

    def close(self):
        if getattr(self, "_h", None):
            self._ctx.lib.bzg_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CutMask:
    """Outcome of one cut (reference ``CutMask``, graph.py:91-126), device-resident."""

    def __init__(self, handle, graph: BezierGraph, counters):
        self._h = handle
        self._graph = graph
        (self.pairs_total, self.pairs_point_hit, self.pairs_hyperplane, self.pairs_qp, self.qp_safe,
         self.qp_unsafe) = (int(x) for x in counters)
        self._alive = None
        self._alive_seen = None
        self._prov = None
        self._prov_codes = None

    @property
    def num_edges(self) -> int:
        """Edge count this mask was cut for (bzg_mask_info)."""
        E = C.c_int64()
        nat.check(self._graph._ctx.lib.bzg_mask_info(self._h, C.byref(E), None))
        return E.value

    def _copy(self):
        E = self.num_edges
        a = np.empty(E, dtype=np.uint8)
        p = np.empty(E, dtype=np.uint8)
        nat.check(self._graph._ctx.lib.bzg_mask_copy(self._h, nat.ptr(a), nat.ptr(p), None))
        self._alive = a.astype(bool)
        self._alive_seen = self._alive.copy()
        self._prov_codes = p

    @property
    def alive(self) -> np.ndarray:
        if self._alive is None:
            self._copy()
        return self._alive

    @alive.setter
    def alive(self, value):
        self._alive = np.asarray(value, dtype=bool)
        self._alive_seen = None  # force a re-upload before the next search

    @property
    def provenance_codes(self) -> np.ndarray:
        if self._prov_codes is None:
            self._copy()
        return self._prov_codes

    @property
    def provenance(self) -> np.ndarray:
        if self._prov is None:
            members = [getattr(_PROV_ENUM, nm) for nm in _PROV_CODES]
            table = np.empty(4, dtype=object)
            table[:] = members
            self._prov = table[self.provenance_codes]
        return self._prov

    @property
    def heuristic_fraction(self) -> float:
        if self.pairs_total == 0:
            return 1.0
        return 1.0 - self.pairs_qp / self.pairs_total

    @property
    def alive_count(self) -> int:
        return int(self.alive.sum())

    def qp_records(self) -> dict:
        """Per-QP diagnostics: edge, obstacle, status (0 solved..3 error), iterations, ||delta||.

        cut_graph skips the polish of SOLVED instances whose ADMM ||delta|| is >= 1e-2
        (BZG_POLISH_SCREEN; verdict-exact), so for those ``delta`` is the ADMM
        iterate's norm, not the polished one the reference's solve() would return (cut_qp
        polishes every instance).  With the re-cut cache on, the records cover the QPs solved by
        the cut that produced this mask (obstacles seen before contribute cached outcomes)."""
        lib = self._graph._ctx.lib
        n = C.c_int64()
        nat.check(lib.bzg_mask_qp_count(self._h, C.byref(n)))
        k = n.value
        out = dict(edge=np.empty(k, np.int64), obstacle=np.empty(k, np.int32), status=np.empty(k, np.int8),
                   iterations=np.empty(k, np.int32), delta=np.empty(k))
        nat.check(lib.bzg_mask_copy_qp(self._h, *(nat.ptr(out[x]) for x in
                                                  ("edge", "obstacle", "status", "iterations", "delta"))))
        return out

    def _device_handle(self):
        """Handle whose alive bits match the (possibly caller-modified) host array."""
        if self._alive is not None and (self._alive_seen is None or not np.array_equal(self._alive, self._alive_seen)):
            a = np.ascontiguousarray(self._alive, dtype=np.uint8)
            cnt = np.array([self.pairs_total, self.pairs_point_hit, self.pairs_hyperplane, self.pairs_qp,
                            self.qp_safe, self.qp_unsafe], dtype=np.int64)
            h = C.c_void_p()
            lib = self._graph._ctx.lib
            nat.check(lib.bzg_mask_from_arrays(self._graph._ctx.handle, self._graph._h, nat.ptr(a),
                                               nat.ptr(np.ascontiguousarray(self.provenance_codes)), nat.ptr(cnt), 0,
                                               C.byref(h)))
            lib.bzg_mask_destroy(self._h)
            self._h = h
            self._alive_seen = self._alive.copy()
        return self._h

    def to_json(self) -> dict:
        counts: dict[str, int] = {}
        for p in self.provenance:
            counts[p.value] = counts.get(p.value, 0) + 1
        return {
            "alive_bitset": np.packbits(self.alive).tobytes().hex(),
            "num_edges": int(self.alive.size),
            "alive": self.alive_count,
            "provenance_counts": counts,
            "pairs_total": self.pairs_total,
            "heuristic_fraction": self.heuristic_fraction,
        }

    def close(self):
        if getattr(self, "_h", None):
            self._graph._ctx.lib.bzg_mask_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _pcg_words(seed) -> tuple[int, int, int, int]:
    """numpy PCG64 (state, inc) for ``default_rng(seed)`` split into 64-bit halves."""
    if isinstance(seed, (int, np.integer)) or (isinstance(seed, (list, tuple)) and
                                                all(isinstance(s, (int, np.integer)) for s in seed)):
        return _pcg_words_cached(int(seed) if not isinstance(seed, (list, tuple)) else tuple(int(s) for s in seed))
    return _pcg_words_uncached(seed)


@functools.lru_cache(maxsize=512)
def _pcg_words_cached(seed) -> tuple[int, int, int, int]:
    return _pcg_words_uncached(list(seed) if isinstance(seed, tuple) else seed)


def _pcg_words_uncached(seed) -> tuple[int, int, int, int]:
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    mask = (1 << 64) - 1
    return s >> 64, s & mask, inc >> 64, inc & mask


def _build_desc(N, spec, oracle, bounds, seed, include, vertices=None, rows=None):
    m, g = int(spec.m), int(spec.gamma)
    n = m * g
    F = _f64(oracle.F)
    G = _f64(oracle.G)
    D = _f64(boundary_matrix(spec))
    xdA = _f64(oracle.Xd.A)
    xdb = _f64(oracle.Xd.b)
    lo = _f64(bounds.lo)
    hi = _f64(bounds.hi)
    inc = None
    if include is not None and len(include):
        inc = _f64(np.atleast_2d(np.asarray(include, dtype=np.float64)))
        if inc.shape[1] != n:
            raise ValueError(f"include rows must be {n}-dimensional")
    keep = [F, G, D, xdA, xdb, lo, hi, inc]
    d = nat.BuildDesc()
    d.m, d.gamma, d.p, d.n_F = m, g, int(spec.p), F.shape[0]
    d.F, d.G, d.D = nat.ptr(F), nat.ptr(G), nat.ptr(D)
    d.eps_geo = EPS_GEO
    d.N = int(N)
    if vertices is None:
        d.pcg_state_hi, d.pcg_state_lo, d.pcg_inc_hi, d.pcg_inc_lo = _pcg_words(seed)
    else:
        vv = _f64(vertices)
        keep.append(vv)
        d.vertices = nat.ptr(vv)
    d.sample_lo, d.sample_hi = nat.ptr(lo), nat.ptr(hi)
    d.xd_rows, d.xd_A, d.xd_b = xdA.shape[0], nat.ptr(xdA), nat.ptr(xdb)
    d.n_include = 0 if inc is None else inc.shape[0]
    d.include = nat.ptr(inc)
    d.row_begin, d.row_end = (0, 0) if rows is None else (int(rows[0]), int(rows[1]))
    return d, keep, D


def build_graph(N, spec, oracle, bounds, seed, include=None, k_nearest=None, *, ctx=None, rows=None):
    """Sample N states and connect every oracle-feasible ordered pair (reference graph.py:129-199).

    ``rows`` (keyword-only extension) restricts the pair test to the source-row block
    [rows[0], rows[1]) — the unit of multi-GPU row sharding.
    """
    if N < 2:
        raise ValueError("need at least two vertices")
    if bounds.dim != spec.n:
        raise ValueError(f"sampling bounds must be {spec.n}-dimensional")
    if k_nearest is not None and int(k_nearest) < 0:
        raise ValueError("k_nearest must be non-negative")
    ctx = ctx or nat.default_context()
    d, keep, D = _build_desc(N, spec, oracle, bounds, seed, include, rows=rows)
    if k_nearest is not None:
        d.k_nearest = int(k_nearest)  # graph.py:162-170, on device (k_knn_rows)
    h = C.c_void_p()
    rc = ctx.lib.bzg_build_graph(ctx.handle, C.byref(d), C.byref(h))
    if rc == nat.BZG_EINVAL:
        raise ValueError(ctx.lib.bzg_last_error().decode())
    nat.check(rc)
    del keep
    gr = BezierGraph(h, ctx, spec, oracle, seed, bounds, D)
    gr._desc_fn = lambda: _build_desc(N, spec, oracle, bounds, seed, include, vertices=None, rows=rows)[:2]
    return gr


def check_edges(oracle, X1, X2, eps: float = EPS_GEO, *, ctx=None) -> np.ndarray:
    """Batched feasibility F[x1;x2] <= G + eps in the separable form (reachability.py:139-142)."""
    ctx = ctx or nat.default_context()
    X1 = _f64(np.atleast_2d(X1))
    X2 = _f64(np.atleast_2d(X2))
    F = _f64(oracle.F)
    G = _f64(oracle.G)
    n = oracle.spec.n
    if X1.shape != X2.shape or X1.shape[1] != n:
        raise ValueError(f"endpoints must have dimension {n}")
    out = np.empty(X1.shape[0], dtype=np.uint8)
    nat.check(ctx.lib.bzg_check_edges(ctx.handle, n, F.shape[0], nat.ptr(F), nat.ptr(G), float(eps), X1.shape[0],
                                      nat.ptr(X1), nat.ptr(X2), nat.ptr(out)))
    return out.astype(bool)


def check_edge(oracle, x1, x2, eps: float = EPS_GEO, *, ctx=None) -> bool:
    """Scalar predicate (reachability.py:130-136) through the device batch kernel.

    Evaluated with check_edges' separable arithmetic fl(x1 F1' + x2 F2') -- build_graph's own
    edge test (graph.py:172-184) -- not the reference's length-2n gemv F @ [x1; x2], whose
    OpenBLAS summation order is not reproduced: for a pair within rounding of a threshold the
    answer can differ from the reference's scalar check_edge (never from its graph)."""
    x1 = np.asarray(x1, dtype=np.float64)
    x2 = np.asarray(x2, dtype=np.float64)
    n = oracle.spec.n
    if x1.shape != (n,) or x2.shape != (n,):
        raise ValueError(f"endpoints must have dimension {n}")
    return bool(check_edges(oracle, x1[None], x2[None], eps, ctx=ctx)[0])


_OBS_CACHE: dict = {}
_OBS_CACHE_SIZE = 8


def _obstacle_arrays(obstacles, m):
    """``_obstacle_arrays_uncached`` with a small identity cache: a replanning loop or a
    benchmark cuts the same obstacle objects again and again.  Only lists whose arrays are all
    read-only (both the reference's and this package's Polytope freeze them) are cached, and an
    entry keeps its obstacles alive so the identities in its key stay unique."""
    obstacles = list(obstacles)
    key = (m,) + tuple((id(ob), id(ob.A), id(ob.b)) for ob in obstacles)
    hit = _OBS_CACHE.get(key)
    if hit is not None:
        return hit[1]
    out = _obstacle_arrays_rows(obstacles, m)
    frozen = all(not np.asarray(ob.A).flags.writeable and not np.asarray(ob.b).flags.writeable
                 for ob in obstacles if isinstance(getattr(ob, "A", None), np.ndarray))
    if frozen and all(isinstance(getattr(ob, "A", None), np.ndarray) for ob in obstacles):
        if len(_OBS_CACHE) >= _OBS_CACHE_SIZE:
            _OBS_CACHE.pop(next(iter(_OBS_CACHE)))
        _OBS_CACHE[key] = (obstacles, out)
    return out


# Per-A-matrix constants of the obstacle preparation (row norms, normalised rows, and for 2m-row
# matrices the box-recovery structure), keyed by the identity of a read-only A: a moving
# obstacle is usually Polytope(A, b + A @ shift) with the same frozen A, so a replanning cycle
# recomputes only b-dependent values.  Entries pin their A so the identities stay unique.
_A_CACHE: dict = {}
_A_CACHE_SIZE = 4096


def _a_constants(A: np.ndarray, m: int):
    hit = _A_CACHE.get(id(A))
    if hit is not None and hit[0] is A:
        return hit[1]
    nrm = np.linalg.norm(A, axis=1)
    An = A / nrm[:, None]
    box = None
    if A.shape[0] == 2 * m:  # recover_boxes(An, bn) on one obstacle, the b-independent part
        n2 = np.linalg.norm(An, axis=1)
        rows = []
        ok = True
        for i in range(2 * m):
            row = An[i] / n2[i]
            ax = int(np.argmax(np.abs(row)))
            unit = np.zeros(m)
            unit[ax] = np.sign(row[ax])
            ok = ok and bool(np.all(np.abs(row - unit) <= 1e-12 + 1e-5 * np.abs(unit)))
            rows.append((ax, bool(row[ax] > 0), float(n2[i])))
        box = (ok, rows)
    const = (nrm, _ro(An), box)
    if not A.flags.writeable:
        if len(_A_CACHE) >= _A_CACHE_SIZE:
            _A_CACHE.pop(next(iter(_A_CACHE)))
        _A_CACHE[id(A)] = (A, const)
    return const


_OB_CACHE: dict = {}
_OB_CACHE_SIZE = 8192


def _one_obstacle(ob, m):
    """(An, bn, is_box, lo, hi) of one obstacle, cached by the identities of its read-only A, b."""
    A = np.asarray(ob.A, dtype=np.float64)
    b = np.asarray(ob.b, dtype=np.float64)
    key = (id(A), id(b))
    hit = _OB_CACHE.get(key)
    if hit is not None and hit[0] is A and hit[1] is b:
        return hit[2]
    if A.ndim != 2 or A.shape[1] != m:
        raise ValueError(f"obstacles must live in the {m}-d output space")
    nrm, An, box = _a_constants(A, m)
    bn = b / nrm
    isb, lo, hi = 0, (0.0,) * m, (0.0,) * m
    if box is not None:
        ok, info = box
        lo_l = [float("nan")] * m
        hi_l = [float("nan")] * m
        for i, (ax, pos, n2) in enumerate(info):
            val = float(bn[i]) / n2
            if pos:
                hi_l[ax] = val
            else:
                lo_l[ax] = -val
        if ok and not any(v != v for v in lo_l + hi_l) and not any(lo_l[j] > hi_l[j] for j in range(m)):
            isb, lo, hi = 1, tuple(lo_l), tuple(hi_l)
    out = (An, bn, isb, lo, hi)
    if not A.flags.writeable and not b.flags.writeable:
        if len(_OB_CACHE) >= _OB_CACHE_SIZE:
            _OB_CACHE.pop(next(iter(_OB_CACHE)))
        _OB_CACHE[key] = (A, b, out)
    return out


def _obstacle_arrays_rows(obstacles, m):
    """``_obstacle_arrays_uncached`` obstacle by obstacle with per-obstacle results cached (a
    replanning cycle recomputes only the moved obstacles): the same float operations in the
    same order (row norm, division, box recovery), so the arrays are bitwise the vectorised
    ones (tests/test_host_obstacles.py)."""
    if not obstacles:
        return _obstacle_arrays_uncached(obstacles, m)
    parts = [_one_obstacle(ob, m) for ob in obstacles]
    rows = [p[0].shape[0] for p in parts]
    offs = np.zeros(len(parts) + 1, np.int32)
    np.cumsum(rows, out=offs[1:])
    An = np.concatenate([p[0] for p in parts])
    bn = np.concatenate([p[1] for p in parts])
    is_box = np.fromiter((p[2] for p in parts), np.uint8, len(parts))
    lo = np.array([p[3] for p in parts], dtype=np.float64).reshape(len(parts), m)
    hi = np.array([p[4] for p in parts], dtype=np.float64).reshape(len(parts), m)
    return offs, An, bn, is_box, lo, hi


def _obstacle_arrays_uncached(obstacles, m):
    """Normalised rows (Polytope.normalized, geometry.py:135-137) and box recovery (as_box,
    geometry.py:155-185), vectorised over obstacles of 2m rows (the box shape)."""
    if not obstacles:
        return (np.zeros(1, np.int32), np.zeros((0, m)), np.zeros(0), np.zeros(0, np.uint8), np.zeros((0, m)),
                np.zeros((0, m)))
    As = [np.asarray(ob.A, dtype=np.float64) for ob in obstacles]
    bs = [np.asarray(ob.b, dtype=np.float64) for ob in obstacles]
    for A in As:
        if A.ndim != 2 or A.shape[1] != m:
            raise ValueError(f"obstacles must live in the {m}-d output space")
    O = len(As)
    rows = np.array([A.shape[0] for A in As])
    is_box = np.zeros(O, np.uint8)
    lo = np.zeros((O, m))
    hi = np.zeros((O, m))
    An_l, bn_l = [None] * O, [None] * O
    sq = np.nonzero(rows == 2 * m)[0]
    if sq.size:
        A3 = np.stack([As[i] for i in sq])
        b2 = np.stack([bs[i] for i in sq])
        nrm = np.linalg.norm(A3, axis=2)
        An3 = A3 / nrm[:, :, None]
        bn2 = b2 / nrm
        ok, l3, h3 = recover_boxes(An3, bn2)
        is_box[sq] = ok
        lo[sq] = l3
        hi[sq] = h3
        for k, i in enumerate(sq):
            An_l[i], bn_l[i] = An3[k], bn2[k]
    for i in np.nonzero(rows != 2 * m)[0]:
        nrm = np.linalg.norm(As[i], axis=1)
        An_l[i], bn_l[i] = As[i] / nrm[:, None], bs[i] / nrm
    offs = np.concatenate([[0], np.cumsum(rows)]).astype(np.int32)
    return offs, _f64(np.vstack(An_l)), _f64(np.concatenate(bn_l)), is_box, _f64(lo), _f64(hi)


def _cut_cfg(cfg) -> nat.CutConfigC:
    q = cfg.qp
    c = nat.CutConfigC()
    c.eps_cut, c.heur_margin, c.eps_geo = float(cfg.eps_cut), float(cfg.heur_margin), float(cfg.eps_geo)
    c.qp_max_iter = int(q.max_iter)
    c.qp_eps_abs, c.qp_eps_rel, c.qp_rho = float(q.eps_abs), float(q.eps_rel), float(q.rho)
    c.qp_sigma, c.qp_alpha, c.qp_eps_pinf = float(q.sigma), float(q.alpha), float(q.eps_pinf)
    c.qp_polish = int(bool(q.polish))
    return c


def cut_graph(graph: BezierGraph, obstacles, cfg: CutConfig | None = None) -> CutMask:
    """Screen every (edge, obstacle) pair, QP the leftovers, keep edges safe for all (graph.py:302-350).

    Obstacles: boxes (as_box) take the closed-form screen, other convex polytopes of up to 32
    rows the general one.  The polish of SOLVED QPs with ADMM ||delta|| >= 1e-2 is skipped
    (verdict-exact; see CutMask.qp_records).  One device synchronisation (the counters)."""
    cfg = cfg or CutConfig()
    ctx = graph._ctx
    arrs = _obstacle_arrays(list(obstacles), graph.spec.m)
    offs, A, b, is_box, lo, hi = arrs
    cc = _cut_cfg(cfg)
    h = C.c_void_p()
    nat.check(ctx.lib.bzg_cut_graph(ctx.handle, graph._h, len(is_box), nat.ptr(offs), nat.ptr(A), nat.ptr(b),
                                    nat.ptr(is_box), nat.ptr(lo), nat.ptr(hi), C.byref(cc), C.byref(h)))
    cnt = np.zeros(6, dtype=np.int64)
    nat.check(ctx.lib.bzg_mask_copy(h, None, None, nat.ptr(cnt)))
    return CutMask(h, graph, cnt)


# the shim swaps this for the reference's enum so verdicts compare equal inside its code
_VERDICT_ENUM = CutVerdict


def _cut_points(points, obstacles, obs_index, cfg, mode, ctx):
    """bzg_cut_points over B control-point sets (B, m, J) (include/bzg.h)."""
    cfg = cfg or CutConfig()
    ctx = ctx or nat.default_context()
    P = _f64(points)
    if P.ndim != 3:
        raise ValueError("points must be (B, m, p+1)")
    B, m, J = P.shape
    obstacles = list(obstacles)
    if not obstacles:
        raise ValueError("need at least one obstacle")
    idx = np.zeros(B, np.int32) if obs_index is None else np.ascontiguousarray(obs_index, dtype=np.int32)
    if idx.shape != (B,):
        raise ValueError("obs_index must have one entry per point set")
    offs, A, b, is_box, lo, hi = _obstacle_arrays(obstacles, m)
    cc = _cut_cfg(cfg)
    code = np.empty(B, np.int8)
    delta = np.empty(B) if mode == 1 else None
    status = np.empty(B, np.int8) if mode == 1 else None
    rc = ctx.lib.bzg_cut_points(ctx.handle, m, J, B, nat.ptr(P), nat.ptr(idx), len(obstacles), nat.ptr(offs),
                                nat.ptr(A), nat.ptr(b), nat.ptr(is_box), nat.ptr(lo), nat.ptr(hi), C.byref(cc), mode,
                                nat.ptr(code), nat.ptr(delta) if delta is not None else None,
                                nat.ptr(status) if status is not None else None)
    nat.check(rc)
    return code, delta, status


def cut_heuristic_batch(points, obstacles, obs_index=None, cfg: CutConfig | None = None, *, ctx=None) -> np.ndarray:
    """cut_heuristic (graph.py:202-221) for B control-point sets (B, m, p+1); set i against
    obstacles[obs_index[i]] (all against obstacles[0] when obs_index is None).  int8 codes
    0 unsafe / 1 safe / 2 indeterminate."""
    return _cut_points(points, obstacles, obs_index, cfg, 0, ctx)[0]


def cut_qp_batch(points, obstacles, obs_index=None, cfg: CutConfig | None = None, *, ctx=None):
    """cut_qp (graph.py:285-299) for B control-point sets: (safe (B,) bool, ||delta*|| (B,),
    solver status (B,) int8: 0 solved, 1 max_iter, 2 infeasible)."""
    code, delta, status = _cut_points(points, obstacles, obs_index, cfg, 1, ctx)
    return code.astype(bool), delta, status


def cut_heuristic(points, obstacle, cfg: CutConfig | None = None, *, ctx=None):
    """Three-branch screen for one edge's output control points (m, p+1) (graph.py:202-221)."""
    pts = np.atleast_2d(_f64(points))
    code = int(cut_heuristic_batch(pts[None], [obstacle], None, cfg, ctx=ctx)[0])
    return (_VERDICT_ENUM.UNSAFE, _VERDICT_ENUM.SAFE, _VERDICT_ENUM.INDETERMINATE)[code]


def cut_qp(points, obstacle, cfg: CutConfig | None = None, *, ctx=None) -> tuple[bool, float]:
    """Slack-minimising hull/obstacle test (graph.py:285-299): (safe, ||delta*||)."""
    pts = np.atleast_2d(_f64(points))
    safe, delta, _ = cut_qp_batch(pts[None], [obstacle], None, cfg, ctx=ctx)
    return bool(safe[0]), float(delta[0])


def find_path(graph: BezierGraph, mask, start, goal, position_only_snap: bool = False,
              require_tube_snap: bool = True):
    """Shortest alive path between the snapped start and goal (graph.py:353-430); None if none."""
    ctx = graph._ctx
    start = _f64(start)
    goal = _f64(goal)
    tube = graph.oracle.tube.error
    tlo, thi = _f64(tube.lo), _f64(tube.hi)
    mh = None
    tmp = None
    if isinstance(mask, CutMask):
        mh = mask._device_handle()
    elif mask is not None:  # a foreign (e.g. reference) CutMask: upload its alive bits
        a = np.ascontiguousarray(mask.alive, dtype=np.uint8)
        h = C.c_void_p()
        nat.check(ctx.lib.bzg_mask_from_arrays(ctx.handle, graph._h, nat.ptr(a), None, None, 0, C.byref(h)))
        mh = tmp = h
    path = np.empty(graph.num_vertices + 1, dtype=np.int64)
    plen = C.c_int64()
    dist = C.c_double()
    try:
        nat.check(ctx.lib.bzg_find_path(ctx.handle, graph._h, mh, nat.ptr(start), nat.ptr(goal), nat.ptr(tlo),
                                        nat.ptr(thi), EPS_GEO, int(bool(position_only_snap)),
                                        int(bool(require_tube_snap)), nat.ptr(path), path.size, C.byref(plen),
                                        C.byref(dist)))
    finally:
        if tmp is not None:
            ctx.lib.bzg_mask_destroy(tmp)
    if plen.value < 0:
        return None
    out = [int(v) for v in path[: plen.value]]
    graph._cache["last_dist"] = (tuple(out), dist.value)
    return out


class PathQuery:
    """Repeated ``find_path(graph, mask, start, goal, ...)`` on one fixed graph and mask -- the
    goal/start updates of a replanning loop (sim.py:275-408 calls graph.find_path every cycle,
    graph.py:353-430) -- as one captured CUDA graph (bzg_query): ``q(start, goal)`` returns what
    ``find_path`` returns with the same options, in one graph launch and one synchronisation.
    Creating it runs one search (warm-up) and the capture; it holds the graph and mask alive and
    becomes stale (ValueError) if the graph's edge set is replaced."""

    def __init__(self, graph: BezierGraph, mask, position_only_snap: bool = False, require_tube_snap: bool = True):
        ctx = graph._ctx
        self._ctx, self._graph, self._mask = ctx, graph, mask
        self._h = None
        self._tmp = None
        tube = graph.oracle.tube.error
        tlo, thi = _f64(tube.lo), _f64(tube.hi)
        mh = None
        if isinstance(mask, CutMask):
            mh = mask._device_handle()
        elif mask is not None:  # a foreign CutMask: its alive bits, owned by the query
            a = np.ascontiguousarray(mask.alive, dtype=np.uint8)
            h = C.c_void_p()
            nat.check(ctx.lib.bzg_mask_from_arrays(ctx.handle, graph._h, nat.ptr(a), None, None, 0, C.byref(h)))
            mh = self._tmp = h
        q = C.c_void_p()
        nat.check(ctx.lib.bzg_query_create(ctx.handle, graph._h, mh, nat.ptr(tlo), nat.ptr(thi), EPS_GEO,
                                           int(bool(position_only_snap)), int(bool(require_tube_snap)), C.byref(q)))
        self._h = q
        self._path = np.empty(graph.num_vertices + 1, dtype=np.int64)
        self._plen = C.c_int64()
        self._dist = C.c_double()

    @property
    def kernels_per_query(self) -> int:
        n = C.c_int64()
        nat.check(self._ctx.lib.bzg_query_kernels(self._h, C.byref(n)))
        return n.value

    def __call__(self, start, goal):
        start, goal = _f64(start), _f64(goal)
        nat.check(self._ctx.lib.bzg_query_run(self._h, nat.ptr(start), nat.ptr(goal), nat.ptr(self._path),
                                              self._path.size, C.byref(self._plen), C.byref(self._dist)))
        if self._plen.value < 0:
            return None
        out = [int(v) for v in self._path[: self._plen.value]]
        self._graph._cache["last_dist"] = (tuple(out), self._dist.value)
        return out

    def close(self):
        if getattr(self, "_h", None):
            self._ctx.lib.bzg_query_destroy(self._h)
            self._h = None
        if getattr(self, "_tmp", None):
            self._ctx.lib.bzg_mask_destroy(self._tmp)
            self._tmp = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def path_cost(graph: BezierGraph, path) -> float:
    """Total edge cost along a vertex path, left-to-right sum (graph.py:453-458)."""
    if len(path) < 2:
        return 0.0
    rp, col = graph.csr()
    costs = graph.costs
    total = 0
    for a, b in zip(path, path[1:]):
        lo, hi = int(rp[a]), int(rp[a + 1])
        k = lo + int(np.searchsorted(col[lo:hi], b))
        if k >= hi or col[k] != b:
            raise KeyError((a, b))
        total = total + costs[k]
    return float(total)
