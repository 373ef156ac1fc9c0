"""Keep-in free-space polytopes (north-star extension of build_graph, configs 1 and 5).

The reference has a single state set X_d (scenario.py:64).  BASELINE.json's configs 1 and 5
ask for graphs over several convex free regions.  The semantics are frozen here, composed
only from reference primitives (SURVEY.md §8(c) "Keep-in free polytopes"):

* region r is a position-space polytope {p : A_r p <= b_r}; its state set is
  X_d,r = Polytope([X_d.A; lift(A_r)], [X_d.b; b_r]) (lift pads the derivative columns
  with zeros) and its oracle is build_oracle(spec, X_d,r, U, tube) (reachability.py:97);
* vertices: per region, build_graph's sampler (graph.py:147-157) with
  bounds = bounding_box(region) x the derivative part of the sample box, accepting in
  X_d,r, and seed default_rng([seed, r]); regions are concatenated in order, then
  ``include`` rows;
* edge i -> j (i != j) iff OR_r check_edges(oracle_r, V[i], V[j]) (reachability.py:139-142,
  the same separable arithmetic as the pair test).

Every region oracle's F contains the base oracle's rows unchanged (the eroded X_d rows and
the input rows are computed row by row by the same products), so the device test is
base(i, j) AND OR_r region_r(i, j), where region_r covers only the rows the region adds:
its first/last-control-point rows are per-vertex membership predicates and its interior
rows are pair intervals.  ``region_rows`` extracts them and checks that claim bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import Box, Polytope, bounding_box
from .reachability import build_oracle


def lift(region: Polytope, n: int) -> Polytope:
    """Position-space rows padded with zeros for the derivative coordinates."""
    A = np.asarray(region.A, dtype=np.float64)
    return Polytope(np.hstack([A, np.zeros((A.shape[0], n - A.shape[1]))]), region.b)


def region_state_set(xd: Polytope, region: Polytope, n: int) -> Polytope:
    L = lift(region, n)
    return Polytope(np.vstack([xd.A, L.A]), np.concatenate([xd.b, L.b]))


def region_oracles(spec, xd: Polytope, U: Box, tube, regions) -> list:
    return [build_oracle(spec, region_state_set(xd, R, spec.n), U, tube) for R in regions]


def region_sample_bounds(region: Polytope, sample: Box, m: int) -> Box:
    bb = bounding_box(region)
    lo = np.concatenate([bb.lo, sample.lo[m:]])
    hi = np.concatenate([bb.hi, sample.hi[m:]])
    return Box(lo, hi)


@dataclass
class RegionRows:
    """Rows a region adds to the base oracle: F (k, 2n) and G (k,) for each region."""

    F: list
    G: list


def region_rows(base, oracles) -> RegionRows:
    """Per region, the F rows (and G) that are not rows of the base oracle.

    Raises if a base row is missing or differs in any bit (the device test relies on
    base(i, j) being a factor of every region's predicate).
    """
    base_rows = {(tuple(f), g) for f, g in zip(np.asarray(base.F), np.asarray(base.G))}
    Fs, Gs = [], []
    for o in oracles:
        F = np.asarray(o.F)
        G = np.asarray(o.G)
        keys = [(tuple(f), g) for f, g in zip(F, G)]
        present = set(keys)
        missing = [k for k in base_rows if k not in present]
        if missing:
            raise ValueError("a region oracle does not contain the base oracle's rows bit for bit")
        extra = np.array([k not in base_rows for k in keys])
        Fs.append(np.ascontiguousarray(F[extra]))
        Gs.append(np.ascontiguousarray(G[extra]))
    return RegionRows(Fs, Gs)


def region_boxes(regions) -> tuple[np.ndarray, np.ndarray]:
    """(R, m) position bounding boxes (membership culling hint for the device)."""
    boxes = [bounding_box(R) for R in regions]
    return (np.ascontiguousarray(np.stack([b.lo for b in boxes])), np.ascontiguousarray(np.stack([b.hi for b in boxes])))


@dataclass
class RegionSampling:
    """Host arrays of bzg_sample_region_states for one (spec, X_d, regions, sample box, seed)."""

    N: np.ndarray        # (R,) int64 samples per region
    pcg: np.ndarray      # (R, 4) uint64 PCG64 words of default_rng([seed, r])
    lo: np.ndarray       # (R, n) sampling boxes
    hi: np.ndarray
    row_off: np.ndarray  # (R+1,) int32 rows of each region's state set
    A: np.ndarray        # (rows, n)
    b: np.ndarray        # (rows,)

    @property
    def total(self) -> int:
        return int(self.N.sum())


def region_sampling(N_per_region, spec, xd: Polytope, regions, sample: Box, seed) -> RegionSampling:
    from .graph import _f64, _pcg_words

    R = len(regions)
    counts = np.full(R, int(N_per_region), np.int64) if np.isscalar(N_per_region) else np.asarray(
        N_per_region, np.int64)
    pcg = np.array([_pcg_words([seed, r]) for r in range(R)], dtype=np.uint64).reshape(R, 4)
    bnds = [region_sample_bounds(Rg, sample, spec.m) for Rg in regions]
    sets = [region_state_set(xd, Rg, spec.n) for Rg in regions]
    off = np.concatenate([[0], np.cumsum([s.A.shape[0] for s in sets])]).astype(np.int32)
    return RegionSampling(counts, np.ascontiguousarray(pcg), _f64(np.stack([b.lo for b in bnds])),
                          _f64(np.stack([b.hi for b in bnds])), off, _f64(np.vstack([s.A for s in sets])),
                          _f64(np.concatenate([s.b for s in sets])))


def sample_region_states(N_per_region, spec, xd: Polytope, regions, sample: Box, seed, *, ctx=None,
                         sampling: RegionSampling | None = None) -> np.ndarray:
    """Per-region samples (build_graph's sampler, default_rng([seed, r])) concatenated in region
    order, all regions in one device call (bzg_sample_region_states)."""
    from . import _native as nat
    from .graph import EPS_GEO

    ctx = ctx or nat.default_context()
    s = sampling or region_sampling(N_per_region, spec, xd, regions, sample, seed)
    out = np.empty((s.total, spec.n))
    if not len(s.N):
        return out
    nat.check(ctx.lib.bzg_sample_region_states(ctx.handle, spec.n, len(s.N), nat.ptr(s.N), nat.ptr(s.pcg),
                                               nat.ptr(s.lo), nat.ptr(s.hi), nat.ptr(s.row_off), nat.ptr(s.A),
                                               nat.ptr(s.b), EPS_GEO, nat.ptr(out)))
    return out


def build_region_graph(N_per_region, spec, oracle, regions, sample: Box, seed, include=None, *, ctx=None,
                       rows=None, rows_added: RegionRows | None = None, sampling: RegionSampling | None = None):
    """Graph over several keep-in regions (module docstring); returns a ``graph.BezierGraph``.

    ``oracle`` is the base ReachOracle (X_d, U, tube); ``regions`` are position-space polytopes.
    ``rows_added`` / ``sampling`` take the host constants (region_rows of the region oracles,
    region_sampling) when the caller keeps them across calls, as it keeps ``oracle``.
    """
    import ctypes as C

    from . import _native as nat
    from . import graph as G

    ctx = ctx or nat.default_context()
    if sample.dim != spec.n:
        raise ValueError(f"sampling bounds must be {spec.n}-dimensional")
    rr = rows_added
    if rr is None:
        rr = region_rows(oracle, region_oracles(spec, oracle.Xd, oracle.U, oracle.tube, regions))
    V = sample_region_states(N_per_region, spec, oracle.Xd, regions, sample, seed, ctx=ctx, sampling=sampling)
    if V.shape[0] < 2:
        raise ValueError("need at least two vertices")
    d, keep, D = G._build_desc(V.shape[0], spec, oracle, sample, seed, include, vertices=V, rows=rows)
    off = np.concatenate([[0], np.cumsum([f.shape[0] for f in rr.F])]).astype(np.int32)
    RF = G._f64(np.vstack(rr.F)) if rr.F else np.zeros((0, 2 * spec.n))
    RG = G._f64(np.concatenate(rr.G)) if rr.G else np.zeros(0)
    blo, bhi = region_boxes(regions)
    keep += [off, RF, RG, blo, bhi]
    d.n_regions = len(regions)
    d.region_row_off, d.region_F, d.region_G = nat.ptr(off), nat.ptr(RF), nat.ptr(RG)
    d.region_box_lo, d.region_box_hi = nat.ptr(blo), nat.ptr(bhi)
    h = C.c_void_p()
    rc = ctx.lib.bzg_build_graph(ctx.handle, C.byref(d), C.byref(h))
    if rc == nat.BZG_EINVAL:
        raise ValueError(ctx.lib.bzg_last_error().decode())
    nat.check(rc)
    gr = G.BezierGraph(h, ctx, spec, oracle, seed, sample, D)
    gr._desc_fn = lambda: (d, keep)
    return gr


def grid_regions(nx: int, ny: int, side_x: float, side_y: float, overlap: float = 0.10) -> list:
    """nx x ny axis-aligned cells of the [0, side_x] x [0, side_y] map, each grown by
    ``overlap`` of its size on every side (clipped to the map) so neighbours overlap."""
    cw, ch = side_x / nx, side_y / ny
    out = []
    for iy in range(ny):
        for ix in range(nx):
            lo = np.array([max(0.0, (ix - overlap) * cw), max(0.0, (iy - overlap) * ch)])
            hi = np.array([min(side_x, (ix + 1 + overlap) * cw), min(side_y, (iy + 1 + overlap) * ch)])
            out.append(Box(lo, hi).to_polytope())
    return out
