"""Keep-in regions restatement (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

No reference function exists for several free regions (SURVEY.md §0 "Gap to flag"); the
semantics frozen in paper_2411_13507_b200/regions.py are composed from reference
primitives, and this module restates that composition with numpy:
* per region r: build_graph's sampler (graph.py:147-157) with seed [seed, r], bounds
  = region bounding box x sample derivative box, acceptance in X_d,r;
* edge i -> j iff i != j and OR_r all(X1 F1_r' + X2 F2_r' <= G_r + eps)
  (check_edges, reachability.py:139-142), in row-major order;
* control points and costs exactly as graph.py:192-197.
Pinned by tests/golden/regions4.npz, generated from the live reference objects.
"""

from __future__ import annotations

import numpy as np

from .graph_ref import EPS_GEO, PAIR_CHUNK, edge_costs, edge_points, sample_states


def sample_regions(N_per, state_sets, bounds, seed):
    """state_sets: [(A, b)] per region; bounds: [(lo, hi)] per region."""
    parts = [sample_states(N_per, lo, hi, A, b, [seed, r]) for r, ((A, b), (lo, hi)) in enumerate(zip(state_sets, bounds))]
    return np.vstack(parts)


def region_edges(V, oracles, n, eps=EPS_GEO):
    """Row-major feasible pairs under OR over region oracles [(F, G)]."""
    proj = [(V @ np.asarray(F)[:, :n].T, V @ np.asarray(F)[:, n:].T, np.asarray(G) + eps) for F, G in oracles]
    Vn = V.shape[0]
    src_l, dst_l = [], []
    for lo in range(0, Vn, PAIR_CHUNK):
        hi = min(lo + PAIR_CHUNK, Vn)
        feas = np.zeros((hi - lo, Vn), dtype=bool)
        for A1, A2, th in proj:
            feas |= np.all(A1[lo:hi][:, None, :] + A2[None, :, :] <= th, axis=2)
        feas[np.arange(hi - lo), np.arange(lo, hi)] = False
        s, d = np.nonzero(feas)
        src_l.append(s + lo)
        dst_l.append(d)
    return np.stack([np.concatenate(src_l), np.concatenate(dst_l)], axis=1).astype(np.int64)


def build_region_graph(V, oracles, D, gamma, m):
    n = gamma * m
    E = region_edges(V, oracles, n)
    pts = edge_points(V, E, D, gamma, m)
    return {"vertices": V, "edges": E, "costs": edge_costs(pts), "edge_points": pts}
