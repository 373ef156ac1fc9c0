"""numpy restatement of the reference graph stage (TEST INFRASTRUCTURE ONLY).

Each function cites the reference lines it restates
(/root/reference/pkg/src/beziergraph/graph.py unless noted).  Expressions
keep the reference's float64 evaluation order so that outputs are bitwise
equal to the live reference on the same host (pinned by
tests/test_oracle_golden.py against tests/golden/).

Inputs are plain arrays or duck-typed objects with the reference's
attribute names (``spec.m/.gamma/.p/.n``, ``oracle.F/.G/.Xd/.tube``,
polytopes with ``A``/``b``), so the same oracle checks either the
reference's objects or the product package's host mirrors.
"""

from __future__ import annotations

import heapq

import numpy as np

from .qp_ref import AdmmSettings, SOLVED, cut_qp_problem, solve_dense_batch

EPS_GEO = 1e-9
PAIR_CHUNK = 32  # graph.py:26

# provenance codes (graph.py:35-39), shared with the device library
HEURISTIC_UNSAFE, HEURISTIC_SAFE, QP_SAFE, QP_UNSAFE = 0, 1, 2, 3


# ---------------------------------------------------------------- a2 sampler
def sample_states(N, lo, hi, xd_A, xd_b, seed, include=None, eps=EPS_GEO):
    """First N accepted rows of one PCG64 stream, then `include` (graph.py:147-159)."""
    rng = np.random.default_rng(seed)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    xd_A = np.asarray(xd_A, np.float64)
    xd_b = np.asarray(xd_b, np.float64)
    parts = []
    need = N
    while need > 0:
        cand = rng.uniform(lo, hi, size=(need, lo.size))  # geometry.py:69-72
        ok = np.all(cand @ xd_A.T <= xd_b + eps, axis=1)  # geometry.py:145-148
        got = cand[ok]
        if got.size:
            parts.append(got)
            need -= got.shape[0]
    V = np.vstack(parts)[:N]
    if include is not None and len(include):
        V = np.vstack([V, np.atleast_2d(np.asarray(include, dtype=np.float64))])
    return V


# ------------------------------------------------------- a3 / a4 pair test
def project(V, F, n):
    """A1 = V F1', A2 = V F2' through BLAS (graph.py:172-175)."""
    F = np.asarray(F, np.float64)
    return V @ F[:, :n].T, V @ F[:, n:].T


def pair_edges(A1, A2, G, eps=EPS_GEO, allowed=None, rows=None):
    """Row-major (src, dst) list of feasible ordered pairs, no self loops (graph.py:176-190).

    ``rows`` restricts the source rows to a contiguous block (multi-GPU row sharding / sampling).
    """
    thresh = np.asarray(G) + eps
    V = A1.shape[0]
    r0, r1 = (0, V) if rows is None else rows
    src_l, dst_l = [], []
    for lo in range(r0, r1, PAIR_CHUNK):
        hi = min(lo + PAIR_CHUNK, r1)
        lhs = A1[lo:hi][:, None, :] + A2[None, :, :]
        feas = np.all(lhs <= thresh, axis=2)
        feas[np.arange(hi - lo), np.arange(lo, hi)] = False
        if allowed is not None:
            feas &= allowed[lo:hi]
        s, d = np.nonzero(feas)
        src_l.append(s + lo)
        dst_l.append(d)
    if not src_l:
        return np.zeros((0, 2), dtype=np.int64)
    return np.stack([np.concatenate(src_l), np.concatenate(dst_l)], axis=1).astype(np.int64)


def eps_band(A1, A2, G, band_eps, eps=EPS_GEO, rows=None):
    """North-star eps-band count over ordered pairs i != j (source rows ``rows``):
    #all(lhs <= (G + eps) + band_eps) - #all(lhs <= (G + eps) - band_eps), lhs = A1[i] + A2[j]
    exactly as graph.py:176-184 forms it.  Returns (band, plus, minus)."""
    th = np.asarray(G) + eps
    hi, lo_ = th + band_eps, th - band_eps
    V = A1.shape[0]
    r0, r1 = (0, V) if rows is None else rows
    plus = minus = 0
    for lo in range(r0, r1, PAIR_CHUNK):
        h = min(lo + PAIR_CHUNK, r1)
        lhs = A1[lo:h][:, None, :] + A2[None, :, :]
        a = np.all(lhs <= hi, axis=2)
        b = np.all(lhs <= lo_, axis=2)
        idx = np.arange(h - lo)
        a[idx, idx + lo] = False
        b[idx, idx + lo] = False
        plus += int(a.sum())
        minus += int(b.sum())
    return plus - minus, plus, minus


def check_edges(F, G, n, X1, X2, eps=EPS_GEO):
    """Separable batched predicate (reference reachability.py:139-142)."""
    F = np.asarray(F, np.float64)
    lhs = X1 @ F[:, :n].T + X2 @ F[:, n:].T
    return np.all(lhs <= np.asarray(G) + eps, axis=1)


# ------------------------------------------------------- a5 points / costs
def edge_points(V, edges, D, gamma, m):
    """Output control points (E, m, p+1) by the boundary map (graph.py:192-196)."""
    x1 = V[edges[:, 0]].reshape(-1, gamma, m)
    x2 = V[edges[:, 1]].reshape(-1, gamma, m)
    bv = np.concatenate([x1, x2], axis=1)
    return np.einsum("pq,eqm->emp", D, bv)


def edge_costs(points):
    """Control-polygon length (graph.py:197)."""
    return np.linalg.norm(np.diff(points, axis=2), axis=1).sum(axis=1)


def knn_allowed(V, m, k_nearest):
    """k_nearest prefilter mask (graph.py:162-170), same numpy calls (argpartition ties included)."""
    pos = V[:, :m]
    d2 = ((pos[:, None, :] - pos[None, :, :]) ** 2).sum(axis=2)
    np.fill_diagonal(d2, np.inf)
    n = V.shape[0]
    k = min(k_nearest, n - 1)
    nbr = np.argpartition(d2, k - 1, axis=1)[:, :k]
    allowed = np.zeros((n, n), dtype=bool)
    allowed[np.repeat(np.arange(n), k), nbr.ravel()] = True
    return allowed


def build_graph(N, spec, oracle, bounds, seed, include=None, D=None, k_nearest=None):
    """Whole ``build_graph`` (graph.py:129-199); returns a dict of arrays."""
    if N < 2:
        raise ValueError("need at least two vertices")
    n = spec.m * spec.gamma
    V = sample_states(N, bounds.lo, bounds.hi, oracle.Xd.A, oracle.Xd.b, seed, include)
    allowed = None if k_nearest is None else knn_allowed(V, spec.m, k_nearest)
    A1, A2 = project(V, oracle.F, n)
    E = pair_edges(A1, A2, oracle.G, allowed=allowed)
    if D is None:
        from paper_2411_13507_b200.bezier import boundary_matrix  # host constant (bezier.py:185-211)
        D = boundary_matrix(spec)
    pts = edge_points(V, E, D, spec.gamma, spec.m)
    return {"vertices": V, "edges": E, "costs": edge_costs(pts), "edge_points": pts}


# ----------------------------------------------------------- a7 heuristic
def normalized(A, b):
    """Unit row normals (geometry.py:135-137)."""
    A = np.asarray(A, np.float64)
    b = np.asarray(b, np.float64)
    nrm = np.linalg.norm(A, axis=1)
    return A / nrm[:, None], b / nrm


def as_box(A, b):
    """Box (lo, hi) when rows are ±unit vectors (geometry.py:166-185), else None."""
    d = A.shape[1]
    if A.shape[0] != 2 * d:
        return None
    nrm = np.linalg.norm(A, axis=1)
    lo = np.full(d, np.nan)
    hi = np.full(d, np.nan)
    for i in range(A.shape[0]):
        row = A[i] / nrm[i]
        j = int(np.argmax(np.abs(row)))
        unit = np.zeros(d)
        unit[j] = np.sign(row[j])
        if not np.allclose(row, unit, atol=1e-12):
            return None
        if row[j] > 0:
            hi[j] = b[i] / nrm[i]
        else:
            lo[j] = -b[i] / nrm[i]
    if np.any(np.isnan(lo)) or np.any(np.isnan(hi)) or np.any(lo > hi):
        return None
    return lo, hi


_PROJ_QP = AdmmSettings(max_iter=20000, eps_abs=1e-10, eps_rel=1e-10, rho=0.1, sigma=1e-6, alpha=1.6,
                        eps_pinf=1e-4, polish=True)  # closest_point's SolveConfig (geometry.py:224)


def closest_point(A, b, x, eps=EPS_GEO):
    """Euclidean projection onto {A y <= b} (geometry.py:202-230): x itself when inside, the
    box clamp for boxes, else the dense ADMM QP with polish.  Raises on an empty polytope."""
    from .qp_ref import INFEASIBLE, _admm, _polish

    x = np.asarray(x, np.float64)
    if np.all(A @ x <= b + eps):  # Polytope.contains (geometry.py:139-143)
        return x.copy()
    box = as_box(A, b)
    if box is not None:
        return np.minimum(np.maximum(x, box[0]), box[1])  # Box.clamp
    d = A.shape[1]
    P = 2.0 * np.eye(d)
    q = -2.0 * x
    lo = np.full(A.shape[0], -np.inf)
    u = b.copy()
    xs, ys, st, _, rp, rd = _admm(P[None], q[None], A[None], lo[None], u[None], _PROJ_QP)
    if st[0] == INFEASIBLE:
        raise ValueError("cannot project onto an empty polytope")
    xo = xs[0]
    if st[0] in (SOLVED, 1):  # polish on SOLVED / MAX_ITER (qpsolver.py:301-303)
        xo, _ = _polish(P, q, A, lo, u, xo, ys[0], float(rp[0]), float(rd[0]))
    return xo


def adjacent_hyperplane(A, b, x, eps=EPS_GEO):
    """(unit normal, offset) of the deepest face active at the projection of x (geometry.py:233-252)."""
    x = np.asarray(x, np.float64)
    nrm = np.linalg.norm(A, axis=1)
    slack = (b - A @ x) / nrm
    if np.all(slack > eps):
        raise ValueError("adjacent_hyperplane requires a point outside the interior")
    y = closest_point(A, b, x, eps)
    residual = (b - A @ y) / nrm
    active = residual <= 1e-7
    if not np.any(active):
        active = np.ones(A.shape[0], dtype=bool)
    idx = int(np.argmax(np.where(active, -slack, -np.inf)))
    n = A[idx]
    nn = np.linalg.norm(n)
    return n / nn, float(b[idx]) / nn  # Hyperplane.__post_init__ (geometry.py:94-100)


def cut_heuristic(points, A, b, eps_geo=EPS_GEO, margin=1e-6):
    """Scalar three-branch screen of one edge (graph.py:202-221): 0 unsafe, 1 safe, 2 indeterminate."""
    pts = np.atleast_2d(np.asarray(points, np.float64))
    OA, Ob = normalized(A, b)
    if np.any(np.all(pts.T @ OA.T <= Ob + eps_geo, axis=1)):  # contains_many (geometry.py:145-148)
        return 0
    proj = [closest_point(OA, Ob, p) for p in pts.T]
    dists = [np.linalg.norm(pr - p) for pr, p in zip(proj, pts.T)]
    anchor = int(np.argmin(dists))
    normal, off = adjacent_hyperplane(OA, Ob, pts[:, anchor])
    return 1 if np.all(normal @ pts - off > margin) else 2


def heuristic_codes(points, A, b, eps_geo=EPS_GEO, margin=1e-6):
    """int8 codes 0 unsafe / 1 safe / 2 indeterminate for one obstacle (graph.py:224-265).

    Boxes take the closed-form branch; other polytopes run cut_heuristic per edge past
    branch 1 (graph.py:242-247).
    """
    E = points.shape[0]
    OA, Ob = normalized(A, b)
    codes = np.full(E, 2, dtype=np.int8)
    vals = np.einsum("cm,emj->ecj", OA, points)
    inside = np.all(vals <= Ob[None, :, None] + eps_geo, axis=1)
    hit = np.any(inside, axis=1)
    codes[hit] = 0
    rest = np.nonzero(~hit)[0]
    if rest.size == 0:
        return codes
    box = as_box(OA, Ob)
    if box is None:
        for e in rest:
            codes[e] = cut_heuristic(points[e], A, b, eps_geo, margin)
        return codes
    lo, hi = box
    pts = points[rest]
    below = np.maximum(lo[None, :, None] - pts, 0.0)
    above = np.maximum(pts - hi[None, :, None], 0.0)
    d2 = ((below + above) ** 2).sum(axis=1)
    k = np.argmin(d2, axis=1)
    v = np.take_along_axis(pts, k[:, None, None], axis=2)[:, :, 0]
    proj = np.clip(v, lo, hi)
    sep = v @ OA.T - Ob
    active = np.abs(proj @ OA.T - Ob) <= 1e-7
    face = np.argmax(np.where(active, sep, -np.inf), axis=1)
    h = OA[face]
    off = Ob[face]
    clear = np.einsum("em,emj->ej", h, pts) - off[:, None] > margin
    codes[rest[np.all(clear, axis=1)]] = 1
    return codes


# ------------------------------------------------------ a9 / a10 cut graph
def cut_graph(points, obstacles, eps_cut=1e-7, eps_geo=EPS_GEO, margin=1e-6, settings=None, record=False):
    """Heuristic screen + batched QP + aggregation (graph.py:302-350).

    ``obstacles`` is a list of (A, b).  Returns dict with alive (E,) bool,
    provenance (E,) int8 codes, the six counters, and (record=True) the per
    obstacle codes and QP outcomes for diagnosis.
    """
    s = settings or AdmmSettings()
    E = points.shape[0]
    J = points.shape[2]
    alive = np.ones(E, dtype=bool)
    prov = np.full(E, HEURISTIC_SAFE, dtype=np.int8)
    qp_saved = np.zeros(E, dtype=bool)
    cnt = dict(pairs_point_hit=0, pairs_hyperplane=0, pairs_qp=0, qp_safe=0, qp_unsafe=0)
    log = []
    for A, b in obstacles:
        codes = heuristic_codes(points, A, b, eps_geo, margin)
        cnt["pairs_point_hit"] += int((codes == 0).sum())
        cnt["pairs_hyperplane"] += int((codes == 1).sum())
        killed = (codes == 0) & alive
        prov[killed] = HEURISTIC_UNSAFE
        alive &= codes != 0
        pend = np.nonzero(codes == 2)[0]
        cnt["pairs_qp"] += int(pend.size)
        entry = {"codes": codes, "pending": pend}
        if pend.size:
            OA, Ob = normalized(A, b)
            probs = [cut_qp_problem(points[e], OA, Ob) for e in pend]
            P, q, Ac, l, u = (np.stack([p[i] for p in probs]) for i in range(5))
            x, st, its = solve_dense_batch(P, q, Ac, l, u, s)
            delta = np.array([float(np.linalg.norm(x[i, J:])) for i in range(pend.size)])
            safe = (st == SOLVED) & (delta > eps_cut)
            cnt["qp_safe"] += int(safe.sum())
            cnt["qp_unsafe"] += int((~safe).sum())
            qp_saved[pend[safe]] = True
            bad = pend[~safe]
            newly = bad[alive[bad]]
            prov[newly] = QP_UNSAFE
            alive[bad] = False
            entry.update(status=st, iters=its, delta=delta, safe=safe)
        if record:
            log.append(entry)
    prov[alive & qp_saved] = QP_SAFE
    out = dict(alive=alive, provenance=prov, pairs_total=E * len(obstacles), **cnt)
    if record:
        out["log"] = log
    return out


# --------------------------------------------------- a11 / a12 / a13 path
def _row_norms(X):
    return np.linalg.norm(X, axis=1)


def reaches_goal(V_count, edges, alive, vg):
    """Vertices with an alive route to vg by reverse DFS (graph.py:433-450)."""
    ae = edges[alive]
    order = np.argsort(ae[:, 1], kind="stable")
    es = ae[order]
    starts = np.searchsorted(es[:, 1], np.arange(V_count + 1))
    seen = np.zeros(V_count, dtype=bool)
    seen[vg] = True
    stack = [vg]
    while stack:
        node = stack.pop()
        for k in range(starts[node], starts[node + 1]):
            s = int(es[k, 0])
            if not seen[s]:
                seen[s] = True
                stack.append(s)
    return seen


def snap(vertices, edges, alive, start, goal, m, tube_lo, tube_hi, position_only_snap=False,
         require_tube_snap=True):
    """(v0, vg) or None exactly as graph.py:369-393."""
    start = np.asarray(start, np.float64)
    goal = np.asarray(goal, np.float64)
    gd = vertices - goal
    vg = int(np.argmin(_row_norms(gd[:, :m] if position_only_snap else gd)))
    sd = vertices - start
    nr = _row_norms(sd[:, :m] if position_only_snap else sd)
    in_tube = np.all((sd >= -tube_hi - EPS_GEO) & (sd <= -tube_lo + EPS_GEO), axis=1)
    if require_tube_snap:
        if not np.any(in_tube):
            return None
        cand = np.where(in_tube, nr, np.inf)
    else:
        ok = reaches_goal(vertices.shape[0], edges, alive, vg)
        if not np.any(ok):
            return None
        cand = np.where(ok, nr, np.inf)
    return int(np.argmin(cand)), vg


def find_path(vertices, edges, costs, alive, start, goal, m, tube_lo, tube_hi,
              position_only_snap=False, require_tube_snap=True):
    """Snapping + heapq Dijkstra + backtrack (graph.py:353-430). Returns (path|None, dist)."""
    sv = snap(vertices, edges, alive, start, goal, m, tube_lo, tube_hi, position_only_snap, require_tube_snap)
    if sv is None:
        return None, np.inf
    v0, vg = sv
    if v0 == vg:
        return [v0], 0.0
    V = vertices.shape[0]
    order = np.argsort(edges[:, 0], kind="stable")
    al = alive[order]
    es = edges[order]
    cs = costs[order]
    starts = np.searchsorted(es[:, 0], np.arange(V + 1))
    dist = np.full(V, np.inf)
    parent = np.full(V, -1, dtype=np.int64)
    dist[v0] = 0.0
    heap = [(0.0, v0)]
    done = np.zeros(V, dtype=bool)
    while heap:
        d, u = heapq.heappop(heap)
        if done[u]:
            continue
        done[u] = True
        if u == vg:
            break
        for k in range(starts[u], starts[u + 1]):
            if not al[k]:
                continue
            w = int(es[k, 1])
            nd = d + cs[k]
            if nd < dist[w]:
                dist[w] = nd
                parent[w] = u
                heapq.heappush(heap, (nd, w))
    if not np.isfinite(dist[vg]):
        return None, np.inf
    path = [vg]
    while path[-1] != v0:
        path.append(int(parent[path[-1]]))
    return path[::-1], float(dist[vg])


def path_cost(edges, costs, path):
    """Sum of edge costs along the path (graph.py:453-458)."""
    if len(path) < 2:
        return 0.0
    lookup = {(int(i), int(j)): c for (i, j), c in zip(edges, costs)}
    return float(sum(lookup[(a, b)] for a, b in zip(path, path[1:])))
