"""Capture golden vectors from the LIVE reference (run in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [case ...]

The reference (/root/reference/pkg/src/beziergraph, pure Python) cannot travel
to the GPU box, so its outputs on seeded inputs are frozen here as .npz
fixtures.  Each fixture records numpy/scipy/BLAS versions and the CPU model.
Large arrays are stored in full when small, otherwise as sha256 digests plus
the full bool/int8 outcome arrays (compressed) and the path.
"""

from __future__ import annotations

import hashlib
import json
import platform
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import beziergraph as bg  # noqa: E402
from beziergraph import geometry as rgeo  # noqa: E402
from beziergraph import graph as rg  # noqa: E402
from beziergraph import qpsolver as rqp  # noqa: E402
from beziergraph import scenario as rsc  # noqa: E402
from beziergraph import sim as rsim  # noqa: E402

OUT = Path(__file__).resolve().parent
PROV = {"heuristic_unsafe": 0, "heuristic_safe": 1, "qp_safe": 2, "qp_unsafe": 3}
STATUS = {"solved": 0, "max_iter": 1, "infeasible": 2, "error": 3}


def digest(a: np.ndarray) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()


def env_info() -> dict:
    cpu = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    import scipy

    blas = {}
    try:
        cfg = np.show_config(mode="dicts")
        blas = cfg["Build Dependencies"]["blas"]
    except Exception:  # pragma: no cover
        pass
    return {"numpy": np.__version__, "scipy": scipy.__version__, "blas": str(blas.get("version", "")),
            "blas_name": str(blas.get("name", "")), "cpu": cpu, "python": platform.python_version()}


def per_obstacle_detail(g, obstacles, cfg):
    """Per-obstacle heuristic codes and QP outcomes, computed with the reference's own internals
    exactly as cut_graph does (graph.py:312-337)."""
    codes_all, pend_o, pend_e, st, it, dl = [], [], [], [], [], []
    J = g.spec.p + 1
    for oi, ob in enumerate(obstacles):
        codes = rg._heuristic_batch(g.edge_points, ob, cfg)
        codes_all.append(codes)
        pending = np.nonzero(codes == 2)[0]
        if pending.size:
            O = ob.normalized()
            sols = rqp.solve_batch([rg._cut_qp_problem(g.edge_points[e], O) for e in pending], cfg.qp)
            for e, s in zip(pending, sols):
                pend_o.append(oi)
                pend_e.append(e)
                st.append(STATUS[s.status.value])
                it.append(s.iterations)
                dl.append(float(np.linalg.norm(s.x[J:])))
    return (np.stack(codes_all) if codes_all else np.zeros((0, g.num_edges), np.int8),
            np.array(pend_o, np.int32), np.array(pend_e, np.int64), np.array(st, np.int8),
            np.array(it, np.int64), np.array(dl))


def recorded_cut(g, obstacles, cfg):
    """Run the reference's own cut_graph once while recording, per QP, what it decided.

    `_heuristic_batch` and `qpsolver.solve_batch` are wrapped (the originals still do all the
    work), so the per-(edge, obstacle) QP outcomes come from the very calls cut_graph makes
    (graph.py:312-337), in its order: obstacle-major, pending edges ascending.
    """
    J = g.spec.p + 1
    state = {"obstacle": -1, "pending": None}
    po, pe, st, it, dl = [], [], [], [], []
    orig_h, orig_s = rg._heuristic_batch, rqp.solve_batch

    def heur(points, obstacle, c):
        codes = orig_h(points, obstacle, c)
        state["obstacle"] += 1
        state["pending"] = np.nonzero(codes == 2)[0]
        return codes

    def solve(probs, c):
        sols = orig_s(probs, c)
        pend = state["pending"]
        assert pend is not None and len(pend) == len(sols)
        po.append(np.full(len(sols), state["obstacle"], np.int32))
        pe.append(pend.astype(np.int64))
        st.append(np.array([STATUS[s.status.value] for s in sols], np.int8))
        it.append(np.array([s.iterations for s in sols], np.int64))
        dl.append(np.array([float(np.linalg.norm(s.x[J:])) for s in sols]))
        return sols

    rg._heuristic_batch, rqp.solve_batch = heur, solve
    try:
        mask = rg.cut_graph(g, obstacles, cfg)
    finally:
        rg._heuristic_batch, rqp.solve_batch = orig_h, orig_s
    cat = lambda l, dt: np.concatenate(l) if l else np.zeros(0, dt)  # noqa: E731
    return mask, (cat(po, np.int32), cat(pe, np.int64), cat(st, np.int8), cat(it, np.int64), cat(dl, np.float64))


def eps_band_count(oracle, V, n, eps=1e-11, chunk=32):
    """Ordered pairs (i != j) whose minimum constraint slack min_r(thresh_r - (a1[i,r] + a2[j,r]))
    lies in (-eps, eps], counted as #feasible(thresh + eps) - #feasible(thresh - eps) with the
    reference's own pair arithmetic (graph.py:172-189: a1 + a2 <= G + EPS_GEO)."""
    A1 = V @ oracle.F[:, :n].T
    A2 = V @ oracle.F[:, n:].T
    th = oracle.G + rg.EPS_GEO
    hi, lo = th + eps, th - eps
    cnt = 0
    for s in range(0, V.shape[0], chunk):
        e = min(s + chunk, V.shape[0])
        lhs = A1[s:e][:, None, :] + A2[None, :, :]
        a = np.all(lhs <= hi, axis=2)
        b = np.all(lhs <= lo, axis=2)
        idx = np.arange(e - s)
        a[idx, idx + s] = False
        b[idx, idx + s] = False
        cnt += int(a.sum()) - int(b.sum())
    return cnt


def capture(name, N, spec, oracle, bounds, seed, include, obstacles, start, goal, *, full, detail,
            goals=None, relaxed_starts=None, band=False, compact_qp=False):
    t0 = time.perf_counter()
    g = rg.build_graph(N, spec, oracle, bounds, seed, include=include)
    t_build = time.perf_counter() - t0
    print(f"{name}: built V={g.num_vertices} E={g.num_edges} in {t_build:.1f}s", flush=True)
    cfg = rg.CutConfig()
    t0 = time.perf_counter()
    if detail == "record":
        mask, qp_detail = recorded_cut(g, obstacles, cfg)
    else:
        mask = rg.cut_graph(g, obstacles, cfg)
    t_cut = time.perf_counter() - t0
    print(f"{name}: cut alive={mask.alive_count} qp={mask.pairs_qp} in {t_cut:.1f}s", flush=True)
    t0 = time.perf_counter()
    path = rg.find_path(g, mask, start, goal)
    t_path = time.perf_counter() - t0
    rec = {
        "N": N, "seed": seed, "V": g.num_vertices, "E": g.num_edges,
        "F": oracle.F, "G": oracle.G, "D": bg.bezier.boundary_matrix(spec),
        "m": spec.m, "gamma": spec.gamma, "p": spec.p, "T": spec.T,
        "bounds_lo": bounds.lo, "bounds_hi": bounds.hi, "xd_A": oracle.Xd.A, "xd_b": oracle.Xd.b,
        "tube_lo": oracle.tube.error.lo, "tube_hi": oracle.tube.error.hi,
        "include": np.zeros((0, spec.n)) if include is None else np.asarray(include, float),
        "obs_n": np.array([o.num_rows for o in obstacles], np.int32),
        "obs_A": np.concatenate([o.A for o in obstacles]) if obstacles else np.zeros((0, spec.m)),
        "obs_b": np.concatenate([o.b for o in obstacles]) if obstacles else np.zeros(0),
        "start": np.asarray(start, float), "goal": np.asarray(goal, float),
        "sha_vertices": digest(g.vertices), "sha_edges": digest(g.edges), "sha_costs": digest(g.costs),
        "sha_points": digest(g.edge_points),
        "alive": mask.alive.copy(),
        "provenance": np.array([PROV[p.value] for p in mask.provenance], np.int8),
        "counters": np.array([mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp,
                              mask.qp_safe, mask.qp_unsafe], np.int64),
        "path": np.array(path if path is not None else [], np.int64),
        "path_none": path is None,
        "path_cost": rg.path_cost(g, path) if path else 0.0,
        "t_build": t_build, "t_cut": t_cut, "t_path": t_path,
        "env": json.dumps(env_info()),
    }
    if full:
        rec.update(vertices=g.vertices, edges=g.edges, costs=g.costs, edge_points=g.edge_points)
    else:
        # enough raw rows to debug a mismatch without shipping the whole graph
        k = min(4096, g.num_edges)
        rec.update(vertices=g.vertices, edges_head=g.edges[:k], costs_head=g.costs[:k],
                   points_head=g.edge_points[:k],
                   row_counts=np.bincount(g.edges[:, 0], minlength=g.num_vertices).astype(np.int64))
    if detail == "record":
        po, pe, st, it, dl = qp_detail
        if compact_qp:  # headline-size graphs: narrow dtypes keep the fixture small
            rec.update(qp_obstacle=po.astype(np.uint8), qp_edge=pe.astype(np.int32), qp_status=st,
                       qp_iters=it.astype(np.int16), qp_delta=dl.astype(np.float32),
                       sha_qp_pairs=digest(pe * 1_000_003 + po))
        else:
            rec.update(qp_obstacle=po, qp_edge=pe, qp_status=st, qp_iters=it, qp_delta=dl)
    elif detail:
        codes, po, pe, st, it, dl = per_obstacle_detail(g, obstacles, cfg)
        rec.update(codes=codes, qp_obstacle=po, qp_edge=pe, qp_status=st, qp_iters=it, qp_delta=dl)
    if band:
        t0 = time.perf_counter()
        rec["eps_band_1e-11"] = eps_band_count(oracle, g.vertices, spec.n, 1e-11)
        rec["eps_band_1e-9"] = eps_band_count(oracle, g.vertices, spec.n, 1e-9)
        print(f"{name}: eps band {rec['eps_band_1e-11']} / {rec['eps_band_1e-9']} in {time.perf_counter()-t0:.1f}s",
              flush=True)
    if goals is not None:
        paths, costs = [], []
        for gl in goals:
            p = rg.find_path(g, mask, start, gl)
            paths.append(p if p is not None else [])
            costs.append(rg.path_cost(g, p) if p else np.inf)
        rec["goals"] = np.asarray(goals)
        rec["goal_path_len"] = np.array([len(p) for p in paths], np.int64)
        rec["goal_paths"] = np.concatenate([np.asarray(p, np.int64) for p in paths]) if paths else np.zeros(0, np.int64)
        rec["goal_costs"] = np.array(costs)
    if relaxed_starts is not None:
        paths = []
        for st_ in relaxed_starts:
            p = rg.find_path(g, mask, st_, goal, position_only_snap=True, require_tube_snap=False)
            paths.append(p if p is not None else [])
        rec["relaxed_starts"] = np.asarray(relaxed_starts)
        rec["relaxed_path_len"] = np.array([len(p) for p in paths], np.int64)
        rec["relaxed_paths"] = np.concatenate([np.asarray(p, np.int64) for p in paths])
    np.savez_compressed(OUT / f"{name}.npz", **rec)
    print(f"{name}: V={g.num_vertices} E={g.num_edges} alive={mask.alive_count} qp={mask.pairs_qp} "
          f"path={path} build={t_build:.2f}s cut={t_cut:.2f}s path={t_path*1e3:.1f}ms", flush=True)


def scenario_case(name, s, *, full, detail, goals=None, relaxed=None, extra=None, band=False):
    oracle = bg.build_oracle(s.spec, s.xd, s.u_bounds, s.tube)
    include = [s.start, s.goal]
    if extra is not None:
        include = list(extra) + include
    capture(name, s.graph_n, s.spec, oracle, s.sample_bounds, s.seed_graph, np.array(include),
            rsim._inflated(s, 0.0), s.start, s.goal, full=full, detail=detail, goals=goals, relaxed_starts=relaxed,
            band=band)


def case_demo():
    s = rsc.demo_scenario()
    s.graph_n = 200
    rng = np.random.default_rng(5)
    relaxed = np.hstack([rng.uniform(0.3, 4.7, (8, 2)), rng.uniform(-0.3, 0.3, (8, 2))])
    scenario_case("demo200", s, full=True, detail=True, relaxed=relaxed)


def case_rf_small():
    s = rsc.random_field_scenario(5, n_obstacles=20, graph_n=300)
    scenario_case("rf300_s5", s, full=True, detail=True)


def case_cfg2():
    s = rsc.random_field_scenario(1, n_obstacles=20, graph_n=2000)
    rng = np.random.default_rng(0)
    goals = np.zeros((100, 4))
    goals[:, :2] = rng.uniform(0.3, 4.7, size=(100, 2))
    scenario_case("cfg2_rf2000", s, full=False, detail="record", goals=goals, band=True)


def case_maze():
    s, grid = rsc.maze_scenario()
    scenario_case("maze", s, full=False, detail="record", extra=grid)


def _hop_spec():
    spec = bg.BezierSpec(m=2, gamma=3, T=1.0)
    xd = rgeo.Box(np.array([0.0, 0.0, -1.5, -1.5, -4.0, -4.0]), np.array([5.0, 5.0, 1.5, 1.5, 4.0, 4.0])).to_polytope()
    u = rgeo.Box(np.array([-30.0, -30.0]), np.array([30.0, 30.0]))
    sample = rgeo.Box(np.array([0.0, 0.0, -0.6, -0.6, -1.0, -1.0]), np.array([5.0, 5.0, 0.6, 0.6, 1.0, 1.0]))
    tube = rsim.design_tube(spec, (6.0, 11.0, 6.0), 0.02)
    return spec, xd, u, sample, tube


def case_hop_small():
    """gamma=3 (degree 5) at reduced size: the cfg3 recipe with N=1500 and 12 boxes."""
    spec, xd, u, sample, tube = _hop_spec()
    oracle = bg.build_oracle(spec, xd, u, tube)
    rng = np.random.default_rng(11)
    obs = []
    for _ in range(12):
        c = rng.uniform(0.4, 4.6, 2)
        w = rng.uniform(0.25, 0.7, 2)
        obs.append(rsc._box_obstacle(c[0], c[1], w[0], w[1]).shape)
    pos = tube.position_box(2)
    obs = [rgeo.inflate(o, pos) for o in obs]
    start = np.array([0.4, 0.4, 0, 0, 0, 0.0])
    goal = np.array([4.6, 4.6, 0, 0, 0, 0.0])
    capture("hop1500", 1500, spec, oracle, sample, 1, np.array([start, goal]), obs, start, goal,
            full=True, detail=True)


def case_reject():
    """Non-box state set with heavy rejection (~half the candidates) to pin the sampler."""
    spec = bg.BezierSpec(m=2, gamma=2, T=1.0)
    xd0, u, sample = rsc._standard_sets()
    # cut the square by the diagonal half-plane x + y <= 5
    A = np.vstack([xd0.A, [[1.0, 1.0, 0.0, 0.0]]])
    b = np.concatenate([xd0.b, [5.0]])
    xd = rgeo.Polytope(A, b)
    tube = rsim.design_tube(spec, (6.0, 5.0), 0.02)
    oracle = bg.build_oracle(spec, xd, u, tube)
    start = np.array([0.5, 0.5, 0, 0.0])
    goal = np.array([3.0, 1.5, 0, 0.0])
    obs = [rgeo.inflate(rsc._box_obstacle(1.5, 1.5, 0.6, 0.6).shape, tube.position_box(2))]
    capture("reject400", 400, spec, oracle, sample, 3, np.array([start, goal]), obs, start, goal,
            full=True, detail=True)


def case_regions4(name="regions4", quads=None):
    """cfg1: 4 overlapping quadrant keep-in regions x 50 samples, composed from reference objects
    (SURVEY.md §8(c)): X_d,r = [X_d; lift(region)], oracle_r = build_oracle(X_d,r), sampler of
    graph.py:147-157 with default_rng([seed, r]), edges = OR_r check_edges(oracle_r)."""
    spec = bg.BezierSpec(m=2, gamma=2, T=1.0)
    xd, U, sample = rsc._standard_sets()
    tube = rsim.design_tube(spec, (6.0, 5.0), 0.02)
    base = bg.build_oracle(spec, xd, U, tube)
    quads = quads or [((0.0, 0.0), (3.0, 3.0)), ((2.0, 0.0), (5.0, 3.0)), ((0.0, 2.0), (3.0, 5.0)), ((2.0, 2.0), (5.0, 5.0))]
    seed, N = 4, 50
    parts, oracles, F_l, G_l = [], [], [], []
    for r, (lo, hi) in enumerate(quads):
        R = rgeo.Box(np.array(lo), np.array(hi)).to_polytope()
        lifted = np.hstack([R.A, np.zeros((R.A.shape[0], spec.n - spec.m))])
        Xr = rgeo.Polytope(np.vstack([xd.A, lifted]), np.concatenate([xd.b, R.b]))
        o = bg.build_oracle(spec, Xr, U, tube)
        oracles.append(o)
        F_l.append(o.F)
        G_l.append(o.G)
        bb = rgeo.bounding_box(R)
        bounds = rgeo.Box(np.concatenate([bb.lo, sample.lo[2:]]), np.concatenate([bb.hi, sample.hi[2:]]))
        rng = np.random.default_rng([seed, r])  # graph.py:147-157 with the region's X_d
        got, need = [], N
        while need > 0:
            cand = bounds.sample(rng, need)
            acc = cand[Xr.contains_many(cand)]
            if acc.size:
                got.append(acc)
                need -= acc.shape[0]
        parts.append(np.vstack(got)[:N])
    start = np.array([0.5, 0.5, 0.0, 0.0])
    goal = np.array([4.5, 4.5, 0.0, 0.0])
    V = np.vstack(parts + [np.array([start, goal])])
    Vn = V.shape[0]
    I, Jx = np.meshgrid(np.arange(Vn), np.arange(Vn), indexing="ij")
    I, Jx = I.ravel(), Jx.ravel()
    feas = np.zeros(I.size, dtype=bool)
    for o in oracles:
        feas |= bg.reachability.check_edges(o, V[I], V[Jx])
    feas &= I != Jx
    E = np.stack([I[feas], Jx[feas]], axis=1).astype(np.int64)
    D = bg.bezier.boundary_matrix(spec)
    x1 = V[E[:, 0]].reshape(-1, spec.gamma, spec.m)
    x2 = V[E[:, 1]].reshape(-1, spec.gamma, spec.m)
    pts = np.einsum("pq,eqm->emp", D, np.concatenate([x1, x2], axis=1))
    costs = np.linalg.norm(np.diff(pts, axis=2), axis=1).sum(axis=1)
    base_only = int(bg.reachability.check_edges(base, V[I], V[Jx])[I != Jx].sum())
    np.savez_compressed(OUT / f"{name}.npz", vertices=V, edges=E, costs=costs, edge_points=pts, seed=seed,
                        N_per=N, quads=np.array(quads, dtype=float), start=start, goal=goal,
                        F_regions=np.stack(F_l), G_regions=np.stack(G_l), base_F=base.F, base_G=base.G, D=D,
                        base_only_edges=base_only, env=json.dumps(env_info()))
    print(f"{name}: V={Vn} E={E.shape[0]} (base oracle alone: {base_only})")


def _regular_polygon(center, radius, k, phase):
    ang = phase + 2 * np.pi * np.arange(k) / k
    A = np.stack([np.cos(ang), np.sin(ang)], axis=1) * 1.7  # non-unit rows: normalisation is exercised
    b = A @ np.asarray(center, float) + radius * 1.7
    return rgeo.Polytope(A, b)


def general_obstacles():
    """Convex non-box obstacles with 3..8 rows (rotated square, triangle, pentagon, hexagon,
    octagon) and one box, in the demo map."""
    return [
        _regular_polygon((2.5, 2.5), 0.45, 4, np.pi / 4 + 0.3),   # rotated square
        _regular_polygon((1.3, 3.7), 0.35, 3, 0.2),               # triangle
        _regular_polygon((3.7, 1.3), 0.40, 5, 0.1),               # pentagon
        _regular_polygon((1.2, 1.6), 0.30, 6, 0.0),               # hexagon
        _regular_polygon((3.6, 3.4), 0.38, 8, np.pi / 8),         # octagon
        rgeo.Box(np.array([2.2, 0.3]), np.array([2.7, 0.9])).to_polytope(),
    ]


def case_general():
    """Graph golden with general (non-box) obstacles: _heuristic_batch's per-edge
    cut_heuristic branch (graph.py:242-247) and the Cut-QP on 3..8-row obstacles."""
    s = rsc.demo_scenario()
    oracle = bg.build_oracle(s.spec, s.xd, s.u_bounds, s.tube)
    capture("general60", 60, s.spec, oracle, s.sample_bounds, 11, np.array([s.start, s.goal]),
            general_obstacles(), s.start, s.goal, full=True, detail=True)


def case_heur_general():
    """Scalar cut_heuristic / closest_point / adjacent_hyperplane on random control polygons
    near general obstacles (geometry.py:202-252, graph.py:202-221)."""
    rng = np.random.default_rng(3)
    obs = general_obstacles()[:5]
    cfg = rg.CutConfig()
    pts_l, oi_l, code_l, proj_l, hp_l = [], [], [], [], []
    for i in range(400):
        oi = i % len(obs)
        O = obs[oi]
        ctr = {0: (2.5, 2.5), 1: (1.3, 3.7), 2: (3.7, 1.3), 3: (1.2, 1.6), 4: (3.6, 3.4)}[oi]
        pts = np.asarray(ctr)[:, None] + rng.uniform(-0.9, 0.9, (2, 1)) + rng.uniform(-0.35, 0.35, (2, 4))
        pts_l.append(pts)
        oi_l.append(oi)
        code_l.append({rg.CutVerdict.UNSAFE: 0, rg.CutVerdict.SAFE: 1, rg.CutVerdict.INDETERMINATE: 2}[
            rg.cut_heuristic(pts, O, cfg)])
        On = O.normalized()
        proj_l.append(np.stack([rgeo.closest_point(On, p) for p in pts.T]))
        try:
            hp = rgeo.adjacent_hyperplane(On, pts[:, 0])
            hp_l.append(np.concatenate([hp.normal, [hp.offset]]))
        except ValueError:
            hp_l.append(np.full(3, np.nan))
    np.savez_compressed(OUT / "heur_general.npz", points=np.stack(pts_l), obstacle=np.array(oi_l, np.int32),
                        codes=np.array(code_l, np.int8), projections=np.stack(proj_l), hyperplanes=np.stack(hp_l),
                        obs_n=np.array([o.num_rows for o in obs], np.int32),
                        obs_A=np.concatenate([o.A for o in obs]), obs_b=np.concatenate([o.b for o in obs]),
                        env=json.dumps(env_info()))
    print("heur_general:", np.bincount(np.array(code_l), minlength=3))


def case_knn():
    """build_graph with the k_nearest prefilter (graph.py:162-170), k in {1, 12, 60} and k >= V-1."""
    s = rsc.random_field_scenario(3, n_obstacles=0, graph_n=400)
    oracle = bg.build_oracle(s.spec, s.xd, s.u_bounds, s.tube)
    rec = {"env": json.dumps(env_info()), "F": oracle.F, "G": oracle.G, "xd_A": oracle.Xd.A, "xd_b": oracle.Xd.b,
           "bounds_lo": s.sample_bounds.lo, "bounds_hi": s.sample_bounds.hi, "m": s.spec.m, "gamma": s.spec.gamma,
           "T": s.spec.T, "N": 400, "seed": 7, "ks": np.array([1, 12, 60, 500])}
    for k in rec["ks"]:
        g = rg.build_graph(400, s.spec, oracle, s.sample_bounds, 7, k_nearest=int(k))
        rec[f"edges_k{k}"] = g.edges
        rec[f"costs_k{k}"] = g.costs
    g = rg.build_graph(400, s.spec, oracle, s.sample_bounds, 7)
    rec["edges_all"] = g.edges
    rec["vertices"] = g.vertices
    np.savez_compressed(OUT / "knn400.npz", **rec)
    print("knn400:", {int(k): rec[f"edges_k{k}"].shape[0] for k in rec["ks"]}, "all", g.num_edges)


def _rotation(rng):
    q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    return q


def general_obstacles_3d():
    """3-D convex non-box obstacles: rotated box (6 rows), octahedron (8), tetrahedron (4)."""
    rng = np.random.default_rng(9)
    out = []
    base = {
        "box": np.vstack([np.eye(3), -np.eye(3)]),
        "octa": np.array([[sx, sy, sz] for sx in (1, -1) for sy in (1, -1) for sz in (1, -1)], float),
        "tetra": np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], float),
    }
    for name, ctr, rad in (("box", (2.5, 2.5, 2.5), 0.5), ("octa", (1.3, 3.6, 2.0), 0.45),
                           ("tetra", (3.6, 1.4, 3.0), 0.35), ("box", (1.2, 1.2, 3.8), 0.3)):
        A = base[name] @ _rotation(rng).T * 1.3
        out.append(rgeo.Polytope(A, A @ np.asarray(ctr) + rad * np.linalg.norm(A, axis=1)))
    return out


def case_heur_general3():
    """Scalar cut_heuristic / closest_point / adjacent_hyperplane for m = 3 polytopes."""
    rng = np.random.default_rng(4)
    obs = general_obstacles_3d()
    ctrs = [(2.5, 2.5, 2.5), (1.3, 3.6, 2.0), (3.6, 1.4, 3.0), (1.2, 1.2, 3.8)]
    cfg = rg.CutConfig()
    pts_l, oi_l, code_l, proj_l, hp_l = [], [], [], [], []
    for i in range(240):
        oi = i % len(obs)
        O = obs[oi]
        pts = np.asarray(ctrs[oi])[:, None] + rng.uniform(-1.0, 1.0, (3, 1)) + rng.uniform(-0.35, 0.35, (3, 4))
        pts_l.append(pts)
        oi_l.append(oi)
        code_l.append({rg.CutVerdict.UNSAFE: 0, rg.CutVerdict.SAFE: 1, rg.CutVerdict.INDETERMINATE: 2}[
            rg.cut_heuristic(pts, O, cfg)])
        On = O.normalized()
        proj_l.append(np.stack([rgeo.closest_point(On, p) for p in pts.T]))
        try:
            hp = rgeo.adjacent_hyperplane(On, pts[:, 0])
            hp_l.append(np.concatenate([hp.normal, [hp.offset]]))
        except ValueError:
            hp_l.append(np.full(4, np.nan))
    np.savez_compressed(OUT / "heur_general3.npz", points=np.stack(pts_l), obstacle=np.array(oi_l, np.int32),
                        codes=np.array(code_l, np.int8), projections=np.stack(proj_l), hyperplanes=np.stack(hp_l),
                        obs_n=np.array([o.num_rows for o in obs], np.int32),
                        obs_A=np.concatenate([o.A for o in obs]), obs_b=np.concatenate([o.b for o in obs]),
                        env=json.dumps(env_info()))
    print("heur_general3:", np.bincount(np.array(code_l), minlength=3))


def case_m1():
    """One output dimension (m=1, gamma=3): numpy's contiguous einsum kernel in the control-point map."""
    spec = bg.BezierSpec(m=1, gamma=3, T=1.0)
    xd = rgeo.Box(np.array([0.0, -1.5, -4.0]), np.array([5.0, 1.5, 4.0])).to_polytope()
    u = rgeo.Box(np.array([-30.0]), np.array([30.0]))
    tube = rsim.design_tube(spec, (6.0, 11.0, 6.0), 0.02)
    oracle = bg.build_oracle(spec, xd, u, tube)
    sample = rgeo.Box(np.array([0.0, -0.6, -1.0]), np.array([5.0, 0.6, 1.0]))
    obs = [rgeo.inflate(rgeo.Box(np.array([c - w / 2]), np.array([c + w / 2])).to_polytope(), tube.position_box(1))
           for c, w in ((1.3, 0.2), (2.6, 0.15), (3.9, 0.3))]
    start = np.array([0.2, 0.0, 0.0])
    goal = np.array([4.8, 0.0, 0.0])
    capture("m1_300", 300, spec, oracle, sample, 6, np.array([start, goal]), obs, start, goal, full=True, detail=True)


def case_m3():
    """Three output dimensions (m=3, gamma=2): 3-D boxes through the whole path."""
    spec = bg.BezierSpec(m=3, gamma=2, T=1.0)
    xd = rgeo.Box(np.array([0.0, 0, 0, -1.5, -1.5, -1.5]), np.array([5.0, 5, 5, 1.5, 1.5, 1.5])).to_polytope()
    u = rgeo.Box(np.full(3, -6.0), np.full(3, 6.0))
    tube = rsim.design_tube(spec, (6.0, 5.0), 0.02)
    oracle = bg.build_oracle(spec, xd, u, tube)
    sample = rgeo.Box(np.array([0.0, 0, 0, -0.6, -0.6, -0.6]), np.array([5.0, 5, 5, 0.6, 0.6, 0.6]))
    rng = np.random.default_rng(2)
    obs = []
    for _ in range(8):
        c = rng.uniform(0.8, 4.2, 3)
        s = rng.uniform(0.3, 0.9, 3)
        obs.append(rgeo.inflate(rgeo.Box(c - s / 2, c + s / 2).to_polytope(), tube.position_box(3)))
    start = np.array([0.3, 0.3, 0.3, 0, 0, 0])
    goal = np.array([4.7, 4.7, 4.7, 0, 0, 0])
    capture("m3_600", 600, spec, oracle, sample, 4, np.array([start, goal]), obs, start, goal, full=True,
            detail=True)


def _clear_boxes(rng, count, lo, hi, start, goal):
    """Random boxes (centre U(lo, hi)^2, side U(0.25, 0.7)^2), redrawn within 0.9 of start/goal
    (the reference random field's rule, scenario.py:373-374)."""
    out = []
    while len(out) < count:
        c = rng.uniform(lo, hi, 2)
        w = rng.uniform(0.25, 0.7, 2)
        if np.linalg.norm(c - start[:2]) < 0.9 or np.linalg.norm(c - goal[:2]) < 0.9:
            continue
        out.append(rsc._box_obstacle(c[0], c[1], w[0], w[1]).shape)
    return out


def case_cfg3():
    """BASELINE cfg3 exactly as bench.py runs it (configs.hopping_deg5): gamma=3, 20,000 samples
    + start/goal, 50 inflated boxes from default_rng(11).  Reference build ~4 min, cut ~20 min.
    Digests for the big arrays, full alive/provenance, per-QP outcomes, path, eps-band counts."""
    spec, xd, u, sample, tube = _hop_spec()
    oracle = bg.build_oracle(spec, xd, u, tube)
    start = np.array([0.4, 0.4, 0, 0, 0, 0.0])
    goal = np.array([4.6, 4.6, 0, 0, 0, 0.0])
    pos = tube.position_box(2)
    obs = [rgeo.inflate(o, pos) for o in _clear_boxes(np.random.default_rng(11), 50, 0.4, 4.6, start, goal)]
    capture("cfg3_hop20k", 20000, spec, oracle, sample, 1, np.array([start, goal]), obs, start, goal,
            full=False, detail="record", band=True, compact_qp=True)


def case_cfg5_10k():
    """BASELINE cfg5 at 10k nodes (configs.scaling_sweep(10000)): 200 keep-in cells (20 x 10 grid,
    10% overlap) on a 5 sqrt(5) map, 50 boxes from default_rng(101), composed from reference
    objects as in case_regions4.  Candidate pairs per region are the vertices inside the region's
    box: exact, because P_0 = x1 and P_p = x2 are control points and the region oracle keeps
    them in the (eroded) region.  Then the reference's own cut_graph and find_path on it."""
    N, seed = 10000, 1
    spec = bg.BezierSpec(m=2, gamma=2, T=1.0)
    side = 5.0 * float(np.sqrt(N / 2000.0))
    xd, U, sample = rsc._standard_sets(side=side)
    tube = rsim.design_tube(spec, (6.0, 5.0), 0.02)
    base = bg.build_oracle(spec, xd, U, tube)
    nx, ny, ov = 20, 10, 0.10
    cw, ch = side / nx, side / ny
    regions = []
    for iy in range(ny):
        for ix in range(nx):
            lo = np.array([max(0.0, (ix - ov) * cw), max(0.0, (iy - ov) * ch)])
            hi = np.array([min(side, (ix + 1 + ov) * cw), min(side, (iy + 1 + ov) * ch)])
            regions.append(rgeo.Box(lo, hi))
    per = N // len(regions)
    t0 = time.perf_counter()
    parts, oracles = [], []
    for r, bx in enumerate(regions):
        R = bx.to_polytope()
        lifted = np.hstack([R.A, np.zeros((R.A.shape[0], spec.n - spec.m))])
        Xr = rgeo.Polytope(np.vstack([xd.A, lifted]), np.concatenate([xd.b, R.b]))
        oracles.append(bg.build_oracle(spec, Xr, U, tube))
        bounds = rgeo.Box(np.concatenate([bx.lo, sample.lo[2:]]), np.concatenate([bx.hi, sample.hi[2:]]))
        rng = np.random.default_rng([seed, r])  # graph.py:147-157 with the region's X_d
        got, need = [], per
        while need > 0:
            cand = bounds.sample(rng, need)
            acc = cand[Xr.contains_many(cand)]
            if acc.size:
                got.append(acc)
                need -= acc.shape[0]
        parts.append(np.vstack(got)[:per])
    start = np.array([0.4, 0.4, 0.0, 0.0])
    goal = np.array([side - 0.4, side - 0.4, 0.0, 0.0])
    V = np.vstack(parts + [np.array([start, goal])])
    Vn = V.shape[0]
    keys = []
    for bx, o in zip(regions, oracles):
        inside = np.nonzero(np.all((V[:, :2] >= bx.lo - 1e-6) & (V[:, :2] <= bx.hi + 1e-6), axis=1))[0]
        I, Jx = np.meshgrid(inside, inside, indexing="ij")
        I, Jx = I.ravel(), Jx.ravel()
        ok = (I != Jx) & bg.reachability.check_edges(o, V[I], V[Jx])
        keys.append(I[ok].astype(np.int64) * Vn + Jx[ok])
    keys = np.unique(np.concatenate(keys))
    E = np.stack([keys // Vn, keys % Vn], axis=1).astype(np.int64)
    D = bg.bezier.boundary_matrix(spec)
    x1 = V[E[:, 0]].reshape(-1, spec.gamma, spec.m)
    x2 = V[E[:, 1]].reshape(-1, spec.gamma, spec.m)
    pts = np.einsum("pq,eqm->emp", D, np.concatenate([x1, x2], axis=1))  # graph.py:192-197
    costs = np.linalg.norm(np.diff(pts, axis=2), axis=1).sum(axis=1)
    t_build = time.perf_counter() - t0
    g = rg.BezierGraph(spec=spec, oracle=base, vertices=V, edges=E, costs=costs, edge_points=pts, seed=seed,
                       sample_bounds=sample)
    print(f"cfg5_10k: V={Vn} E={E.shape[0]} built in {t_build:.1f}s", flush=True)
    rng = np.random.default_rng(seed + 100)
    obs = [rgeo.inflate(o, tube.position_box(2)) for o in _clear_boxes(rng, 50, 0.4, side - 0.4, start, goal)]
    cfg = rg.CutConfig()
    t0 = time.perf_counter()
    mask, (po, pe, st, it, dl) = recorded_cut(g, obs, cfg)
    t_cut = time.perf_counter() - t0
    t0 = time.perf_counter()
    path = rg.find_path(g, mask, start, goal)
    t_path = time.perf_counter() - t0
    np.savez_compressed(
        OUT / "cfg5_10k.npz", N=N, N_per=per, seed=seed, side=side, V=Vn, E=E.shape[0],
        region_lo=np.stack([b.lo for b in regions]), region_hi=np.stack([b.hi for b in regions]),
        F_base=base.F, G_base=base.G, start=start, goal=goal,
        obs_n=np.array([o.num_rows for o in obs], np.int32), obs_A=np.concatenate([o.A for o in obs]),
        obs_b=np.concatenate([o.b for o in obs]),
        sha_vertices=digest(V), sha_edges=digest(E), sha_costs=digest(costs), sha_points=digest(pts),
        vertices=V, row_counts=np.bincount(E[:, 0], minlength=Vn).astype(np.int64),
        alive=mask.alive.copy(), provenance=np.array([PROV[p.value] for p in mask.provenance], np.int8),
        counters=np.array([mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp,
                           mask.qp_safe, mask.qp_unsafe], np.int64),
        qp_obstacle=po, qp_edge=pe, qp_status=st, qp_iters=it, qp_delta=dl,
        path=np.array(path if path is not None else [], np.int64), path_none=path is None,
        path_cost=rg.path_cost(g, path) if path else 0.0, t_build=t_build, t_cut=t_cut, t_path=t_path,
        env=json.dumps(env_info()))
    print(f"cfg5_10k: alive={mask.alive_count} qp={mask.pairs_qp} path={path} cut={t_cut:.1f}s", flush=True)


def case_m3g3():
    """m = 3, gamma = 3 (n = 9): snapping's full-state norm takes numpy's pairwise order (n >= 8),
    plus 3-D degree-5 edges through the whole path; several goals exercise the snap."""
    spec = bg.BezierSpec(m=3, gamma=3, T=1.0)
    side = 2.0
    lo = np.concatenate([np.zeros(3), np.full(3, -1.5), np.full(3, -4.0)])
    hi = np.concatenate([np.full(3, side), np.full(3, 1.5), np.full(3, 4.0)])
    xd = rgeo.Box(lo, hi).to_polytope()
    u = rgeo.Box(np.full(3, -30.0), np.full(3, 30.0))
    tube = rsim.design_tube(spec, (6.0, 11.0, 6.0), 0.02)
    oracle = bg.build_oracle(spec, xd, u, tube)
    slo = np.concatenate([np.zeros(3), np.full(3, -0.3), np.full(3, -0.5)])
    shi = np.concatenate([np.full(3, side), np.full(3, 0.3), np.full(3, 0.5)])
    sample = rgeo.Box(slo, shi)
    rng = np.random.default_rng(12)
    obs = []
    for _ in range(4):
        c = rng.uniform(0.5, side - 0.5, 3)
        sd = rng.uniform(0.2, 0.4, 3)
        obs.append(rgeo.inflate(rgeo.Box(c - sd / 2, c + sd / 2).to_polytope(), tube.position_box(3)))
    start = np.concatenate([np.full(3, 0.15), np.zeros(6)])
    goal = np.concatenate([np.full(3, side - 0.15), np.zeros(6)])
    goals = np.zeros((24, 9))
    goals[:, :3] = rng.uniform(0.15, side - 0.15, (24, 3))
    goals[:, 3:] = rng.uniform(-0.3, 0.3, (24, 6))
    capture("m3g3_1500", 1500, spec, oracle, sample, 8, np.array([start, goal]), obs, start, goal, full=True,
            detail=True, goals=goals)


def general_obstacles_big():
    """Convex polygons with 10..32 faces (the paper's segmented obstacles are convex hulls with
    many faces) plus one box, in the demo map."""
    return [
        _regular_polygon((2.5, 2.5), 0.45, 12, 0.3),
        _regular_polygon((1.3, 3.7), 0.35, 32, 0.2),
        _regular_polygon((3.7, 1.3), 0.40, 10, 0.1),
        _regular_polygon((1.2, 1.6), 0.30, 20, 0.0),
        _regular_polygon((3.6, 3.4), 0.38, 16, np.pi / 16),
        rgeo.Box(np.array([2.2, 0.3]), np.array([2.7, 0.9])).to_polytope(),
    ]


def case_general_big():
    """Graph golden with 10..32-face obstacles: the general heuristic and the Cut-QP beyond the
    8-row records (build -> cut -> path with per-QP detail)."""
    s = rsc.demo_scenario()
    oracle = bg.build_oracle(s.spec, s.xd, s.u_bounds, s.tube)
    capture("general_big60", 60, s.spec, oracle, s.sample_bounds, 11, np.array([s.start, s.goal]),
            general_obstacles_big(), s.start, s.goal, full=True, detail=True)


def case_heur_general_big():
    """Scalar cut_heuristic / closest_point / adjacent_hyperplane on 10..32-face polygons."""
    rng = np.random.default_rng(13)
    obs = general_obstacles_big()[:5]
    ctrs = [(2.5, 2.5), (1.3, 3.7), (3.7, 1.3), (1.2, 1.6), (3.6, 3.4)]
    cfg = rg.CutConfig()
    pts_l, oi_l, code_l, proj_l, hp_l = [], [], [], [], []
    for i in range(300):
        oi = i % len(obs)
        O = obs[oi]
        pts = np.asarray(ctrs[oi])[:, None] + rng.uniform(-0.9, 0.9, (2, 1)) + rng.uniform(-0.35, 0.35, (2, 4))
        pts_l.append(pts)
        oi_l.append(oi)
        code_l.append({rg.CutVerdict.UNSAFE: 0, rg.CutVerdict.SAFE: 1, rg.CutVerdict.INDETERMINATE: 2}[
            rg.cut_heuristic(pts, O, cfg)])
        On = O.normalized()
        proj_l.append(np.stack([rgeo.closest_point(On, p) for p in pts.T]))
        try:
            hp = rgeo.adjacent_hyperplane(On, pts[:, 0])
            hp_l.append(np.concatenate([hp.normal, [hp.offset]]))
        except ValueError:
            hp_l.append(np.full(3, np.nan))
    np.savez_compressed(OUT / "heur_general_big.npz", points=np.stack(pts_l), obstacle=np.array(oi_l, np.int32),
                        codes=np.array(code_l, np.int8), projections=np.stack(proj_l), hyperplanes=np.stack(hp_l),
                        obs_n=np.array([o.num_rows for o in obs], np.int32),
                        obs_A=np.concatenate([o.A for o in obs]), obs_b=np.concatenate([o.b for o in obs]),
                        env=json.dumps(env_info()))
    print("heur_general_big:", np.bincount(np.array(code_l), minlength=3))


def case_g4():
    """gamma = 4 (degree 7, snap norm over n = 8 terms -> numpy's pairwise order): 2-D boxes
    through build -> cut -> path."""
    spec = bg.BezierSpec(m=2, gamma=4, T=1.0)
    lo = np.array([0.0, 0.0, -1.5, -1.5, -4.0, -4.0, -20.0, -20.0])
    hi = np.array([5.0, 5.0, 1.5, 1.5, 4.0, 4.0, 20.0, 20.0])
    xd = rgeo.Box(lo, hi).to_polytope()
    u = rgeo.Box(np.full(2, -200.0), np.full(2, 200.0))
    tube = rsim.design_tube(spec, (24.0, 50.0, 35.0, 10.0), 0.02)
    oracle = bg.build_oracle(spec, xd, u, tube)
    sample = rgeo.Box(np.array([0.0, 0.0, -0.5, -0.5, -1.0, -1.0, -2.0, -2.0]),
                      np.array([5.0, 5.0, 0.5, 0.5, 1.0, 1.0, 2.0, 2.0]))
    obs = [rgeo.inflate(rsc._box_obstacle(c[0], c[1], w[0], w[1]).shape, tube.position_box(2))
           for c, w in (((2.5, 2.5), (0.8, 0.8)), ((1.3, 3.6), (0.6, 0.5)), ((3.7, 1.4), (0.5, 0.7)))]
    start = np.array([0.4, 0.4, 0, 0, 0, 0, 0, 0.0])
    goal = np.array([4.6, 4.6, 0, 0, 0, 0, 0, 0.0])
    rng = np.random.default_rng(21)
    goals = np.zeros((16, 8))
    goals[:, :2] = rng.uniform(0.3, 4.7, (16, 2))
    goals[:, 2:4] = rng.uniform(-0.3, 0.3, (16, 2))
    capture("g4_800", 800, spec, oracle, sample, 5, np.array([start, goal]), obs, start, goal, full=True,
            detail=True, goals=goals)


CASES = {"regions4": case_regions4, "general": case_general, "heur_general": case_heur_general, "knn": case_knn,
         "m3": case_m3, "m1": case_m1, "heur_general3": case_heur_general3,
         "regions4gap": lambda: case_regions4("regions4gap", [((0.0, 0.0), (2.4, 2.4)), ((2.6, 0.0), (5.0, 2.4)),
                                                              ((0.0, 2.6), (2.4, 5.0)), ((2.6, 2.6), (5.0, 5.0)),
                                                              ((1.5, 1.5), (3.5, 3.5))]), "demo": case_demo, "rf_small": case_rf_small, "hop_small": case_hop_small, "reject": case_reject,
         "cfg2": case_cfg2, "maze": case_maze, "cfg3": case_cfg3, "cfg5_10k": case_cfg5_10k,
         "m3g3": case_m3g3, "general_big": case_general_big, "heur_general_big": case_heur_general_big,
         "g4": case_g4}

if __name__ == "__main__":
    which = sys.argv[1:] or list(CASES)
    for w in which:
        CASES[w]()
