"""Parity at BASELINE.json's full cfg3 size (20,002 vertices, 4.0e8 ordered pairs, 50 boxes).

The CPU oracle cannot build or cut the whole graph in test time (~1,200 s on one core), so
the full-size run is checked through what does not depend on size:
* vertices bitwise (the oracle sampler is cheap at any size);
* CSR structure: rows non-decreasing, columns strictly increasing inside a row, no self loops;
* bitwise edges, control points and costs on sampled source-row blocks. The oracle's
  ``pair_edges(rows=...)`` restricts the pair test to those rows (the multi-GPU row-block cut);
* the cut on those rows' edges against ``oracle.cut_graph``. The heuristic's pending set is
  bitwise. QP verdict differences must fall in the solver-sensitive class.
  alive/provenance must match on every edge no such difference touches;
* the shortest path: the oracle's heapq Dijkstra on the device's full graph and mask gives the
  same node sequence and the same cost, bitwise.
"""

import numpy as np
import pytest

import oracle
from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import configs
from paper_2411_13507_b200 import graph as G
from paper_2411_13507_b200.bezier import boundary_matrix
from tests.helpers import qp_solver_sensitive

pytestmark = pytest.mark.gpu

ROW_BLOCKS = [(0, 24), (9_990, 10_014), (19_978, 20_002)]  # the last block holds start and goal


@pytest.fixture(scope="module")
def cfg3():
    ctx = nat.Context(0)
    nat.set_default_context(ctx)
    w = configs.BUILDERS["cfg3"]()
    g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    mask = G.cut_graph(g, w.obstacles)
    path = G.find_path(g, mask, w.start, w.goal)
    yield w, g, mask, path
    nat.set_default_context(None)


def _oracle_vertices(w):
    return oracle.sample_states(w.N, w.sample_bounds.lo, w.sample_bounds.hi, w.oracle.Xd.A, w.oracle.Xd.b, w.seed,
                                w.include)


def test_cfg3_vertices_and_csr(cfg3):
    w, g, _, _ = cfg3
    assert g.num_vertices == 20_002 and g.num_edges > 4_000_000
    assert g.vertices.tobytes() == _oracle_vertices(w).tobytes()
    rp, col = g.csr()
    assert rp[0] == 0 and rp[-1] == g.num_edges and np.all(np.diff(rp) >= 0)
    src = np.repeat(np.arange(g.num_vertices), np.diff(rp))
    assert not np.any(src == col)
    same_row = src[1:] == src[:-1]
    assert np.all(col[1:][same_row] > col[:-1][same_row])
    assert np.array_equal(g.edges[:, 0], src) and np.array_equal(g.edges[:, 1], col)


def _block(w, g, V, r0, r1):
    n = w.spec.m * w.spec.gamma
    A1, A2 = oracle.project(V, w.oracle.F, n)
    E = oracle.pair_edges(A1, A2, w.oracle.G, rows=(r0, r1))
    rp, _ = g.csr()
    lo, hi = int(rp[r0]), int(rp[r1])
    return E, lo, hi


@pytest.mark.parametrize("r0,r1", ROW_BLOCKS)
def test_cfg3_row_block_edges_points_costs_bitwise(cfg3, r0, r1):
    w, g, _, _ = cfg3
    V = g.vertices
    E, lo, hi = _block(w, g, V, r0, r1)
    assert E.shape[0] == hi - lo > 0
    assert np.array_equal(g.edges[lo:hi], E)
    pts = oracle.edge_points(V, E, boundary_matrix(w.spec), w.spec.gamma, w.spec.m)
    assert g.edge_points[lo:hi].tobytes() == pts.tobytes()
    assert g.costs[lo:hi].tobytes() == oracle.edge_costs(pts).tobytes()


def test_cfg3_cut_on_row_blocks(cfg3):
    w, g, mask, _ = cfg3
    V = g.vertices
    idx = np.concatenate([np.arange(*_block(w, g, V, r0, r1)[1:]) for r0, r1 in ROW_BLOCKS])
    obstacles = [(o.A, o.b) for o in w.obstacles]
    ref = oracle.cut_graph(g.edge_points[idx], obstacles, record=True)
    # per-(edge, obstacle) QP outcomes of both sides, keyed by (global edge, obstacle)
    keys_r, st_r, it_r, dl_r = [], [], [], []
    for oi, entry in enumerate(ref["log"]):
        if entry["pending"].size:
            keys_r.append(idx[entry["pending"]] * 64 + oi)
            st_r.append(entry["status"]); it_r.append(entry["iters"]); dl_r.append(entry["delta"])
    keys_r = np.concatenate(keys_r)
    rec = mask.qp_records()
    keys_d = rec["edge"].astype(np.int64) * 64 + rec["obstacle"]
    sel = np.isin(rec["edge"], idx)
    keys_d = keys_d[sel]
    od, orr = np.argsort(keys_d), np.argsort(keys_r)
    assert np.array_equal(keys_d[od], keys_r[orr]), "heuristic pending sets differ"
    st_d, it_d, dl_d = (np.asarray(rec[k])[sel][od] for k in ("status", "iterations", "delta"))
    st_r, it_r, dl_r = (np.concatenate(a)[orr] for a in (st_r, it_r, dl_r))
    v_d = (st_d == 0) & (dl_d > 1e-7)
    v_r = (st_r == 0) & (dl_r > 1e-7)
    diff = v_d != v_r
    sens = qp_solver_sensitive(st_d, it_d, dl_d, st_r, it_r, dl_r)
    print(f"cfg3 row blocks: {idx.size} edges, {keys_r.size} QPs, {int(diff.sum())} verdict differences "
          f"({int((diff & sens).sum())} solver-sensitive)")
    assert not np.any(diff & ~sens)
    touched = np.isin(idx, keys_r[orr][diff] // 64)
    assert np.array_equal(mask.alive[idx][~touched], ref["alive"][~touched])
    assert np.array_equal(mask.provenance_codes[idx][~touched], ref["provenance"][~touched])


def test_cfg3_path_matches_oracle_dijkstra(cfg3):
    w, g, mask, path = cfg3
    tube = w.oracle.tube.error
    ref_path, ref_dist = oracle.find_path(g.vertices, g.edges, g.costs, mask.alive, w.start, w.goal, w.spec.m,
                                          tube.lo, tube.hi)
    assert path is not None and ref_path is not None
    assert path == list(ref_path)
    assert G.path_cost(g, path) == float(ref_dist)


def test_cfg3_relaxed_snap_pull_reach(cfg3, monkeypatch):
    """Relaxed mid-run snapping at full size (graph.py:388-392, _reaches_goal 433-450): the
    reverse reachability of a graph this large is pulled bottom-up over the forward CSR
    (k_reach_pull); its snapped start must be the oracle's (reverse DFS on the device's
    graph and mask) and its paths those of the edge-sweep schedule (BZG_REACH_IMPL=grid)."""
    w, g, mask, _ = cfg3
    V = g.vertices
    rng = np.random.default_rng(29)
    kw = dict(position_only_snap=True, require_tube_snap=False)
    cases = [(w.start, w.goal)] + [(V[rng.integers(0, len(V))], V[rng.integers(0, len(V))]) for _ in range(5)]
    tube = w.oracle.tube.error
    for s, t in cases[:2]:
        want = oracle.snap(V, g.edges, mask.alive, s, t, w.spec.m, tube.lo, tube.hi, **kw)
        got = G.find_path(g, mask, s, t, **kw)
        assert (got is None) == (want is None)
        if got is not None:
            assert (got[0], got[-1]) == want
    pull = [G.find_path(g, mask, s, t, **kw) for s, t in cases]
    monkeypatch.setenv("BZG_REACH_IMPL", "grid")

    class Fresh:  # a new device mask: no reach set cached from the pull runs
        alive = mask.alive

    sweeps = [G.find_path(g, Fresh(), s, t, **kw) for s, t in cases]
    assert pull == sweeps
    assert sum(p is not None for p in pull) >= 3


# ---------------------------------------------------------------- the live reference at full size
def _golden_or_skip(name):
    from tests.conftest import GOLDEN, load_golden

    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"golden {name} not captured")
    return load_golden(name)


def test_cfg3_whole_graph_against_live_reference(cfg3):
    """Every array of the headline run against the unmodified reference's own build_graph /
    cut_graph / find_path on the same inputs (tests/golden/make_golden.py case_cfg3): the
    whole 4.5 M-edge graph, all 226 M (edge, obstacle) outcomes, all 1.7 M QPs and the path."""
    import json

    from tests.helpers import assert_cut_parity, compare_cut, digest

    gd = _golden_or_skip("cfg3_hop20k")
    w, g, mask, path = cfg3
    assert g.oracle.F.tobytes() == gd["F"].tobytes() and g.oracle.G.tobytes() == gd["G"].tobytes()
    assert digest(g.vertices) == str(gd["sha_vertices"])
    assert digest(g.edges) == str(gd["sha_edges"])
    assert digest(g.costs) == str(gd["sha_costs"])
    assert np.array_equal(np.diff(g.csr()[0]), gd["row_counts"])
    assert digest(g.edge_points) == str(gd["sha_points"])
    band = g.eps_band(1e-11)
    print("cfg3 eps band", band)
    assert band["band"] == int(gd["eps_band_1e-11"])
    assert g.eps_band(1e-9)["band"] == int(gd["eps_band_1e-9"])
    rep = compare_cut(mask, gd)
    print("cfg3", json.dumps(rep))
    assert_cut_parity(rep)

    class RefMask:  # the reference's own alive mask: the search alone, bitwise
        alive = gd["alive"]

    ref_mask_path = G.find_path(g, RefMask(), w.start, w.goal)
    assert ref_mask_path == list(gd["path"])
    assert G.path_cost(g, ref_mask_path) == float(gd["path_cost"])
    # the device's own mask differs from the reference's only on the few edges of solver-
    # sensitive QPs; dropping edges that are off the reference path cannot change it (the path
    # through the device's own mask is checked against the oracle's Dijkstra separately)
    on_path = set(zip(gd["path"][:-1].tolist(), gd["path"][1:].tolist()))
    e = g.edges
    flip = np.nonzero(mask.alive != gd["alive"])[0]
    gained = bool((mask.alive[flip] & ~gd["alive"][flip]).any())
    if not gained and not any((int(e[k, 0]), int(e[k, 1])) in on_path for k in flip):
        assert path == list(gd["path"])
        assert G.path_cost(g, path) == float(gd["path_cost"])


def test_cfg5_10k_keepin_against_live_reference():
    """BASELINE cfg5 at 10 k nodes (200 keep-in cells, 50 boxes): the device's region graph, cut
    and path against the golden composed from the reference's build_oracle / check_edges /
    cut_graph / find_path (make_golden.py case_cfg5_10k)."""
    import json

    from paper_2411_13507_b200 import regions as R
    from tests.helpers import assert_cut_parity, compare_cut, digest

    gd = _golden_or_skip("cfg5_10k")
    ctx = nat.Context(0)
    w = configs.scaling_sweep(10000)
    lo, hi = R.region_boxes(w.extra["regions"])
    assert lo.tobytes() == gd["region_lo"].tobytes() and hi.tobytes() == gd["region_hi"].tobytes()
    g = R.build_region_graph(w.extra["per_region"], w.spec, w.oracle, w.extra["regions"], w.sample_bounds, w.seed,
                             include=w.include, ctx=ctx)
    assert g.vertices.tobytes() == gd["vertices"].tobytes()
    assert digest(g.edges) == str(gd["sha_edges"])
    assert digest(g.costs) == str(gd["sha_costs"])
    assert digest(g.edge_points) == str(gd["sha_points"])
    mask = G.cut_graph(g, w.obstacles)
    rep = compare_cut(mask, gd)
    print("cfg5_10k", json.dumps(rep))
    assert_cut_parity(rep)
    path = G.find_path(g, mask, w.start, w.goal)
    if rep["verdict_mismatch"] == 0:
        assert path == list(gd["path"])
        assert G.path_cost(g, path) == float(gd["path_cost"])
