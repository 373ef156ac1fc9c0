"""Device parity against the reference goldens and the CPU oracle (run on a B200).

Every call goes through libbzg.so (the C ABI) via the drop-in Python API.
Bit-exact: vertices, edges/CSR, costs, control points, heuristic outcomes,
path node sequences and path costs.  QP-decided pairs: verdict differences
must fall in the solver-sensitive class and are reported.
"""

import json

import numpy as np
import pytest

import oracle
from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import graph as G
from tests.helpers import assert_cut_parity, compare_cut, digest, inputs_from_golden

pytestmark = pytest.mark.gpu

FULL = ["demo200", "rf300_s5", "hop1500", "reject400", "m3_600", "m1_300", "m3g3_1500", "g4_800"]


@pytest.fixture(scope="module")
def ctx():
    c = nat.Context(0)
    nat.set_default_context(c)
    yield c
    nat.set_default_context(None)


def _build(g, ctx):
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    return G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx), obstacles, start, goal


@pytest.mark.parametrize("name", FULL)
def test_build_bitwise(ctx, golden, name):
    g = golden(name)
    gr, *_ = _build(g, ctx)
    assert gr.num_vertices == int(g["V"]) and gr.num_edges == int(g["E"])
    assert gr.vertices.tobytes() == g["vertices"].tobytes()
    assert np.array_equal(gr.edges, g["edges"])
    assert gr.costs.tobytes() == g["costs"].tobytes()
    assert gr.edge_points.tobytes() == g["edge_points"].tobytes()
    rp, col = gr.csr()
    assert np.array_equal(np.diff(rp), np.bincount(g["edges"][:, 0], minlength=gr.num_vertices))
    assert np.array_equal(col, g["edges"][:, 1])


@pytest.mark.parametrize("name", FULL)
def test_cut_and_path(ctx, golden, name):
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)
    mask = G.cut_graph(gr, obstacles)
    rep = compare_cut(mask, g)
    print(name, json.dumps(rep))
    assert_cut_parity(rep)
    path = G.find_path(gr, mask, start, goal)
    if rep["verdict_mismatch"] == 0:
        if bool(g["path_none"]):
            assert path is None
        else:
            assert path == list(g["path"])
            assert G.path_cost(gr, path) == float(g["path_cost"])


def test_path_on_golden_mask(ctx, golden):
    """find_path against the reference's own alive mask: node sequence and cost bitwise."""
    for name in FULL:
        g = golden(name)
        gr, obstacles, start, goal = _build(g, ctx)

        class RefMask:
            alive = g["alive"]

        path = G.find_path(gr, RefMask(), start, goal)
        if bool(g["path_none"]):
            assert path is None
        else:
            assert path == list(g["path"]), name
            assert G.path_cost(gr, path) == float(g["path_cost"])


def test_relaxed_snapping(ctx, golden):
    g = golden("demo200")
    gr, obstacles, start, goal = _build(g, ctx)

    class RefMask:
        alive = g["alive"]

    lens, flat = g["relaxed_path_len"], g["relaxed_paths"]
    off = 0
    for k, st in enumerate(g["relaxed_starts"]):
        p = G.find_path(gr, RefMask(), st, goal, position_only_snap=True, require_tube_snap=False)
        assert (p or []) == list(flat[off:off + lens[k]]), k
        off += lens[k]


def test_cfg2_build_cut_path_and_replanning(ctx, golden):
    g = golden("cfg2_rf2000")
    gr, obstacles, start, goal = _build(g, ctx)
    assert digest(gr.vertices) == str(g["sha_vertices"])
    assert digest(gr.edges) == str(g["sha_edges"])
    assert digest(gr.costs) == str(g["sha_costs"])
    assert digest(gr.edge_points) == str(g["sha_points"])
    mask = G.cut_graph(gr, obstacles)
    rep = compare_cut(mask, g)  # every one of the 106,827 QPs against the live reference's
    print("cfg2", json.dumps(rep))
    assert_cut_parity(rep)
    assert rep["verdict_mismatch"] == 0, rep  # exact on this golden
    assert G.find_path(gr, mask, start, goal) == list(g["path"])

    class RefMask:
        alive = g["alive"]

    path = G.find_path(gr, RefMask(), start, goal)
    assert path == list(g["path"])
    assert G.path_cost(gr, path) == float(g["path_cost"])
    # cfg4: 100 goal updates on the fixed (graph, mask)
    lens, flat = g["goal_path_len"], g["goal_paths"]
    off = 0
    for k, gl in enumerate(g["goals"]):
        p = G.find_path(gr, RefMask(), start, gl)
        assert (p or []) == list(flat[off:off + lens[k]]), k
        if p:
            assert G.path_cost(gr, p) == float(g["goal_costs"][k])
        off += lens[k]


def test_maze_ties(ctx, golden):
    """Grid vertices via include, 424 wall boxes, tied parents: path bitwise on the golden mask."""
    g = golden("maze")
    gr, obstacles, start, goal = _build(g, ctx)
    assert digest(gr.vertices) == str(g["sha_vertices"])
    assert digest(gr.edges) == str(g["sha_edges"])
    assert digest(gr.costs) == str(g["sha_costs"])

    class RefMask:
        alive = g["alive"]

    path = G.find_path(gr, RefMask(), start, goal)
    assert path == list(g["path"])
    mask = G.cut_graph(gr, obstacles)
    rep = compare_cut(mask, g)  # 424 walls, 57,006 QPs
    print("maze", json.dumps(rep))
    assert_cut_parity(rep)
    if rep["verdict_mismatch"] == 0:
        assert G.find_path(gr, mask, start, goal) == list(g["path"])


def test_check_edges_vs_oracle(ctx, golden):
    g = golden("hop1500")
    N, spec, orc, *_ = inputs_from_golden(g)
    rng = np.random.default_rng(0)
    V = g["vertices"]
    i = rng.integers(0, V.shape[0], 20000)
    j = rng.integers(0, V.shape[0], 20000)
    dev = G.check_edges(orc, V[i], V[j], ctx=ctx)
    ref = oracle.check_edges(g["F"], g["G"], spec.n, V[i], V[j])
    assert np.array_equal(dev, ref)
    assert dev.any() and not dev.all()


def test_argument_errors(ctx, golden):
    g = golden("demo200")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    with pytest.raises(ValueError, match="at least two"):
        G.build_graph(1, spec, orc, bounds, seed, ctx=ctx)
    from paper_2411_13507_b200.geometry import Box

    with pytest.raises(ValueError, match="4-dimensional"):
        G.build_graph(10, spec, orc, Box(np.zeros(3), np.ones(3)), seed, ctx=ctx)


def test_edge_cases(ctx, golden):
    g = golden("demo200")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    # N = 2 and start == goal: singleton path
    gr = G.build_graph(2, spec, orc, bounds, seed, include=np.array([start]), ctx=ctx)
    mask = G.cut_graph(gr, [])
    assert mask.pairs_total == 0 and mask.heuristic_fraction == 1.0
    assert G.find_path(gr, mask, start, start) == [2]
    # no obstacles: everything alive, all heuristic-safe
    gr = G.build_graph(200, spec, orc, bounds, seed, include=include, ctx=ctx)
    mask = G.cut_graph(gr, [])
    assert mask.alive.all() and (mask.provenance_codes == 1).all()
    ref = oracle.build_graph(200, spec, orc, bounds, seed, include, D=g["D"])
    assert np.array_equal(gr.edges, ref["edges"])
    # sharded row blocks concatenate to the full edge list
    parts = [G.build_graph(200, spec, orc, bounds, seed, include, ctx=ctx, rows=(a, b))
             for a, b in ((0, 67), (67, 150), (150, 202))]
    cat = np.concatenate([p.edges for p in parts])
    assert np.array_equal(cat, ref["edges"])
    assert np.concatenate([p.costs for p in parts]).tobytes() == ref["costs"].tobytes()


@pytest.mark.parametrize("name", ["hop1500", "rf300_s5", "cfg2_rf2000"])
def test_polish_screen_keeps_verdicts(ctx, golden, name, monkeypatch):
    """The ADMM-norm screen on the polish never changes a cut outcome."""
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)
    monkeypatch.setenv("BZG_POLISH_SCREEN", "0")
    full = G.cut_graph(gr, obstacles)
    monkeypatch.delenv("BZG_POLISH_SCREEN")
    fast = G.cut_graph(gr, obstacles)
    assert np.array_equal(full.alive, fast.alive)
    assert np.array_equal(full.provenance_codes, fast.provenance_codes)
    assert (full.qp_safe, full.qp_unsafe) == (fast.qp_safe, fast.qp_unsafe)
    assert np.array_equal(full.alive, g["alive"])


def test_knn_prefilter(ctx, golden):
    """build_graph(k_nearest=k) on device (k_knn_rows) against the live reference's edges and costs."""
    from tests.test_oracle_golden import _knn_inputs

    g = golden("knn400")
    spec, orc, bounds = _knn_inputs(g)
    for k in g["ks"]:
        gr = G.build_graph(int(g["N"]), spec, orc, bounds, int(g["seed"]), k_nearest=int(k), ctx=ctx)
        assert np.array_equal(gr.edges, g[f"edges_k{k}"]), k
        assert gr.costs.tobytes() == g[f"costs_k{k}"].tobytes(), k
    gr = G.build_graph(int(g["N"]), spec, orc, bounds, int(g["seed"]), k_nearest=0, ctx=ctx)
    assert gr.num_edges == 0
    with pytest.raises(ValueError):
        G.build_graph(int(g["N"]), spec, orc, bounds, int(g["seed"]), k_nearest=-1, ctx=ctx)


def test_obstacle_grid_prescreen_is_exact(ctx, monkeypatch):
    """The spatial obstacle pre-screen (ObsGrid, large maps) leaves every cut outcome unchanged:
    cfg5's 10 k-node keep-in map (50 boxes on a ~11 x 11 map, where the grid is used) cut with
    and without it."""
    from paper_2411_13507_b200 import configs
    from paper_2411_13507_b200 import regions as R

    w = configs.scaling_sweep(10000)
    g = R.build_region_graph(w.extra["per_region"], w.spec, w.oracle, w.extra["regions"], w.sample_bounds, w.seed,
                             include=w.include, ctx=ctx)
    m_grid = G.cut_graph(g, w.obstacles)
    monkeypatch.setenv("BZG_NO_OBS_GRID", "1")
    m_full = G.cut_graph(g, w.obstacles)
    cnt = lambda m: [m.pairs_total, m.pairs_point_hit, m.pairs_hyperplane, m.pairs_qp, m.qp_safe, m.qp_unsafe]  # noqa: E731
    assert cnt(m_grid) == cnt(m_full)
    assert np.array_equal(m_grid.alive, m_full.alive)
    assert np.array_equal(m_grid.provenance_codes, m_full.provenance_codes)


@pytest.mark.parametrize("name", ["cfg2_rf2000", "maze", "hop1500"])
def test_obstacle_window_is_exact(ctx, golden, name, monkeypatch):
    """The sorted x-window of heuristic pass 1 (obstacles farther than the edge's extent
    along x certified code 1 without a test) leaves every cut outcome unchanged."""
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)
    m_win = G.cut_graph(gr, obstacles)
    monkeypatch.setenv("BZG_NO_OBS_WINDOW", "1")
    m_all = G.cut_graph(gr, obstacles)
    cnt = lambda m: [m.pairs_total, m.pairs_point_hit, m.pairs_hyperplane, m.pairs_qp, m.qp_safe, m.qp_unsafe]  # noqa: E731
    assert cnt(m_win) == cnt(m_all)
    assert np.array_equal(m_win.alive, m_all.alive)
    assert np.array_equal(m_win.provenance_codes, m_all.provenance_codes)


@pytest.mark.parametrize("name", ["demo200", "hop1500", "cfg2_rf2000"])
def test_eps_band_counts(ctx, golden, name):
    """North-star eps-band report (bzg_graph_eps_band) against the oracle's count on the same
    vertices, at the reported eps (1e-11) and at widths that make the band non-empty."""
    g = golden(name)
    gr, *_ = _build(g, ctx)
    V = gr.vertices
    A1, A2 = oracle.project(V, g["F"], V.shape[1])
    for eps in (1e-11, 1e-4, 1e-2):
        dev = gr.eps_band(eps)
        band, plus, minus = oracle.eps_band(A1, A2, g["G"], eps)
        assert (dev["band"], dev["feasible_plus"], dev["feasible_minus"]) == (band, plus, minus), (name, eps)
        assert minus <= gr.num_edges <= plus
    if "eps_band_1e-11" in g:
        assert gr.eps_band(1e-11)["band"] == int(g["eps_band_1e-11"])


@pytest.mark.parametrize("name", ["m3g3_1500", "g4_800"])
def test_full_state_snapping_pairwise_norm(ctx, golden, name):
    """n = m*gamma = 9 (m = 3, gamma = 3) and 8 (m = 2, gamma = 4): the full-state snap norm
    follows numpy's pairwise summation (n >= 8), so goal snapping and the resulting paths match
    the live reference on every goal."""
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)

    class RefMask:
        alive = g["alive"]

    lens, flat = g["goal_path_len"], g["goal_paths"]
    off = 0
    for k, gl in enumerate(g["goals"]):
        p = G.find_path(gr, RefMask(), start, gl)
        assert (p or []) == list(flat[off:off + lens[k]]), k
        off += lens[k]


@pytest.mark.parametrize("name", ["rf300_s5", "hop1500", "general60", "m3_600", "m1_300", "cfg2_rf2000"])
def test_admm_schedules_iterates_bitwise(ctx, golden, name, monkeypatch):
    """Every ADMM schedule yields the same iterates: one pass of k_qp_admm (the plain
    persistent kernel), the default tail-compaction passes (AdmmPass: thinned warps park
    their instances and a later launch resumes them densely), aggressive parking
    (BZG_ADMM_DUMP=32: any non-full drained warp parks), and k_qp_admm2 (two lanes per
    instance).  Same status, iteration count and ||delta|| bits for every QP, same mask.
    Covers the canonical box (m = 1, 2, 3 -- odd stored-row count at m = 3), general polygons
    (C = 8) and gamma = 2, 3."""
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)
    variants = {"plain": {"BZG_ADMM_LANES": "1", "BZG_ADMM_PASSES": "1"},
                "compact": {"BZG_ADMM_LANES": "1"},
                "park_all": {"BZG_ADMM_LANES": "1", "BZG_ADMM_PASSES": "4", "BZG_ADMM_DUMP": "32"},
                "two_lane": {"BZG_ADMM_LANES": "2"}}
    out = {}
    for nm, env in variants.items():
        for k in ("BZG_ADMM_LANES", "BZG_ADMM_PASSES", "BZG_ADMM_DUMP"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        m = G.cut_graph(gr, obstacles)
        r = m.qp_records()
        # the work list is appended by warp atomics: compare in (edge, obstacle) order
        o = np.argsort(r["edge"] * 1_000_003 + r["obstacle"], kind="stable")
        out[nm] = (m, {k: v[o] for k, v in r.items()})
    m0, r0 = out["plain"]
    assert r0["status"].size > 0
    for nm, (m, r) in out.items():
        for k in ("edge", "obstacle", "status", "iterations"):
            assert np.array_equal(r0[k], r[k]), (nm, k)
        assert r0["delta"].tobytes() == r["delta"].tobytes(), nm
        assert np.array_equal(m0.alive, m.alive) and np.array_equal(m0.provenance_codes, m.provenance_codes), nm


def _moved(ob, t):
    from paper_2411_13507_b200.geometry import Polytope

    A = np.asarray(ob.A, dtype=np.float64)
    return Polytope(A, np.asarray(ob.b, dtype=np.float64) + A @ np.asarray(t, dtype=np.float64))


def _same_cut(a, b):
    assert np.array_equal(a.alive, b.alive)
    assert np.array_equal(a.provenance_codes, b.provenance_codes)
    ca = [a.pairs_total, a.pairs_point_hit, a.pairs_hyperplane, a.pairs_qp, a.qp_safe, a.qp_unsafe]
    cb = [b.pairs_total, b.pairs_point_hit, b.pairs_hyperplane, b.pairs_qp, b.qp_safe, b.qp_unsafe]
    assert ca == cb, (ca, cb)


@pytest.mark.parametrize("name", ["rf300_s5", "hop1500", "general60", "m3_600"])
def test_recut_cache_equals_full_cut(ctx, golden, name):
    """The re-cut cache (bzg_graph_set_cut_cache): a replanning sequence -- first cut, one obstacle
    moved, obstacles reordered and duplicated, the first list again, a list larger than the cache
    -- gives masks identical to uncached cuts of the same lists (alive, provenance, counters)."""
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)
    ref = G.build_graph(*inputs_from_golden(g)[:6], ctx=ctx)  # same graph, no cache
    m = gr.spec.m
    moved = list(obstacles)
    moved[0] = _moved(obstacles[0], np.full(m, 0.07))
    lists = [list(obstacles), moved, moved[::-1] + moved[:1], list(obstacles)]
    gr.set_cut_cache(len(obstacles) + 2)
    for lst in lists:
        _same_cut(G.cut_graph(gr, lst), G.cut_graph(ref, lst))
    if m == 2:  # a failing cut (an empty obstacle: ValueError) leaves the cache consistent
        from paper_2411_13507_b200.geometry import Polytope

        empty = Polytope(np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]]), np.array([0.0, -1.0, 1.0]))
        with pytest.raises(ValueError):
            G.cut_graph(gr, [_moved(obstacles[0], np.full(m, 0.03)), empty])
        lst = [_moved(obstacles[0], np.full(m, 0.03))] + list(obstacles[1:])
        _same_cut(G.cut_graph(gr, lst), G.cut_graph(ref, lst))
    big = list(obstacles) + [_moved(o, np.full(m, -0.05)) for o in obstacles]  # larger than the cache
    _same_cut(G.cut_graph(gr, big), G.cut_graph(ref, big))
    _same_cut(G.cut_graph(gr, moved), G.cut_graph(ref, moved))
    gr.set_cut_cache(0)
    _same_cut(G.cut_graph(gr, moved), G.cut_graph(ref, moved))


@pytest.mark.parametrize("impl", ["queue", "scan", "async", "cluster", "cta"])
@pytest.mark.parametrize("name", ["cfg2_rf2000", "maze", "hop1500"])
def test_bellman_ford_variants_reach_the_reference_paths(ctx, golden, name, impl, monkeypatch):
    """Every Bellman-Ford schedule (frontier queue, rescan, barrier-free asynchronous, single
    thread-block cluster, one block in shared memory) reaches the
    same fixed point: the paths (and costs) through the reference's own mask are the golden's,
    and so are the cfg4 goal updates (cfg2)."""
    monkeypatch.setenv("BZG_BF_IMPL", impl)
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)

    class RefMask:
        alive = g["alive"]

    path = G.find_path(gr, RefMask(), start, goal)
    assert path == (None if bool(g["path_none"]) else list(g["path"]))
    if path:
        assert G.path_cost(gr, path) == float(g["path_cost"])
    if "goals" in g:
        lens, flat = g["goal_path_len"], g["goal_paths"]
        off = 0
        for k, gl in enumerate(g["goals"][:40]):
            p = G.find_path(gr, RefMask(), start, gl)
            assert (p or []) == list(flat[off:off + lens[k]]), k
            off += lens[k]


@pytest.mark.parametrize("cs", [1, 2, 4, 8, 16])
def test_bellman_ford_cluster_sizes(ctx, golden, cs, monkeypatch):
    """k_bf_cluster at every cluster size (the owned slices, DSMEM relaxations and the cluster
    barrier schedule change with it): the golden paths of cfg2 and its goal updates."""
    monkeypatch.setenv("BZG_BF_IMPL", "cluster")
    monkeypatch.setenv("BZG_BF_CLUSTER", str(cs))
    g = golden("cfg2_rf2000")
    gr, obstacles, start, goal = _build(g, ctx)

    class RefMask:
        alive = g["alive"]

    assert G.find_path(gr, RefMask(), start, goal) == list(g["path"])
    lens, flat = g["goal_path_len"], g["goal_paths"]
    off = 0
    for k, gl in enumerate(g["goals"][:20]):
        assert (G.find_path(gr, RefMask(), start, gl) or []) == list(flat[off:off + lens[k]]), k
        off += lens[k]


def test_edge_cases_round2(ctx, golden):
    """Degenerate inputs of the round-2 entry points: empty obstacle lists under the re-cut cache,
    an unreachable goal (None) and start == goal through the one-sync search, eps_band on a
    row block, project_on_path on 0/1-state paths."""
    from paper_2411_13507_b200 import replan

    g = golden("demo200")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    gr = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
    gr.set_cut_cache(8)
    m0 = G.cut_graph(gr, [])
    assert m0.alive.all() and m0.pairs_total == 0
    m1 = G.cut_graph(gr, obstacles)
    m2 = G.cut_graph(gr, obstacles)  # all hits
    assert np.array_equal(m1.alive, m2.alive) and m1.qp_safe == m2.qp_safe and m2.pairs_qp == m1.pairs_qp
    assert np.array_equal(m1.alive, g["alive"])
    # start == goal -> [v]; a goal whose snapped vertex has no alive in-edges -> None

    class NoEdges:
        alive = np.zeros(gr.num_edges, dtype=bool)

    assert G.find_path(gr, NoEdges(), start, start) == [N]
    assert G.find_path(gr, NoEdges(), start, goal) is None
    # eps band of a row block = its share of the whole
    rb = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx, rows=(0, 101))
    rb2 = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx, rows=(101, N + 2))
    full = gr.eps_band(1e-3)
    a, b = rb.eps_band(1e-3), rb2.eps_band(1e-3)
    assert a["band"] + b["band"] == full["band"] and a["feasible_plus"] + b["feasible_plus"] == full["feasible_plus"]
    # project_on_path: no hop -> 0
    assert replan.project_on_path(np.zeros((0, spec.n)), spec, 0.1, start) == 0.0
    assert replan.project_on_path(start[None], spec, 0.1, start) == 0.0


@pytest.mark.parametrize("name", ["demo200", "maze", "cfg2_rf2000", "hop1500"])
def test_reverse_reachability_schedules(ctx, golden, name, monkeypatch):
    """Relaxed mid-run snapping (graph.py:388-392, _reaches_goal 433-450): the reverse
    reachability by cooperative grid sweeps, by one thread-block cluster and pulled bottom-up
    over the forward CSR (k_reach_pull) give the same
    snapped starts and paths, for many starts and goals."""
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)

    class RefMask:
        alive = g["alive"]

    rng = np.random.default_rng(17)
    V = gr.vertices
    cases = [(start, goal)] + [(V[rng.integers(0, len(V))], V[rng.integers(0, len(V))]) for _ in range(12)]
    out = {}
    for impl in ("grid", "cluster", "pull"):
        monkeypatch.setenv("BZG_REACH_IMPL", impl)
        out[impl] = [G.find_path(gr, RefMask(), s, t, position_only_snap=True, require_tube_snap=False)
                     for s, t in cases]
    assert out["grid"] == out["cluster"] == out["pull"]
    assert sum(p is not None for p in out["grid"]) >= 2


@pytest.mark.parametrize("name", ["demo200", "hop1500", "m3g3_1500", "cfg2_rf2000"])
def test_snap_block_equals_grid_snap(ctx, golden, name, monkeypatch):
    """The one-block snap of small graphs (k_snap_block) picks the same vertices as the grid
    snap (k_snap + k_snap_final): goal and tube / relaxed start, targets at vertices, between
    two vertices (exact ties) and far away."""
    g = golden(name)
    gr, obstacles, start, goal = _build(g, ctx)

    class RefMask:
        alive = g["alive"]

    V = gr.vertices
    rng = np.random.default_rng(23)
    cases = [(start, goal)]
    for _ in range(10):
        a, b = V[rng.integers(0, len(V))], V[rng.integers(0, len(V))]
        cases += [(a, b), ((a + b) / 2, b), (a, (a + b) / 2), (a + 50.0, b)]
    out = {}
    for impl in ("grid", "block"):
        if impl == "grid":
            monkeypatch.setenv("BZG_SNAP_GRID", "1")
        else:
            monkeypatch.delenv("BZG_SNAP_GRID", raising=False)
        res = []
        for s, t in cases:
            res.append(G.find_path(gr, RefMask(), s, t))
            res.append(G.find_path(gr, RefMask(), s, t, position_only_snap=True, require_tube_snap=False))
        out[impl] = res
    assert out["grid"] == out["block"]
