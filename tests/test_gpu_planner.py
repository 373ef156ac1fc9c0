"""Planner (bzg_planner): build -> cut -> find_path of one scene captured as one CUDA graph.

Each call must equal the eager ``build_graph`` + ``cut_graph`` + ``find_path`` on the same
seed, included vertices, obstacles, start and goal: vertices, edges, costs, alive set,
provenance, counters, path and cost -- and, on the golden seed, the live reference's golden.
"""

import numpy as np
import pytest

from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import graph as G
from paper_2411_13507_b200.geometry import Polytope
from paper_2411_13507_b200.plan import Planner
from tests.helpers import inputs_from_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = nat.Context(0)
    nat.set_default_context(c)
    yield c
    nat.set_default_context(None)


def _moved(ob, shift):
    A = np.asarray(ob.A, float)
    return Polytope(A, np.asarray(ob.b, float) + A @ np.asarray(shift, float))


def _eager(ctx, N, spec, orc, bounds, seed, include, obstacles, start, goal, kw):
    g = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
    m = G.cut_graph(g, obstacles)
    p = G.find_path(g, m, start, goal, **kw)
    return g, m, p, g._cache.get("last_dist")


def _check(pl, eager, path):
    g0, m0, p0, d0 = eager
    assert path == p0
    if p0 is not None:
        assert pl.last_dist == d0[1]
    g1, m1 = pl.result()
    assert g1.num_edges == g0.num_edges == pl.num_edges
    assert g1.vertices.tobytes() == g0.vertices.tobytes()
    assert np.array_equal(g1.edges, g0.edges)
    assert g1.costs.tobytes() == g0.costs.tobytes()
    assert np.array_equal(m1.alive, m0.alive)
    assert np.array_equal(m1.provenance_codes, m0.provenance_codes)
    assert list(pl.counters) == [m0.pairs_total, m0.pairs_point_hit, m0.pairs_hyperplane, m0.pairs_qp, m0.qp_safe,
                                 m0.qp_unsafe]


@pytest.mark.parametrize("name", ["demo200", "rf300_s5", "hop1500", "m3_600", "cfg2_rf2000"])
@pytest.mark.parametrize("relaxed", [False, True])
def test_planner_equals_eager_pipeline(ctx, golden, name, relaxed):
    gd = golden(name)
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(gd)
    kw = dict(position_only_snap=True, require_tube_snap=False) if relaxed else {}
    obstacles = list(obstacles)
    pl = Planner(N, spec, orc, bounds, obstacles, seed=seed, include=include, **kw)
    # the golden's own call: the live reference's vertices, edges, costs and alive set
    path = pl(seed, obstacles, start, goal, include=include)
    g1, m1 = pl.result()
    if "edges" in gd:
        assert g1.vertices.tobytes() == gd["vertices"].tobytes()
        assert np.array_equal(g1.edges, gd["edges"])
        assert g1.costs.tobytes() == gd["costs"].tobytes()
    else:  # (cfg2's golden keeps digests)
        from tests.helpers import digest

        assert digest(g1.edges) == str(gd["sha_edges"]) and digest(g1.costs) == str(gd["sha_costs"])
    assert np.array_equal(m1.alive, gd["alive"])
    _check(pl, _eager(ctx, N, spec, orc, bounds, seed, include, obstacles, start, goal, kw), path)
    rng = np.random.default_rng(7)
    for k in range(3):  # new seeds, moved obstacles, new start / goal rows
        s2 = int(seed) + 1 + k
        obstacles[k % len(obstacles)] = _moved(obstacles[k % len(obstacles)], rng.normal(0, 0.05, spec.m))
        inc2 = np.asarray(include, float) + rng.normal(0, 0.02, np.shape(include))
        path = pl(s2, obstacles, inc2[0], inc2[-1], include=inc2)
        _check(pl, _eager(ctx, N, spec, orc, bounds, s2, inc2, obstacles, inc2[0], inc2[-1], kw), path)
    info = pl.info()
    assert info["calls"] == 4 and info["eager_calls"] == 0 and info["kernels_per_call"] >= 25, info
    pl.close()


def test_planner_shape_change_reruns_eagerly(ctx, golden):
    gd = golden("demo200")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(gd)
    obstacles = list(obstacles)
    pl = Planner(N, spec, orc, bounds, obstacles, seed=seed, include=include)
    ang = np.linspace(0, 2 * np.pi, 7)[:-1]
    nrm = np.stack([np.cos(ang), np.sin(ang)], 1)
    hexagon = Polytope(nrm, 0.3 + nrm @ [2.0, 2.5])
    mixed = obstacles[:-1] + [hexagon]
    path = pl(seed, mixed, start, goal, include=include)
    assert pl.last_eager
    _check(pl, _eager(ctx, N, spec, orc, bounds, seed, include, mixed, start, goal, {}), path)
    path = pl(seed + 1, mixed, start, goal, include=include)
    assert not pl.last_eager
    _check(pl, _eager(ctx, N, spec, orc, bounds, seed + 1, include, mixed, start, goal, {}), path)
    with pytest.raises(ValueError, match="obstacle count"):
        pl(seed, obstacles[:-1], start, goal, include=include)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg5"])
def test_planner_keep_in_regions(ctx, cfg):
    """Keep-in regions (configs 1 and 5, regions.build_region_graph): the captured single-round
    region sampler and the region rows uploaded once give the eager pipeline's graph, mask and
    path for several seeds."""
    import bench
    from paper_2411_13507_b200 import regions as RG

    w = bench.workload(cfg, 10000)
    regs, per = w.extra["regions"], w.extra["per_region"]
    obstacles = list(w.obstacles)
    pl = Planner(None, w.spec, w.oracle, w.sample_bounds, obstacles, seed=w.seed, include=w.include,
                 regions=regs, per_region=per)
    rng = np.random.default_rng(3)
    for k in range(3):
        seed = w.seed + k
        if k:
            obstacles[k % len(obstacles)] = _moved(obstacles[k % len(obstacles)], rng.normal(0, 0.05, w.spec.m))
        path = pl(seed, obstacles, w.start, w.goal, include=w.include)
        g0 = RG.build_region_graph(per, w.spec, w.oracle, regs, w.sample_bounds, seed, include=w.include, ctx=ctx)
        m0 = G.cut_graph(g0, obstacles)
        p0 = G.find_path(g0, m0, w.start, w.goal)
        _check(pl, (g0, m0, p0, g0._cache.get("last_dist")), path)
    info = pl.info()
    assert info["calls"] == 3 and info["eager_calls"] == 0, info


def test_planner_edge_cases(ctx, golden):
    """No obstacles, no included vertices, an unreachable goal (None), start == goal."""
    gd = golden("demo200")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(gd)
    pl = Planner(N, spec, orc, bounds, [], seed=seed)  # no include rows, no obstacles
    path = pl(seed + 3, [], start, goal)
    g0 = G.build_graph(N, spec, orc, bounds, seed + 3, None, ctx=ctx)
    m0 = G.cut_graph(g0, [])
    _check(pl, (g0, m0, G.find_path(g0, m0, start, goal), g0._cache.get("last_dist")), path)
    far = np.asarray(goal, float) + 1e3  # snaps to the farthest corner vertex; compare with eager
    path = pl(seed + 3, [], start, far)
    assert path == G.find_path(g0, m0, start, far)
    same = pl(seed + 3, [], start, start)
    assert same == G.find_path(g0, m0, start, start)
    with pytest.raises(ValueError, match="includes"):
        Planner(N, spec, orc, bounds, obstacles, seed=seed, include=include)(seed, obstacles, start, goal)
    assert pl.info()["eager_calls"] == 0


@pytest.mark.parametrize("cfg", ["cfg1-demo", "cfg1"])
def test_planner_fallbacks_equal_eager(ctx, cfg, monkeypatch):
    """BZG_PLAN_STRESS=1 captures with a sampler round and an edge capacity far too small: every
    call's check fails (sampler short / edge capacity), runs the checked eager path on the
    plan's own objects and re-captures -- with the eager API's results."""
    import bench
    from paper_2411_13507_b200 import regions as RG

    monkeypatch.setenv("BZG_PLAN_STRESS", "1")
    w = bench.workload(cfg)
    kw = {}
    if w.extra.get("regions"):
        kw = dict(regions=w.extra["regions"], per_region=w.extra["per_region"])
    obstacles = list(w.obstacles)
    pl = Planner(w.N, w.spec, w.oracle, w.sample_bounds, obstacles, seed=w.seed, include=w.include, **kw)
    for k in range(3):
        seed = w.seed + k
        path = pl(seed, obstacles, w.start, w.goal, include=w.include)
        assert pl.last_eager
        if kw:
            g0 = RG.build_region_graph(kw["per_region"], w.spec, w.oracle, kw["regions"], w.sample_bounds, seed,
                                       include=w.include, ctx=ctx)
        else:
            g0 = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, seed, w.include, ctx=ctx)
        m0 = G.cut_graph(g0, obstacles)
        _check(pl, (g0, m0, G.find_path(g0, m0, w.start, w.goal), g0._cache.get("last_dist")), path)
    info = pl.info()
    assert info["eager_calls"] == 3 and info["last_eager_reason"] in ("sampler round short", "edge capacity"), info
