"""Replanner (bzg_replanner): the cut + find_path cycle of a replanning loop captured as one CUDA
graph (sim.py:324-330 re-cut, graph.py:302-430 cut_graph / find_path).

Every cycle must equal the eager ``cut_graph`` + ``find_path`` on the same obstacles, start and
goal: alive set, provenance, counters, path and its cost -- while obstacles move, while the
obstacle-grid bounds change, when the list changes shape (eager cycle, re-capture) and when the
QP work list outgrows the captured capacity (eager cycle, re-capture).
"""

import numpy as np
import pytest

from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import graph as G
from paper_2411_13507_b200.geometry import Polytope
from paper_2411_13507_b200.replan import Replanner
from tests.helpers import inputs_from_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = nat.Context(0)
    nat.set_default_context(c)
    yield c
    nat.set_default_context(None)


def _scene(ctx, golden, name):
    g = golden(name)
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    gr = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
    return gr, list(obstacles), np.asarray(start, float), np.asarray(goal, float)


def _moved(ob, shift):
    A = np.asarray(ob.A, float)
    return Polytope(A, np.asarray(ob.b, float) + A @ np.asarray(shift, float))


def _same(gr, rp, obstacles, s, t, kw):
    got = rp(obstacles, s, t)
    got_cost = gr._cache.get("last_dist")
    mask = G.cut_graph(gr, obstacles)
    want = G.find_path(gr, mask, s, t, **kw)
    assert got == want
    if want is not None:
        assert got_cost == gr._cache["last_dist"]
    m = rp.mask()
    assert np.array_equal(m.alive, mask.alive)
    assert np.array_equal(m.provenance_codes, mask.provenance_codes)
    assert list(rp.counters) == [mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp,
                                 mask.qp_safe, mask.qp_unsafe]
    return want


@pytest.mark.parametrize("name", ["demo200", "rf300_s5", "maze", "cfg2_rf2000", "m3_600", "m1_300"])
@pytest.mark.parametrize("relaxed", [False, True])
def test_replanner_moving_obstacle(ctx, golden, name, relaxed):
    gr, obstacles, start, goal = _scene(ctx, golden, name)
    kw = dict(position_only_snap=True, require_tube_snap=False) if relaxed else {}
    rp = Replanner(gr, obstacles, **kw)
    rng = np.random.default_rng(5)
    V = gr.vertices
    found = 0
    for k in range(8):
        i = k % len(obstacles)
        obstacles[i] = _moved(obstacles[i], rng.normal(0, 0.05, gr.spec.m))
        s = start if k % 2 == 0 else V[rng.integers(0, len(V))]
        found += _same(gr, rp, obstacles, s, goal, kw) is not None
    info = rp.info()
    assert info["cycles"] == 8 and info["eager_cycles"] == 0 and info["kernels_per_cycle"] >= 10
    assert found >= 1 or bool(golden(name)["path_none"])  # some scenes have no path at all
    rp.close()


@pytest.mark.parametrize("name", ["general60", "general_big60"])
def test_replanner_general_obstacles(ctx, golden, name):
    """General (non-box) polytopes, up to 8 and up to 32 rows: the general screen, its work list
    and the Cut-QP with the large obstacle records in the capture."""
    gr, obstacles, start, goal = _scene(ctx, golden, name)
    rp = Replanner(gr, obstacles)
    for k in range(4):
        obstacles[k] = _moved(obstacles[k], [0.03 * (k + 1), -0.02])
        _same(gr, rp, obstacles, start, goal, {})
    assert rp.info()["eager_cycles"] == 0


def test_replanner_shape_change_and_overflow(ctx, golden):
    """A box that becomes a hexagon changes the list's shape: that cycle runs eagerly and the
    graph is re-captured; obstacles moved from far away into the graph overflow the captured QP
    capacity: eager cycle, re-capture, and the next cycle uses the graph again."""
    gr, obstacles, start, goal = _scene(ctx, golden, "cfg2_rf2000")
    partial = obstacles[:1] + [_moved(ob, [50.0, 50.0]) for ob in obstacles[1:]]  # a few QPs only
    rp = Replanner(gr, partial)
    _same(gr, rp, partial, start, goal, {})
    assert not rp.last_eager
    _same(gr, rp, obstacles, start, goal, {})  # thousands of QPs where the capture saw none
    assert rp.last_eager
    _same(gr, rp, obstacles, start, goal, {})
    assert not rp.last_eager
    ang = np.linspace(0, 2 * np.pi, 7)[:-1]
    hexagon = Polytope(np.stack([np.cos(ang), np.sin(ang)], 1), 0.3 + np.stack([np.cos(ang), np.sin(ang)], 1) @ [2.5, 2.5])
    mixed = obstacles[:-1] + [hexagon]
    _same(gr, rp, mixed, start, goal, {})
    assert rp.last_eager
    _same(gr, rp, mixed, start, goal, {})
    assert not rp.last_eager
    info = rp.info()
    assert info["eager_cycles"] == 2 and info["captures"] == 3
    with pytest.raises(ValueError, match="obstacle count"):
        rp(obstacles[:-1], start, goal)


@pytest.mark.parametrize("name", ["demo200", "maze", "cfg2_rf2000", "general_big60"])
def test_replanner_static_dynamic_split(ctx, golden, name):
    """Static obstacles cut once (outcome rows kept), the dynamic ones every cycle, the mask
    rebuilt in list order: equal to the eager full cut every cycle, also when a static obstacle
    is changed (its rows are re-cut; the captured graph stays in use)."""
    gr, obstacles, start, goal = _scene(ctx, golden, name)
    n = len(obstacles)
    moving = [1 % n, (n // 2) % n] if n > 2 else [0]
    dynamic = np.zeros(n, bool)
    dynamic[moving] = True
    rp = Replanner(gr, obstacles, dynamic=dynamic, position_only_snap=True, require_tube_snap=False)
    kw = dict(position_only_snap=True, require_tube_snap=False)
    rng = np.random.default_rng(9)
    for k in range(6):
        i = moving[k % len(moving)]
        obstacles[i] = _moved(obstacles[i], rng.normal(0, 0.04, gr.spec.m))
        if k == 3 and n > 2:  # a static obstacle changes once
            j = next(o for o in range(n) if not dynamic[o])
            obstacles[j] = _moved(obstacles[j], [0.02] * gr.spec.m)
        _same(gr, rp, obstacles, start, goal, kw)
        assert not rp.last_eager
    assert rp.info()["eager_cycles"] == 0
