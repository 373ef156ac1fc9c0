"""PathQuery (bzg_query): find_path captured as one CUDA graph, replayed with new start/goal.

Every query answer must equal ``find_path`` with the same options on the same graph and mask
(reference graph.py:353-430): node sequence and cost, for tube snapping, relaxed mid-run
snapping (position_only_snap, require_tube_snap=False -> the reverse-reachability sweep), no
mask, unreachable goals (None), a cached tree (repeated start) and alternating starts.
"""

import ctypes as C

import numpy as np
import pytest

from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import graph as G
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
    return gr, G.cut_graph(gr, obstacles), np.asarray(start, float), np.asarray(goal, float)


def _queries(gr, start, goal, rng, k=24):
    """(start, goal) pairs: the golden's, repeated starts (tree cache), alternating starts,
    vertices as targets, and far-away points (snapping still finds a vertex)."""
    V = gr.vertices
    pairs = [(start, goal), (start, goal)]
    for i in range(k):
        s = start if i % 3 == 0 else V[rng.integers(0, len(V))] + rng.normal(0, 0.05, V.shape[1])
        t = V[rng.integers(0, len(V))] + rng.normal(0, 0.05, V.shape[1])
        pairs.append((s, t))
    pairs.append((start, V[0] + 100.0))
    return pairs


@pytest.mark.parametrize("name", ["demo200", "hop1500", "rf300_s5"])
@pytest.mark.parametrize("mode", ["tube", "relaxed", "no_mask"])
def test_query_equals_find_path(ctx, golden, name, mode):
    gr, mask, start, goal = _scene(ctx, golden, name)
    rng = np.random.default_rng(11)
    m = None if mode == "no_mask" else mask
    kw = dict(position_only_snap=True, require_tube_snap=False) if mode == "relaxed" else {}
    q = G.PathQuery(gr, m, **kw)
    assert q.kernels_per_query >= 6
    n_paths = 0
    for s, t in _queries(gr, start, goal, rng):
        want = G.find_path(gr, m, s, t, **kw)
        want_cost = gr._cache.get("last_dist")
        got = q(s, t)
        assert got == want, (s, t)
        if want is not None:
            assert gr._cache["last_dist"] == want_cost
            n_paths += 1
    assert n_paths >= 2
    q.close()


def test_query_cfg2_moving_start(ctx):
    """BASELINE cfg2 (V = 2002: the rescan Bellman-Ford) with alternating starts, as cfg4."""
    from paper_2411_13507_b200 import configs

    w = configs.BUILDERS["cfg2"]()
    gr = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
    mask = G.cut_graph(gr, w.obstacles)
    goals = configs.replanning_goals(w, 30)
    near = np.argsort(np.linalg.norm(gr.vertices - np.asarray(w.start), axis=1))
    starts = [np.asarray(w.start, float), gr.vertices[int(near[1])].copy()]
    q = G.PathQuery(gr, mask)
    found = 0
    for k, gl in enumerate(goals):
        want = G.find_path(gr, mask, starts[k % 2], gl)
        got = q(starts[k % 2], gl)
        assert got == want
        found += want is not None
    assert found >= 10


def test_query_stale_after_edge_change(ctx, golden):
    gr, mask, start, goal = _scene(ctx, golden, "demo200")
    q = G.PathQuery(gr, None)
    assert q(start, goal) == G.find_path(gr, None, start, goal)
    e = np.ascontiguousarray(gr.edges.astype(np.int32))
    c = np.ascontiguousarray(gr.costs)
    src, dst = np.ascontiguousarray(e[:, 0]), np.ascontiguousarray(e[:, 1])
    nat.check(ctx.lib.bzg_graph_set_edges(gr._h, C.c_int64(len(c)), nat.ptr(src), nat.ptr(dst), nat.ptr(c), 0))
    with pytest.raises(ValueError, match="stale query"):
        q(start, goal)
    q.close()
