"""General (non-box) obstacles and the scalar cut entry points on device.

* cut_heuristic on explicit control points (graph.py:202-221) vs the live reference's codes
  (tests/golden/heur_general.npz) and vs the oracle on box obstacles;
* cut_qp (graph.py:285-299) vs the oracle's dense ADMM + polish;
* a whole build -> cut -> path on a graph with 3..8-row obstacles (tests/golden/general60.npz).

The projection QPs inside the general heuristic run the reference's ADMM settings in a
reduced (Cholesky) form, so this row's parity class is the epsilon band: codes must agree
except where the reference's own decision sits within solver noise of a threshold.
"""

import json

import numpy as np
import pytest

import oracle
from oracle.qp_ref import AdmmSettings, cut_qp_problem, solve_dense_batch
from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import graph as G
from paper_2411_13507_b200.geometry import Box, Polytope
from tests.helpers import compare_cut, inputs_from_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = nat.Context(0)
    nat.set_default_context(c)
    yield c
    nat.set_default_context(None)


def _golden_polytopes(g):
    off = np.concatenate([[0], np.cumsum(g["obs_n"])])
    return [Polytope(g["obs_A"][off[i]:off[i + 1]], g["obs_b"][off[i]:off[i + 1]]) for i in range(len(g["obs_n"]))]


@pytest.mark.parametrize("name", ["heur_general", "heur_general3"])
def test_cut_heuristic_general_vs_reference(ctx, golden, name):
    g = golden(name)
    obs = _golden_polytopes(g)
    codes = G.cut_heuristic_batch(g["points"], obs, g["obstacle"], ctx=ctx)
    mism = np.nonzero(codes != g["codes"])[0]
    print(name, "codes", np.bincount(codes, minlength=3), "mismatch", mism.tolist())
    assert mism.size == 0
    for i in range(0, 40, 7):  # the scalar drop-in agrees with the batch
        v = G.cut_heuristic(g["points"][i], obs[int(g["obstacle"][i])])
        assert v == (G.CutVerdict.UNSAFE, G.CutVerdict.SAFE, G.CutVerdict.INDETERMINATE)[int(g["codes"][i])]


def _random_sets(rng, n, J, centre, spread, jitter):
    base = centre[None, :, None] + rng.uniform(-spread, spread, (n, 2, 1))
    return base + rng.uniform(-jitter, jitter, (n, 2, J))


@pytest.mark.parametrize("J", [2, 4, 6])
def test_cut_heuristic_boxes_vs_oracle(ctx, J):
    """Box obstacles through the scalar path (contains_many, clamp projection,
    adjacent_hyperplane): bit-for-bit the oracle's codes."""
    rng = np.random.default_rng(J)
    boxes = [Box(np.array([1.0, 1.0]), np.array([2.0, 1.5])), Box(np.array([-0.5, 0.2]), np.array([0.0, 0.3]))]
    polys = [b.to_polytope() for b in boxes] + [Polytope(np.array([[2.0, 0.0], [0.0, 3.0], [-1.0, 0.0], [0.0, -0.5]]),
                                                         np.array([4.0, 4.5, -1.0, -0.5]))]
    P = _random_sets(rng, 600, J, np.array([1.2, 1.0]), 1.2, 0.4)
    idx = rng.integers(0, len(polys), 600).astype(np.int32)
    codes = G.cut_heuristic_batch(P, polys, idx, ctx=ctx)
    ref = np.array([oracle.graph_ref.cut_heuristic(P[i], polys[k].A, polys[k].b) for i, k in enumerate(idx)])
    assert np.array_equal(codes, ref), np.nonzero(codes != ref)[0][:10]
    assert set(np.unique(ref)) >= {0, 1}


def _oracle_cut_qp(P, poly):
    OA, Ob = oracle.graph_ref.normalized(poly.A, poly.b)
    probs = [cut_qp_problem(P[i], OA, Ob) for i in range(P.shape[0])]
    Pm, q, A, lo, hi = (np.stack([p[k] for p in probs]) for k in range(5))
    x, st, it = solve_dense_batch(Pm, q, A, lo, hi, AdmmSettings())
    J = P.shape[2]
    delta = np.linalg.norm(x[:, J:], axis=1)
    return st, it, delta


@pytest.mark.parametrize("kind", ["box", "rotated", "hexagon"])
def test_cut_qp_vs_oracle(ctx, kind):
    rng = np.random.default_rng(7)
    if kind == "box":
        poly = Box(np.array([1.0, 1.0]), np.array([2.0, 1.6])).to_polytope()
    else:
        k = 4 if kind == "rotated" else 6
        ang = 0.35 + 2 * np.pi * np.arange(k) / k
        A = np.stack([np.cos(ang), np.sin(ang)], axis=1) * 2.5
        poly = Polytope(A, A @ np.array([1.5, 1.3]) + 0.5 * 2.5)
    P = _random_sets(rng, 300, 4, np.array([1.5, 1.3]), 1.3, 0.5)
    safe, delta, status = G.cut_qp_batch(P, [poly], None, ctx=ctx)
    st, it, dl = _oracle_cut_qp(P, poly)
    v_ref = (st == 0) & (dl > 1e-7)
    sens = (st == 1) | (status == 1) | (np.abs(dl - 1e-7) < 1e-8)
    print(kind, "status equal", float((status == st).mean()), "safe", int(safe.sum()), "sensitive", int(sens.sum()))
    assert not np.any((safe != v_ref) & ~sens)
    ok = (status == 0) & (st == 0)
    assert np.allclose(delta[ok], dl[ok], rtol=1e-6, atol=1e-7)
    assert (status == st).mean() > 0.97
    # scalar drop-in
    s0, d0 = G.cut_qp(P[0], poly)
    assert s0 == bool(safe[0]) and d0 == float(delta[0])


def test_general_graph_vs_reference(ctx, golden):
    g = golden("general60")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    gr = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
    assert gr.edge_points.tobytes() == g["edge_points"].tobytes()
    mask = G.cut_graph(gr, obstacles)
    rep = compare_cut(mask, g)
    print("general60", json.dumps(rep))
    assert rep["same_pending"], rep
    assert rep["counters_dev"][:4] == rep["counters_ref"][:4]
    assert rep["mismatch_outside_sensitive"] == 0, rep
    assert rep["alive_mismatch_untouched"] == 0 and rep["prov_mismatch_untouched"] == 0, rep
    path = G.find_path(gr, mask, start, goal)
    if rep["verdict_mismatch"] == 0:
        assert np.array_equal(mask.alive, g["alive"])
        if bool(g["path_none"]):
            assert path is None
        else:
            assert path == list(g["path"])


def test_general_errors(ctx):
    pts = np.array([[3.0, 3.2, 3.4, 3.6], [0.0, 0.1, 0.2, 0.3]])
    empty = Polytope(np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]]), np.array([0.0, -1.0, 1.0]))
    with pytest.raises(ValueError):
        G.cut_heuristic(pts, empty)
    ang = 2 * np.pi * np.arange(9) / 9
    nine = Polytope(np.stack([np.cos(ang), np.sin(ang)], axis=1), np.ones(9))
    with pytest.raises(nat.BzgError) as e:
        G.cut_heuristic(pts, nine)
    assert e.value.code == nat.BZG_EUNSUPPORTED
