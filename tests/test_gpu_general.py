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


@pytest.mark.parametrize("name", ["heur_general", "heur_general3", "heur_general_big"])
def test_cut_heuristic_general_vs_reference(ctx, golden, name):
    from tests.conftest import GOLDEN

    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"golden {name} not captured")
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


@pytest.mark.parametrize("kind", ["box", "rotated", "hexagon", "20-gon", "32-gon"])
def test_cut_qp_vs_oracle(ctx, kind):
    rng = np.random.default_rng(7)
    if kind == "box":
        poly = Box(np.array([1.0, 1.0]), np.array([2.0, 1.6])).to_polytope()
    else:
        k = {"rotated": 4, "hexagon": 6, "20-gon": 20, "32-gon": 32}[kind]
        ang = 0.35 + 2 * np.pi * np.arange(k) / k
        A = np.stack([np.cos(ang), np.sin(ang)], axis=1) * 2.5
        poly = Polytope(A, A @ np.array([1.5, 1.3]) + 0.5 * 2.5)
    P = _random_sets(rng, 300, 4, np.array([1.5, 1.3]), 1.3, 0.5)
    safe, delta, status = G.cut_qp_batch(P, [poly], None, ctx=ctx)
    st, it, dl = _oracle_cut_qp(P, poly)
    v_ref = (st == 0) & (dl > 1e-7)
    from tests.helpers import qp_solver_sensitive

    sens = qp_solver_sensitive(st, it, dl, status, it, delta)
    print(kind, "status equal", float((status == st).mean()), "safe", int(safe.sum()), "sensitive", int(sens.sum()))
    assert not np.any((safe != v_ref) & ~sens)
    ok = (status == 0) & (st == 0)
    assert np.allclose(delta[ok], dl[ok], rtol=1e-6, atol=1e-7)
    assert (status == st).mean() > 0.97
    # scalar drop-in
    s0, d0 = G.cut_qp(P[0], poly)
    assert s0 == bool(safe[0]) and d0 == float(delta[0])


@pytest.mark.parametrize("name", ["general60", "general_big60"])
def test_general_graph_vs_reference(ctx, golden, name):
    """build -> cut -> path with general polygons against the live reference: 3..8 faces
    (general60) and 10..32 faces (general_big60: the kObsRowsBig records and a C = 32 Cut-QP)."""
    from tests.conftest import GOLDEN

    if not (GOLDEN / f"{name}.npz").exists():
        pytest.skip(f"golden {name} not captured")
    g = golden(name)
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    gr = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
    assert gr.edge_points.tobytes() == g["edge_points"].tobytes()
    mask = G.cut_graph(gr, obstacles)
    rep = compare_cut(mask, g)
    print(name, json.dumps(rep))
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


def _polygon(center, radius, k, phase):
    ang = phase + 2 * np.pi * np.arange(k) / k
    A = np.stack([np.cos(ang), np.sin(ang)], axis=1) * 1.7
    return Polytope(A, A @ np.asarray(center, float) + radius * 1.7)


def test_general_errors(ctx):
    pts = np.array([[3.0, 3.2, 3.4, 3.6], [0.0, 0.1, 0.2, 0.3]])
    empty = Polytope(np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0]]), np.array([0.0, -1.0, 1.0]))
    with pytest.raises(ValueError):
        G.cut_heuristic(pts, empty)
    ang = 2 * np.pi * np.arange(33) / 33
    many = Polytope(np.stack([np.cos(ang), np.sin(ang)], axis=1), np.ones(33))
    with pytest.raises(nat.BzgError) as e:
        G.cut_heuristic(pts, many)
    assert e.value.code == nat.BZG_EUNSUPPORTED


def test_gamma4_build_cut_path_vs_oracle(ctx):
    """gamma = 4 (degree-7 curves, n = 8: the snap norm takes numpy's pairwise order) through
    build -> cut (boxes: heuristic + Cut-QP with J = 8) -> path, against the CPU oracle."""
    from paper_2411_13507_b200 import configs
    from paper_2411_13507_b200.bezier import BezierSpec, boundary_matrix
    from paper_2411_13507_b200.geometry import inflate
    from paper_2411_13507_b200.reachability import build_oracle
    from tests.helpers import qp_solver_sensitive

    spec = BezierSpec(m=2, gamma=4, T=1.0)
    xd = Box(np.array([0.0, 0.0, -1.5, -1.5, -4.0, -4.0, -20.0, -20.0]),
             np.array([5.0, 5.0, 1.5, 1.5, 4.0, 4.0, 20.0, 20.0])).to_polytope()
    U = Box(np.full(2, -200.0), np.full(2, 200.0))
    tube = configs.design_tube(spec, (24.0, 50.0, 35.0, 10.0), 0.02)
    orc = build_oracle(spec, xd, U, tube)
    sample = Box(np.array([0.0, 0.0, -0.5, -0.5, -1.0, -1.0, -2.0, -2.0]), np.array([5.0, 5.0, 0.5, 0.5, 1.0, 1.0, 2.0, 2.0]))
    obs = [inflate(Box(np.array([2.1, 2.1]), np.array([2.9, 2.9])).to_polytope(), tube.position_box(2)),
           inflate(Box(np.array([1.0, 3.3]), np.array([1.6, 3.8])).to_polytope(), tube.position_box(2))]
    start = np.array([0.4, 0.4, 0, 0, 0, 0, 0, 0.0])
    goal = np.array([4.6, 4.6, 0, 0, 0, 0, 0, 0.0])
    inc = np.array([start, goal])
    gr = G.build_graph(800, spec, orc, sample, 5, inc, ctx=ctx)
    ref = oracle.build_graph(800, spec, orc, sample, 5, inc, D=boundary_matrix(spec))
    assert gr.vertices.tobytes() == ref["vertices"].tobytes()
    assert np.array_equal(gr.edges, ref["edges"]) and gr.num_edges > 1000  # 1,508 at this seed
    assert gr.costs.tobytes() == ref["costs"].tobytes()
    assert gr.edge_points.tobytes() == ref["edge_points"].tobytes()
    mask = G.cut_graph(gr, obs)
    cut = oracle.cut_graph(ref["edge_points"], [(o.A, o.b) for o in obs], record=True)
    assert [mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp] == \
        [cut["pairs_total"], cut["pairs_point_hit"], cut["pairs_hyperplane"], cut["pairs_qp"]]
    assert mask.pairs_qp > 0
    rec = mask.qp_records()
    kd = rec["edge"] * 64 + rec["obstacle"]
    kr, st_r, it_r, dl_r = [], [], [], []
    for oi, entry in enumerate(cut["log"]):
        if entry["pending"].size:
            kr.append(entry["pending"] * 64 + oi)
            st_r.append(entry["status"]); it_r.append(entry["iters"]); dl_r.append(entry["delta"])
    kr = np.concatenate(kr)
    od, orr = np.argsort(kd), np.argsort(kr)
    assert np.array_equal(kd[od], kr[orr])
    st_r, it_r, dl_r = (np.concatenate(a)[orr] for a in (st_r, it_r, dl_r))
    st_d, it_d, dl_d = rec["status"][od], rec["iterations"][od], rec["delta"][od]
    diff = ((st_d == 0) & (dl_d > 1e-7)) != ((st_r == 0) & (dl_r > 1e-7))
    assert not np.any(diff & ~qp_solver_sensitive(st_d, it_d, dl_d, st_r, it_r, dl_r))
    path = G.find_path(gr, mask, start, goal)
    rpath, rdist = oracle.find_path(gr.vertices, gr.edges, gr.costs, mask.alive, start, goal, 2, tube.error.lo,
                                    tube.error.hi)
    assert path == (list(rpath) if rpath is not None else None)
