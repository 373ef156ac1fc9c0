"""Pin the CPU oracle (oracle/, a numpy restatement of the reference) to golden
vectors captured from the live reference (tests/golden/make_golden.py).

Bitwise: vertices, edges, costs, control points, per-obstacle heuristic codes,
QP status/iterations/||delta||, alive, provenance, counters, path and its cost.
"""

import numpy as np
import pytest

import oracle
from oracle.qp_ref import AdmmSettings
from tests.helpers import digest, inputs_from_golden

FULL = ["demo200", "rf300_s5", "hop1500", "reject400", "m3_600", "m1_300", "m3g3_1500", "g4_800"]


@pytest.mark.parametrize("name", FULL)
def test_build_bitwise(golden, name):
    g = golden(name)
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    out = oracle.build_graph(N, spec, orc, bounds, seed, include, D=g["D"])
    assert out["vertices"].tobytes() == g["vertices"].tobytes()
    assert np.array_equal(out["edges"], g["edges"])
    assert out["costs"].tobytes() == g["costs"].tobytes()
    assert out["edge_points"].tobytes() == g["edge_points"].tobytes()
    assert digest(out["edges"]) == str(g["sha_edges"])


@pytest.mark.parametrize("name", FULL)
def test_cut_and_path_bitwise(golden, name):
    g = golden(name)
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    pts = g["edge_points"]
    res = oracle.cut_graph(pts, [(o.A, o.b) for o in obstacles], settings=AdmmSettings(), record=True)
    assert np.array_equal(res["alive"], g["alive"])
    assert np.array_equal(res["provenance"], g["provenance"])
    cnt = [res[k] for k in ("pairs_total", "pairs_point_hit", "pairs_hyperplane", "pairs_qp", "qp_safe", "qp_unsafe")]
    assert cnt == list(g["counters"])
    codes = np.stack([e["codes"] for e in res["log"]])
    assert np.array_equal(codes, g["codes"])
    st = np.concatenate([e.get("status", np.zeros(0, np.int8)) for e in res["log"]])
    it = np.concatenate([e.get("iters", np.zeros(0, np.int64)) for e in res["log"]])
    dl = np.concatenate([e.get("delta", np.zeros(0)) for e in res["log"]])
    assert np.array_equal(st, g["qp_status"])
    assert np.array_equal(it, g["qp_iters"])
    assert dl.tobytes() == g["qp_delta"].tobytes()
    path, dist = oracle.find_path(g["vertices"], g["edges"], g["costs"], res["alive"], start, goal, spec.m,
                                  g["tube_lo"], g["tube_hi"])
    if bool(g["path_none"]):
        assert path is None
    else:
        assert path == list(g["path"])
        assert dist == float(g["path_cost"])
        assert oracle.path_cost(g["edges"], g["costs"], path) == float(g["path_cost"])


def test_relaxed_snapping(golden):
    g = golden("demo200")
    spec_m = int(g["m"])
    lens = g["relaxed_path_len"]
    flat = g["relaxed_paths"]
    off = 0
    for k, st in enumerate(g["relaxed_starts"]):
        path, _ = oracle.find_path(g["vertices"], g["edges"], g["costs"], g["alive"], st, g["goal"], spec_m,
                                   g["tube_lo"], g["tube_hi"], position_only_snap=True, require_tube_snap=False)
        want = list(flat[off:off + lens[k]])
        off += lens[k]
        assert (path or []) == want


def test_cfg2_build_digests(golden):
    """cfg2 (2,002 vertices, 249,437 edges): build digests and Dijkstra on the golden mask."""
    g = golden("cfg2_rf2000")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    out = oracle.build_graph(N, spec, orc, bounds, seed, include, D=g["D"])
    assert digest(out["vertices"]) == str(g["sha_vertices"])
    assert digest(out["edges"]) == str(g["sha_edges"])
    assert digest(out["costs"]) == str(g["sha_costs"])
    assert digest(out["edge_points"]) == str(g["sha_points"])
    path, dist = oracle.find_path(out["vertices"], out["edges"], out["costs"], g["alive"], start, goal, spec.m,
                                  g["tube_lo"], g["tube_hi"])
    assert path == list(g["path"]) and dist == float(g["path_cost"])
    # cfg4: the first 10 replanning goals on the fixed map
    lens, flat = g["goal_path_len"], g["goal_paths"]
    off = 0
    for k in range(10):
        p, _ = oracle.find_path(out["vertices"], out["edges"], out["costs"], g["alive"], start, g["goals"][k],
                                spec.m, g["tube_lo"], g["tube_hi"])
        assert (p or []) == list(flat[off:off + lens[k]])
        off += lens[k]


def test_check_edges_matches_pair_test(golden):
    g = golden("demo200")
    V, E = g["vertices"], g["edges"]
    n = V.shape[1]
    ok = oracle.check_edges(g["F"], g["G"], n, V[E[:, 0]], V[E[:, 1]])
    assert ok.all()


def _golden_obstacles(g):
    off = np.concatenate([[0], np.cumsum(g["obs_n"])])
    return [(g["obs_A"][off[i]:off[i + 1]], g["obs_b"][off[i]:off[i + 1]]) for i in range(len(g["obs_n"]))]


@pytest.mark.parametrize("name", ["heur_general", "heur_general3"])
def test_general_heuristic_bitwise(golden, name):
    """Scalar cut_heuristic / closest_point / adjacent_hyperplane on non-box polytopes
    (graph.py:202-221, geometry.py:202-252), m = 2 and 3, against the live reference (a
    subset: each projection is a 20000-iteration-capped ADMM in numpy)."""
    g = golden(name)
    obs = _golden_obstacles(g)
    gr = oracle.graph_ref
    for i in range(0, len(g["codes"]), 8):
        A, b = obs[int(g["obstacle"][i])]
        pts = g["points"][i]
        assert gr.cut_heuristic(pts, A, b) == int(g["codes"][i]), i
        OA, Ob = gr.normalized(A, b)
        proj = np.stack([gr.closest_point(OA, Ob, p) for p in pts.T])
        assert proj.tobytes() == g["projections"][i].tobytes(), i
        try:
            n, o = gr.adjacent_hyperplane(OA, Ob, pts[:, 0])
            hp = np.concatenate([n, [o]])
        except ValueError:
            hp = np.full(g["hyperplanes"].shape[1], np.nan)
        assert np.array_equal(hp, g["hyperplanes"][i], equal_nan=True), i


def _knn_inputs(g):
    from types import SimpleNamespace

    from paper_2411_13507_b200.bezier import BezierSpec
    from paper_2411_13507_b200.geometry import Box, Polytope

    spec = BezierSpec(int(g["m"]), int(g["gamma"]), float(g["T"]))
    orc = SimpleNamespace(F=g["F"], G=g["G"], Xd=Polytope(g["xd_A"], g["xd_b"]))
    return spec, orc, Box(g["bounds_lo"], g["bounds_hi"])


def test_knn_prefilter_bitwise(golden):
    """k_nearest prefilter (graph.py:162-170) against the live reference."""
    g = golden("knn400")
    spec, orc, bounds = _knn_inputs(g)
    for k in g["ks"]:
        out = oracle.build_graph(int(g["N"]), spec, orc, bounds, int(g["seed"]), D=np.eye(4), k_nearest=int(k))
        assert np.array_equal(out["edges"], g[f"edges_k{k}"]), k


def test_eps_band_oracle_matches_live_reference_count(golden):
    """The oracle's eps-band count equals the one the golden script computed from the live
    reference's own F, G and vertices (cfg2: no pair within 1e-9 of a threshold)."""
    import oracle
    from tests.helpers import inputs_from_golden

    g = golden("cfg2_rf2000")
    N, spec, orc, *_ = inputs_from_golden(g)
    A1, A2 = oracle.project(g["vertices"], g["F"], spec.n)
    for eps, key in ((1e-11, "eps_band_1e-11"), (1e-9, "eps_band_1e-9")):
        band, plus, minus = oracle.eps_band(A1, A2, g["G"], eps)
        assert band == int(g[key])
        assert minus <= int(g["E"]) <= plus
