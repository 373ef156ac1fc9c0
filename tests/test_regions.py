"""Keep-in free regions (configs 1 and 5): host composition, CPU oracle and device build
against goldens composed from the live reference (tests/golden/make_golden.py regions4*)."""

import numpy as np
import pytest

import oracle.regions_ref as RR
from paper_2411_13507_b200 import configs
from paper_2411_13507_b200 import regions as R
from paper_2411_13507_b200.bezier import boundary_matrix
from paper_2411_13507_b200.geometry import Box

CASES = ["regions4", "regions4gap"]


def _setup(g):
    w = configs.demo(200)  # standard sets, tube (6, 5), w_max 0.02 -- the golden's inputs
    regions = [Box(np.array(lo), np.array(hi)).to_polytope() for lo, hi in g["quads"]]
    return w, regions


@pytest.mark.parametrize("name", CASES)
def test_region_oracles_match_reference(golden, name):
    g = golden(name)
    w, regions = _setup(g)
    ors = R.region_oracles(w.spec, w.oracle.Xd, w.oracle.U, w.oracle.tube, regions)
    for o, F, G in zip(ors, g["F_regions"], g["G_regions"]):
        assert o.F.tobytes() == F.tobytes() and o.G.tobytes() == G.tobytes()
    rr = R.region_rows(w.oracle, ors)
    n = w.spec.n
    for F in rr.F:  # added rows are one-sided (position rows of a minimal-degree curve)
        assert np.all(np.all(F[:, :n] == 0, 1) | np.all(F[:, n:] == 0, 1))


@pytest.mark.parametrize("name", CASES)
def test_region_oracle_port_bitwise(golden, name):
    g = golden(name)
    w, regions = _setup(g)
    sets = [R.region_state_set(w.oracle.Xd, reg, w.spec.n) for reg in regions]
    bnds = [R.region_sample_bounds(reg, w.sample_bounds, w.spec.m) for reg in regions]
    V = RR.sample_regions(int(g["N_per"]), [(s.A, s.b) for s in sets], [(b.lo, b.hi) for b in bnds], int(g["seed"]))
    V = np.vstack([V, np.array([g["start"], g["goal"]])])
    assert V.tobytes() == g["vertices"].tobytes()
    out = RR.build_region_graph(V, list(zip(g["F_regions"], g["G_regions"])), boundary_matrix(w.spec), 2, 2)
    assert np.array_equal(out["edges"], g["edges"])
    assert out["costs"].tobytes() == g["costs"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_region_graph_device_bitwise(golden, name):
    from paper_2411_13507_b200 import _native as nat

    g = golden(name)
    w, regions = _setup(g)
    ctx = nat.Context(0)
    gr = R.build_region_graph(int(g["N_per"]), w.spec, w.oracle, regions, w.sample_bounds, int(g["seed"]),
                              include=np.array([g["start"], g["goal"]]), ctx=ctx)
    assert gr.vertices.tobytes() == g["vertices"].tobytes()
    assert np.array_equal(gr.edges, g["edges"])
    assert gr.costs.tobytes() == g["costs"].tobytes()
    assert gr.edge_points.tobytes() == g["edge_points"].tobytes()


@pytest.mark.gpu
def test_region_graph_cut_and_path_vs_oracle(golden):
    """cfg1 keep-in graph (regions4) through the rest of the path: the demo's three boxes cut on
    the device against the oracle's cut of the golden's control points (codes, QP verdicts within
    the solver-sensitive class), then the search against the oracle's heapq Dijkstra."""
    import oracle
    from paper_2411_13507_b200 import _native as nat
    from paper_2411_13507_b200 import graph as G
    from tests.helpers import qp_solver_sensitive

    g = golden("regions4")
    w, regions = _setup(g)
    ctx = nat.Context(0)
    gr = R.build_region_graph(int(g["N_per"]), w.spec, w.oracle, regions, w.sample_bounds, int(g["seed"]),
                              include=np.array([g["start"], g["goal"]]), ctx=ctx)
    mask = G.cut_graph(gr, w.obstacles)
    ref = oracle.cut_graph(g["edge_points"], [(o.A, o.b) for o in w.obstacles], record=True)
    assert [mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp] == \
        [ref["pairs_total"], ref["pairs_point_hit"], ref["pairs_hyperplane"], ref["pairs_qp"]]
    rec = mask.qp_records()
    kd = rec["edge"] * 64 + rec["obstacle"]
    kr, st_r, it_r, dl_r = [], [], [], []
    for oi, entry in enumerate(ref["log"]):
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
    if not diff.any():
        assert np.array_equal(mask.alive, ref["alive"])
        assert np.array_equal(mask.provenance_codes, ref["provenance"])
    tube = w.oracle.tube.error
    path = G.find_path(gr, mask, g["start"], g["goal"])
    rpath, _ = oracle.find_path(g["vertices"], g["edges"], g["costs"], mask.alive, g["start"], g["goal"], 2, tube.lo,
                                tube.hi)
    assert path == (list(rpath) if rpath is not None else None)
