"""The reference's OWN pipeline on the device stage (SURVEY.md §4 tier 3).

``shim.install(beziergraph)`` patches ``beziergraph.graph``'s build_graph / cut_graph /
find_path / path_cost / cut_heuristic / cut_qp with this package's device functions; the
unmodified reference simulator (``sim.plan_once``, sim.py:242-272, and
``sim.run_closed_loop``, sim.py:275-408, with its MPC, tracking controller and disturbance
model) then runs on top of them.  Each run is compared with the same call on the unpatched
reference: graph, mask, path, MPC outcome, closed-loop trajectory, cut history and events.

The reference is imported from /root/reference/pkg/src (the build container) or from
baseline/_ref, the unmodified package installed by ``pip install --target baseline/_ref``
(it travels to the GPU box with the repo; __graft_entry__.build() installs it).
"""

import dataclasses
import importlib
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2411_13507_b200 import shim

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CANDIDATES = [Path("/root/reference/pkg/src"), ROOT / "baseline" / "_ref"]


@pytest.fixture(scope="module")
def ref():
    for p in CANDIDATES:
        if (p / "beziergraph" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            return importlib.import_module("beziergraph")
    pytest.skip("the reference package is neither at /root/reference nor in baseline/_ref")


def _patched(ref, fn, *args, cut_cache=0, **kw):
    shim.install(ref, cut_cache=cut_cache)
    try:
        return fn(*args, **kw)
    finally:
        shim.uninstall(ref)


def _prov(mask):
    return np.array([p.value for p in mask.provenance])


def _same_graph(g0, g1):
    assert g1.vertices.tobytes() == g0.vertices.tobytes()
    assert np.array_equal(g1.edges, g0.edges)
    assert g1.costs.tobytes() == g0.costs.tobytes()
    assert g1.edge_points.tobytes() == g0.edge_points.tobytes()


def _same_mask(m0, m1):
    assert np.array_equal(m1.alive, m0.alive)
    assert np.array_equal(_prov(m1), _prov(m0))
    for f in ("pairs_total", "pairs_point_hit", "pairs_hyperplane", "pairs_qp", "qp_safe", "qp_unsafe"):
        assert getattr(m1, f) == getattr(m0, f), f
    assert m1.to_json() == m0.to_json()


def test_plan_once_demo_patched_equals_reference(ref):
    """sim.plan_once(demo_scenario, 200 samples): build -> cut -> find_path on the device, the
    reference's MPC refinement on top; everything equals the unpatched run."""
    s = dataclasses.replace(ref.scenario.demo_scenario(), graph_n=200)
    r0 = ref.sim.plan_once(s)
    r1 = _patched(ref, ref.sim.plan_once, s)
    _same_graph(r0.graph, r1.graph)
    _same_mask(r0.mask, r1.mask)
    assert r1.path == r0.path and r1.path is not None
    assert r1.ok == r0.ok
    assert (r1.solution is None) == (r0.solution is None)
    if r0.solution is not None:
        assert r1.solution.status == r0.solution.status
        # the MPC runs on identical inputs, so its iterates are the same host arithmetic
        assert r1.solution.iterations == r0.solution.iterations
        assert r1.solution.states.tobytes() == r0.solution.states.tobytes()
        assert r1.solution.inputs.tobytes() == r0.solution.inputs.tobytes()
        for a, b in zip(r0.solution.curves, r1.solution.curves):
            assert np.array_equal(a.P, b.P)


def test_plan_once_cfg2_against_live_reference_golden(ref, golden):
    """BASELINE cfg2 through the reference's own plan_once (random_field_scenario(1, 20, 2000)):
    the device graph, mask and path against the golden the unpatched reference produced on the
    same scenario (tests/golden/make_golden.py case_cfg2; the unpatched cut takes ~75 s)."""
    import hashlib

    g = golden("cfg2_rf2000")
    s = ref.scenario.random_field_scenario(1, n_obstacles=20, graph_n=2000)
    r = _patched(ref, ref.sim.plan_once, s)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(r.graph.vertices) == str(g["sha_vertices"])
    assert sha(r.graph.edges) == str(g["sha_edges"])
    assert sha(r.graph.costs) == str(g["sha_costs"])
    assert np.array_equal(r.mask.alive, g["alive"])
    prov = {"heuristic_unsafe": 0, "heuristic_safe": 1, "qp_safe": 2, "qp_unsafe": 3}
    assert np.array_equal(np.array([prov[p.value] for p in r.mask.provenance], np.int8), g["provenance"])
    assert [r.mask.pairs_total, r.mask.pairs_point_hit, r.mask.pairs_hyperplane, r.mask.pairs_qp, r.mask.qp_safe,
            r.mask.qp_unsafe] == [int(x) for x in g["counters"]]
    assert r.path == list(g["path"])
    assert r.ok


def test_closed_loop_moving_obstacle_patched_equals_reference(ref):
    """sim.run_closed_loop with a moving obstacle (ObstacleTrack.at, scenario.py:45-48): a recut
    every 0.1 s on the fixed device graph, relaxed mid-run snapping (position_only_snap,
    require_tube_snap=False -> the device reverse-reachability sweep), the reference MPC and
    simulator.  Trajectory, inputs, cut history, events and final path equal the unpatched run."""
    base = dataclasses.replace(ref.scenario.demo_scenario(), graph_n=200)
    ob = base.obstacles[1]
    moving = ref.scenario.ObstacleTrack(ob.shape, motion=((0.0, np.zeros(2)), (2.0, np.array([0.5, -0.4]))))
    s = dataclasses.replace(base, obstacles=[base.obstacles[0], moving, base.obstacles[2]], timeout=2.0)
    t0 = ref.sim.run_closed_loop(s)
    t1 = _patched(ref, ref.sim.run_closed_loop, s)
    t2 = _patched(ref, ref.sim.run_closed_loop, s, cut_cache=16)  # static obstacles reused
    assert t2.cut_history == t0.cut_history and t2.states.tobytes() == t0.states.tobytes()
    assert t2.final_path == t0.final_path
    assert len(t0.cut_history) == len(t1.cut_history) == 20
    assert t1.cut_history == t0.cut_history
    assert t1.events == t0.events
    assert np.array_equal(t1.times, t0.times)
    assert t1.states.tobytes() == t0.states.tobytes()
    assert t1.inputs.tobytes() == t0.inputs.tobytes()
    assert t1.final_path == t0.final_path
    assert t1.summary() == t0.summary()
    _same_mask(t0.final_mask, t1.final_mask)


def test_to_json_wire_formats_match_reference(ref, golden):
    """BezierGraph.to_json / CutMask.to_json (graph.py:83-88, 115-126): the device objects'
    wire formats equal the reference's on the same graph and mask (demo200 golden)."""
    from paper_2411_13507_b200 import _native as nat
    from paper_2411_13507_b200 import graph as G
    from tests.helpers import inputs_from_golden

    g = golden("demo200")
    N, spec, orc, bounds, seed, include, obstacles, start, goal = inputs_from_golden(g)
    ctx = nat.Context(0)
    gr = G.build_graph(N, spec, orc, bounds, seed, include, ctx=ctx)
    mask = G.cut_graph(gr, obstacles)
    rg = ref.graph
    ref_spec = ref.BezierSpec(int(g["m"]), int(g["gamma"]), float(g["T"]))
    ref_graph = rg.BezierGraph(spec=ref_spec, oracle=None, vertices=g["vertices"].copy(), edges=g["edges"].copy(),
                               costs=g["costs"].copy(), edge_points=g["edge_points"].copy(), seed=int(g["seed"]),
                               sample_bounds=None)
    assert gr.to_json() == ref_graph.to_json()
    assert gr.to_json(max_edges=100) == ref_graph.to_json(max_edges=100)
    names = ["HEURISTIC_UNSAFE", "HEURISTIC_SAFE", "QP_SAFE", "QP_UNSAFE"]
    prov = np.array([getattr(rg.CutProvenance, names[k]) for k in g["provenance"]], dtype=object)
    c = [int(x) for x in g["counters"]]
    ref_mask = rg.CutMask(alive=g["alive"].copy(), provenance=prov, pairs_total=c[0], pairs_point_hit=c[1],
                          pairs_hyperplane=c[2], pairs_qp=c[3], qp_safe=c[4], qp_unsafe=c[5])
    assert mask.to_json() == ref_mask.to_json()


def test_project_on_path_matches_reference(ref, golden):
    """replan.project_on_path (bzg_project_on_path) vs the reference's sim._project_on_path
    (sim.py:220-239) on paths of the demo graph and random vehicle states: the same grid time,
    bit for bit (gamma = 2 and the gamma = 3 hop1500 graph)."""
    from paper_2411_13507_b200 import replan

    rng = np.random.default_rng(3)
    for name, spec_args, hs in (("demo200", (2, 2, 1.0), (0.1, 0.05, 0.2)), ("hop1500", (2, 3, 1.0), (0.1, 0.25))):
        g = golden(name)
        spec = ref.BezierSpec(*spec_args)
        V = g["vertices"]
        path = np.asarray(g["path"], dtype=np.int64)
        n_cases = 0
        for h in hs:
            for L in (1, 2, 3, len(path)):
                states = V[path[:L]]
                for _ in range(12):
                    x = V[rng.integers(0, V.shape[0])] + rng.normal(0, 0.2, V.shape[1])
                    want = ref.sim._project_on_path(states, spec, h, x)
                    got = replan.project_on_path(states, spec, h, x)
                    assert got == want, (name, h, L, got, want)
                    n_cases += 1
        assert n_cases > 50
