"""Randomised scenes beyond the goldens: random output dimension m (1..3), curve order
gamma (1..3), horizon T, state/input sets, box obstacles and seeds.  The device path is
compared with the oracle (itself pinned bitwise to the live reference by
test_oracle_golden.py): vertices, edges, costs, control points, per-obstacle heuristic
codes and the QP pending set bitwise; QP verdicts up to the solver-sensitive class; the
path whenever no verdict differs.
"""

import numpy as np
import pytest

import oracle
from oracle.qp_ref import AdmmSettings
from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import graph as G
from paper_2411_13507_b200.bezier import BezierSpec
from paper_2411_13507_b200.configs import design_tube
from paper_2411_13507_b200.geometry import Box, Polytope, inflate
from paper_2411_13507_b200.reachability import build_oracle
from tests.helpers import qp_solver_sensitive

pytestmark = pytest.mark.gpu

GAINS = {1: (5.0,), 2: (6.0, 5.0), 3: (6.0, 11.0, 6.0)}
DERIV = {0: (0.0, 5.0), 1: (-1.5, 1.5), 2: (-4.0, 4.0)}      # X_d per derivative order
SAMPLE = {0: (0.0, 5.0), 1: (-0.6, 0.6), 2: (-1.0, 1.0)}


@pytest.fixture(scope="module")
def ctx():
    c = nat.Context(0)
    nat.set_default_context(c)
    yield c
    nat.set_default_context(None)


def _scene(seed):
    rng = np.random.default_rng(1000 + seed)
    m, gamma = 1 + seed % 3, 1 + (seed // 3) % 3  # every (m, gamma) in 1..3 x 1..3
    spec = BezierSpec(m, gamma, float(rng.choice([0.5, 1.0, 1.5])))
    lo = np.concatenate([np.full(m, DERIV[k][0]) for k in range(gamma)])
    hi = np.concatenate([np.full(m, DERIV[k][1]) for k in range(gamma)])
    xd = Box(lo, hi).to_polytope()
    if seed % 3 == 1:  # a non-box state set: one extra coupled position row
        row = np.zeros(spec.n)
        row[: min(m, 2)] = 1.0
        xd = Polytope(np.vstack([xd.A, row]), np.concatenate([xd.b, [7.5]]))
    umax = {1: 6.0, 2: 6.0, 3: 30.0}[gamma]
    U = Box(np.full(m, -umax), np.full(m, umax))
    tube = design_tube(spec, GAINS[gamma], 0.02)
    orc = build_oracle(spec, xd, U, tube)
    s_lo = np.concatenate([np.full(m, SAMPLE[k][0]) for k in range(gamma)])
    s_hi = np.concatenate([np.full(m, SAMPLE[k][1]) for k in range(gamma)])
    sample = Box(s_lo, s_hi)
    obstacles = []
    for _ in range(int(rng.integers(3, 9))):
        c = rng.uniform(0.8, 4.2, m)
        w = rng.uniform(0.2, 0.8, m)
        obstacles.append(inflate(Box(c - w / 2, c + w / 2).to_polytope(), tube.position_box(m)))
    start = np.zeros(spec.n)
    goal = np.zeros(spec.n)
    start[:m] = 0.25
    goal[:m] = 4.75
    return spec, orc, sample, obstacles, start, goal, int(rng.integers(0, 2**31))


@pytest.mark.parametrize("seed", range(9))
def test_random_scene_matches_oracle(ctx, seed):
    spec, orc, sample, obstacles, start, goal, gseed = _scene(seed)
    N = 220
    include = np.array([start, goal])
    gr = G.build_graph(N, spec, orc, sample, gseed, include, ctx=ctx)
    ref = oracle.build_graph(N, spec, orc, sample, gseed, include)
    assert gr.vertices.tobytes() == ref["vertices"].tobytes()
    assert np.array_equal(gr.edges, ref["edges"])
    assert gr.costs.tobytes() == ref["costs"].tobytes()
    assert gr.edge_points.tobytes() == ref["edge_points"].tobytes()
    mask = G.cut_graph(gr, obstacles)
    rc = oracle.cut_graph(ref["edge_points"], [(o.A, o.b) for o in obstacles], settings=AdmmSettings(), record=True)
    dev = [mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp]
    assert dev == [rc["pairs_total"], rc["pairs_point_hit"], rc["pairs_hyperplane"], rc["pairs_qp"]]
    # per-instance QP verdicts: identical outside the solver-sensitive class
    rec = mask.qp_records()
    dk = rec["edge"].astype(np.int64) * 4096 + rec["obstacle"]
    o_e, o_o, o_st, o_it, o_dl = [], [], [], [], []
    for oi, entry in enumerate(rc["log"]):
        if entry["pending"].size:
            o_e.append(entry["pending"])
            o_o.append(np.full(entry["pending"].size, oi))
            o_st.append(entry["status"])
            o_it.append(entry["iters"])
            o_dl.append(entry["delta"])
    if o_e:
        ok_ = np.concatenate(o_e).astype(np.int64) * 4096 + np.concatenate(o_o)
        di, oi_ = np.argsort(dk, kind="stable"), np.argsort(ok_, kind="stable")
        assert np.array_equal(dk[di], ok_[oi_])
        st_o, it_o, dl_o = (np.concatenate(x)[oi_] for x in (o_st, o_it, o_dl))
        st_d, it_d, dl_d = rec["status"][di], rec["iterations"][di], rec["delta"][di]
        v_o = (st_o == 0) & (dl_o > 1e-7)
        v_d = (st_d == 0) & (dl_d > 1e-7)
        sens = qp_solver_sensitive(st_o, it_o, dl_o, st_d, it_d, dl_d)
        assert not np.any((v_o != v_d) & ~sens)
        mism = int((v_o != v_d).sum())
    else:
        assert dk.size == 0
        mism = 0
    print(f"seed {seed}: m={spec.m} gamma={spec.gamma} T={spec.T} V={gr.num_vertices} E={gr.num_edges} "
          f"qp={mask.pairs_qp} verdict mismatches={mism}")
    if mism == 0:
        assert np.array_equal(mask.alive, rc["alive"])
        assert np.array_equal(mask.provenance_codes, rc["provenance"])
        p_dev = G.find_path(gr, mask, start, goal)
        p_ref, _ = oracle.find_path(ref["vertices"], ref["edges"], ref["costs"], rc["alive"], start, goal, spec.m,
                                 orc.tube.error.lo, orc.tube.error.hi)
        assert p_dev == (None if p_ref is None else list(p_ref))
