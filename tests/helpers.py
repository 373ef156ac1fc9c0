"""Shared test helpers: rebuild inputs from golden records, compare cut outcomes."""

from __future__ import annotations

import hashlib
from types import SimpleNamespace

import numpy as np

from paper_2411_13507_b200.bezier import BezierSpec
from paper_2411_13507_b200.geometry import Box, Polytope


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def inputs_from_golden(g: dict):
    """(N, spec, oracle, bounds, seed, include, obstacles, start, goal) for a golden record."""
    spec = BezierSpec(int(g["m"]), int(g["gamma"]), float(g["T"]))
    tube = SimpleNamespace(error=Box(g["tube_lo"], g["tube_hi"]))
    oracle = SimpleNamespace(F=g["F"], G=g["G"], Xd=Polytope(g["xd_A"], g["xd_b"]), tube=tube, spec=spec)
    bounds = Box(g["bounds_lo"], g["bounds_hi"])
    obstacles = []
    off = 0
    for k in g["obs_n"]:
        obstacles.append(Polytope(g["obs_A"][off:off + k], g["obs_b"][off:off + k]))
        off += int(k)
    include = g["include"] if g["include"].size else None
    return int(g["N"]), spec, oracle, bounds, int(g["seed"]), include, obstacles, g["start"], g["goal"]


def qp_solver_sensitive(status_a, iters_a, delta_a, status_b, iters_b, delta_b, eps_cut=1e-7, eps_abs=1e-7):
    """QP pairs whose verdict may legitimately depend on the solver's rounding --
    MAX_ITER or an infeasibility certificate on either side (the verdict then hinges on where
    the iteration stopped), or ||delta|| within eps_abs of eps_cut on either side: the ADMM
    stops once its residuals are below eps_abs (CutConfig.qp, graph.py:47-49), so a ||delta||
    that close to the threshold is only known to that accuracy.  (Measured at cfg3 against the
    live reference: the four both-SOLVED verdict differences have ||delta|| in [7.0e-8,
    1.65e-7] on the two sides, iteration counts 1-2 apart.)  A differing iteration count alone
    does NOT excuse a verdict difference (iters_* are kept in the signature for the report)."""
    del iters_a, iters_b
    return ((status_a == 1) | (status_b == 1) | (status_a == 2) | (status_b == 2)
            | (np.abs(delta_a - eps_cut) < eps_abs) | (np.abs(delta_b - eps_cut) < eps_abs))


def compare_cut(mask, g: dict, eps_cut: float = 1e-7) -> dict:
    """Compare a device CutMask with a golden record that holds per-QP detail.

    Returns a report; heuristic outcomes (pending set, counters 0-3) must match exactly,
    QP verdict differences are classified as solver-sensitive or not, and alive /
    provenance must match on every edge not touched by a QP verdict difference.
    """
    rec = mask.qp_records()
    dk = rec["edge"].astype(np.int64) * 1_000_003 + rec["obstacle"]
    gk = g["qp_edge"].astype(np.int64) * 1_000_003 + g["qp_obstacle"]
    do, go = np.argsort(dk, kind="stable"), np.argsort(gk, kind="stable")
    same_set = dk.size == gk.size and np.array_equal(dk[do], gk[go])
    rep = {"same_pending": bool(same_set), "n_qp": int(gk.size)}
    cnt = [mask.pairs_total, mask.pairs_point_hit, mask.pairs_hyperplane, mask.pairs_qp, mask.qp_safe, mask.qp_unsafe]
    rep["counters_dev"] = [int(x) for x in cnt]
    rep["counters_ref"] = [int(x) for x in g["counters"]]
    if not same_set:
        return rep
    st_d, it_d, dl_d = rec["status"][do], rec["iterations"][do].astype(np.int64), rec["delta"][do]
    st_g, it_g = g["qp_status"][go], g["qp_iters"][go].astype(np.int64)
    dl_g = g["qp_delta"][go].astype(np.float64)
    v_d = (st_d == 0) & (dl_d > eps_cut)
    v_g = (st_g == 0) & (dl_g > eps_cut)
    sens = qp_solver_sensitive(st_g, it_g, dl_g, st_d, it_d, dl_d, eps_cut)
    mism = v_d != v_g
    rep["verdict_mismatch"] = int(mism.sum())
    out = np.nonzero(mism & ~sens)[0][:10]
    rep["outside_examples"] = [[int(st_g[i]), int(st_d[i]), int(it_g[i]), int(it_d[i]), float(dl_g[i]), float(dl_d[i])]
                               for i in out]
    rep["mismatch_outside_sensitive"] = int((mism & ~sens).sum())
    rep["solver_sensitive"] = int(sens.sum())
    rep["status_equal"] = float((st_d == st_g).mean()) if st_d.size else 1.0
    rep["iters_equal"] = float((it_d == it_g).mean()) if it_d.size else 1.0
    dit = np.abs(it_d - it_g)
    rep["iters_absdiff_max_solved"] = int(dit[(st_d == 0) & (st_g == 0)].max()) if ((st_d == 0) & (st_g == 0)).any() else 0
    rep["iters_absdiff_p999"] = float(np.quantile(dit, 0.999)) if dit.size else 0.0
    both = (st_d == 0) & (st_g == 0) & (dl_g > 1e-6)
    rep["delta_rel_max_solved"] = float((np.abs(dl_d[both] - dl_g[both]) / dl_g[both]).max()) if both.any() else 0.0
    touched = np.zeros(g["alive"].size, dtype=bool)
    touched[g["qp_edge"][go][mism]] = True
    rep["alive_mismatch_untouched"] = int(((mask.alive != g["alive"]) & ~touched).sum())
    rep["prov_mismatch_untouched"] = int(((mask.provenance_codes != g["provenance"]) & ~touched).sum())
    rep["alive_mismatch"] = int((mask.alive != g["alive"]).sum())
    rep["prov_mismatch"] = int((mask.provenance_codes != g["provenance"]).sum())
    return rep


def assert_cut_parity(rep: dict, *, max_mismatch_frac: float = 1e-4) -> None:
    """The cut parity bar: heuristic outcomes exact, every QP verdict
    difference solver-sensitive and rare, alive/provenance exact away from those edges, and the
    six counters exact unless a (sensitive) verdict differs."""
    assert rep["same_pending"], rep
    assert rep["counters_dev"][:4] == rep["counters_ref"][:4], rep
    assert rep["mismatch_outside_sensitive"] == 0, rep
    assert rep["verdict_mismatch"] <= max(1, int(max_mismatch_frac * rep["n_qp"])), rep
    assert rep["alive_mismatch_untouched"] == 0 and rep["prov_mismatch_untouched"] == 0, rep
    assert rep["status_equal"] >= 0.99 and rep["iters_equal"] >= 0.97, rep
    if rep["verdict_mismatch"] == 0:
        assert rep["counters_dev"] == rep["counters_ref"], rep
        assert rep["alive_mismatch"] == 0 and rep["prov_mismatch"] == 0, rep
