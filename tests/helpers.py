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


def qp_solver_sensitive(status_a, iters_a, delta_a, status_b, iters_b, delta_b, eps_cut=1e-7):
    """pairs whose verdict is solver-dependent — MAX_ITER on either side,
    ||delta|| within 1e-8 of eps_cut, or different iteration counts."""
    return ((status_a == 1) | (status_b == 1) | (np.abs(delta_a - eps_cut) < 1e-8) | (np.abs(delta_b - eps_cut) < 1e-8)
            | (iters_a != iters_b))


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
    rep["counters_dev"] = cnt
    rep["counters_ref"] = [int(x) for x in g["counters"]]
    if not same_set:
        return rep
    st_d, it_d, dl_d = rec["status"][do], rec["iterations"][do], rec["delta"][do]
    st_g, it_g, dl_g = g["qp_status"][go], g["qp_iters"][go], g["qp_delta"][go]
    v_d = (st_d == 0) & (dl_d > eps_cut)
    v_g = (st_g == 0) & (dl_g > eps_cut)
    sens = qp_solver_sensitive(st_g, it_g, dl_g, st_d, it_d, dl_d, eps_cut)
    mism = v_d != v_g
    rep["verdict_mismatch"] = int(mism.sum())
    rep["mismatch_outside_sensitive"] = int((mism & ~sens).sum())
    rep["solver_sensitive"] = int(sens.sum())
    rep["status_equal"] = float((st_d == st_g).mean()) if st_d.size else 1.0
    rep["iters_equal"] = float((it_d == it_g).mean()) if it_d.size else 1.0
    touched = np.zeros(g["alive"].size, dtype=bool)
    touched[g["qp_edge"][go][mism]] = True
    rep["alive_mismatch_untouched"] = int(((mask.alive != g["alive"]) & ~touched).sum())
    rep["prov_mismatch_untouched"] = int(((mask.provenance_codes != g["provenance"]) & ~touched).sum())
    rep["alive_mismatch"] = int((mask.alive != g["alive"]).sum())
    return rep
