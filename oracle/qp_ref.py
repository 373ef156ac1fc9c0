"""Cut-QP restatement (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Restates, with the same float64 numpy expressions so results are bitwise
equal on the same host:

* the slack-minimising hull/obstacle QP of reference graph.py:268-282
  (``_cut_qp_problem``):  vars [lambda (J); delta (C)],
  min delta'delta  s.t.  (A_O P) lambda - delta <= b_O,  lambda >= 0,
  sum(lambda) = 1;
* the dense batched ADMM of reference qpsolver.py:129-233
  (``_dense_kernel``): KKT inverse per instance, rho = 1 (1e3 on equality
  rows), sigma, alpha over-relaxation, per-iteration termination on
  eps_abs/eps_rel, primal-infeasibility certificate, MAX_ITER snapshot;
* the active-set polish of reference qpsolver.py:236-279 (``_polish_one``).

Status codes: 0 SOLVED, 1 MAX_ITER, 2 INFEASIBLE, 3 ERROR (qpsolver.py:29-33).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SOLVED, MAX_ITER, INFEASIBLE, ERROR = 0, 1, 2, 3
_EQ_TOL = 1e-9  # qpsolver.py:26


@dataclass
class AdmmSettings:
    """Values of CutConfig.qp (reference graph.py:47-49) over SolveConfig defaults (qpsolver.py:60-72)."""

    max_iter: int = 500
    eps_abs: float = 1e-7
    eps_rel: float = 0.0
    rho: float = 1.0
    sigma: float = 1e-6
    alpha: float = 1.6
    eps_pinf: float = 1e-4
    polish: bool = True


def cut_qp_problem(points: np.ndarray, A_O: np.ndarray, b_O: np.ndarray):
    """(P, q, A, l, u) for one edge's control points (m, J) vs a normalised obstacle (graph.py:268-282)."""
    _, J = points.shape
    C = A_O.shape[0]
    nv = J + C
    P = np.zeros((nv, nv))
    P[J:, J:] = 2.0 * np.eye(C)
    q = np.zeros(nv)
    A = np.zeros((C + J + 1, nv))
    A[:C, :J] = A_O @ points
    A[:C, J:] = -np.eye(C)
    A[C:C + J, :J] = np.eye(J)
    A[C + J, :J] = 1.0
    lo = np.concatenate([np.full(C, -np.inf), np.zeros(J), [1.0]])
    hi = np.concatenate([b_O, np.full(J, np.inf), [1.0]])
    return P, q, A, lo, hi


def _admm(P, q, A, l, u, s: AdmmSettings):
    """Batched ADMM over stacks (B, ...) of same-shape instances (qpsolver.py:129-233)."""
    B, n = q.shape
    mc = l.shape[1]
    rho = np.where((u - l) <= _EQ_TOL, s.rho * 1e3, s.rho)
    rinv = 1.0 / rho

    K = np.zeros((B, n + mc, n + mc))
    K[:, :n, :n] = P
    K[:, np.arange(n), np.arange(n)] += s.sigma
    K[:, :n, n:] = np.swapaxes(A, 1, 2)
    K[:, n:, :n] = A
    K[:, n + np.arange(mc), n + np.arange(mc)] = -rinv
    Kinv = np.linalg.inv(K)

    x = np.zeros((B, n))
    y = np.zeros((B, mc))
    z = np.zeros((B, mc))

    done = np.zeros(B, dtype=bool)
    out_x = np.zeros((B, n))
    out_y = np.zeros((B, mc))
    out_it = np.zeros(B, dtype=np.int64)
    out_rp = np.full(B, np.inf)
    out_rd = np.full(B, np.inf)
    out_st = np.full(B, MAX_ITER, dtype=np.int8)

    def snap(sel, it, xs, ys, rps, rds, st):
        done[sel] = True
        out_x[sel] = xs
        out_y[sel] = ys
        out_it[sel] = it
        out_rp[sel] = rps
        out_rd[sel] = rds
        out_st[sel] = st

    ids = np.arange(B)
    qn = np.abs(q).max(axis=1, initial=0.0)
    finished_early = False
    for it in range(1, s.max_iter + 1):
        rhs = np.concatenate([s.sigma * x - q, z - rinv * y], axis=1)
        sol = np.einsum("bij,bj->bi", Kinv, rhs)
        xt = sol[:, :n]
        zt = z + rinv * (sol[:, n:] - y)
        xn = s.alpha * xt + (1.0 - s.alpha) * x
        zr = s.alpha * zt + (1.0 - s.alpha) * z
        zn = np.clip(zr + rinv * y, l, u)
        yn = y + rho * (zr - zn)

        Ax = np.einsum("bij,bj->bi", A, xn)
        Px = np.einsum("bij,bj->bi", P, xn)
        ATy = np.einsum("bji,bj->bi", A, yn)
        rp = np.abs(Ax - zn).max(axis=1, initial=0.0)
        rd = np.abs(Px + q + ATy).max(axis=1)
        ep = s.eps_abs + s.eps_rel * np.maximum(np.abs(Ax).max(axis=1, initial=0.0), np.abs(zn).max(axis=1, initial=0.0))
        ed = s.eps_abs + s.eps_rel * np.maximum(
            np.maximum(np.abs(Px).max(axis=1), np.abs(ATy).max(axis=1, initial=0.0)), qn)
        conv = (rp <= ep) & (rd <= ed) & ~done[ids]
        if np.any(conv):
            snap(ids[conv], it, xn[conv], yn[conv], rp[conv], rd[conv], SOLVED)

        dy = yn - y
        dyn = np.abs(dy).max(axis=1, initial=0.0)
        cand = (dyn > 1e-13) & ~done[ids]
        if np.any(cand):
            ATdy = np.einsum("bji,bj->bi", A, dy)
            pos = np.where(dy > 0, dy, 0.0)
            neg = np.where(dy < 0, dy, 0.0)
            supp = (np.where(pos > 0, u, 0.0) * pos + np.where(neg < 0, l, 0.0) * neg).sum(axis=1)
            cert = cand & (np.abs(ATdy).max(axis=1) <= s.eps_pinf * dyn) & (supp <= -s.eps_pinf * dyn)
            if np.any(cert):
                snap(ids[cert], it, xn[cert], yn[cert], rp[cert], rd[cert], INFEASIBLE)

        x, y, z = xn, yn, zn
        live = ~done[ids]
        if not live.any():
            finished_early = True
            break
        if live.sum() <= ids.size // 2 and ids.size > 1:
            x, y, z = x[live], y[live], z[live]
            Kinv, P, q, A, l, u = Kinv[live], P[live], q[live], A[live], l[live], u[live]
            rho, rinv, qn = rho[live], rinv[live], qn[live]
            ids = ids[live]
    if not finished_early:
        left = ~done[ids]
        if np.any(left):
            Ax = np.einsum("bij,bj->bi", A, x)
            Px = np.einsum("bij,bj->bi", P, x)
            ATy = np.einsum("bji,bj->bi", A, y)
            rp = np.abs(Ax - z).max(axis=1, initial=0.0)
            rd = np.abs(Px + q + ATy).max(axis=1)
            snap(ids[left], s.max_iter, x[left], y[left], rp[left], rd[left], MAX_ITER)
    return out_x, out_y, out_st, out_it, out_rp, out_rd


def _polish(P, q, A, l, u, x, y, rp, rd):
    """Equality-constrained re-solve on the detected active set (qpsolver.py:236-279)."""
    mc = l.shape[0]
    zc = A @ x
    tol = max(1e-7, 10.0 * rp)
    at_lo = (zc - l) <= tol
    at_hi = (u - zc) <= tol
    act = at_lo | at_hi
    if not np.any(act):
        y0 = np.zeros(mc)
        rd0 = float(np.abs(P @ x + q).max())
        return (x, y0) if rd0 <= rd else (x, y)
    Gm = A[act]
    g = np.where(at_lo[act], l[act], u[act])
    n = x.shape[0]
    k = Gm.shape[0]
    reg = 1e-8
    K = np.zeros((n + k, n + k))
    K[:n, :n] = P + reg * np.eye(n)
    K[:n, n:] = Gm.T
    K[n:, :n] = Gm
    K[n:, n:] = -reg * np.eye(k)
    rhs = np.concatenate([-q, g])
    try:
        w = np.linalg.solve(K, rhs)
        for _ in range(2):
            w = w + np.linalg.solve(K, rhs - K @ w)
    except np.linalg.LinAlgError:
        w, *_ = np.linalg.lstsq(K, rhs, rcond=None)
    xp = w[:n]
    yp = np.zeros(mc)
    yp[act] = w[n:]
    Axp = A @ xp
    rpp = float(np.maximum(Axp - u, 0.0).max(initial=0.0) + np.maximum(l - Axp, 0.0).max(initial=0.0))
    rdp = float(np.abs(P @ xp + q + A.T @ yp).max())
    if max(rpp, rdp) < max(rp, rd):
        return xp, yp
    return x, y


def solve_dense_batch(P, q, A, l, u, settings: AdmmSettings | None = None, chunk: int = 65536):
    """Solve stacked same-shape QPs; returns (x (B,n), status (B,), iterations (B,)).

    Mirrors ``qpsolver._solve_dense_group`` (qpsolver.py:282-304), which
    feeds ``_BATCH_CHUNK = 65536`` instances per kernel call.
    """
    s = settings or AdmmSettings()
    B = q.shape[0]
    xs = np.zeros_like(q)
    st = np.zeros(B, dtype=np.int8)
    its = np.zeros(B, dtype=np.int64)
    for lo in range(0, B, chunk):
        hi = min(lo + chunk, B)
        x, y, status, it, rp, rd = _admm(P[lo:hi], q[lo:hi], A[lo:hi], l[lo:hi], u[lo:hi], s)
        for i in range(hi - lo):
            xi = x[i]
            if s.polish and status[i] in (SOLVED, MAX_ITER):
                xi, _ = _polish(P[lo + i], q[lo + i], A[lo + i], l[lo + i], u[lo + i], xi, y[i],
                                float(rp[i]), float(rd[i]))
            xs[lo + i] = xi
        st[lo:hi] = status
        its[lo:hi] = it
    return xs, st, its
