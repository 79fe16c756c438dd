"""CPU restatement of the spec-only Newton solve -- TEST INFRASTRUCTURE ONLY.

The reference ships no Newton code, so parity for this
component is UNPINNED by reference code: this module restates
SPEC.md:286-315 (gradient, Hessian, Jacobi-PCG, KMT damping, init_weights)
and SPEC.md:322-335 (sign convention, tolerances 1e-3 / 1e-4, floor with
|V(psi0)|) literally in numpy, with every cell evaluation done by the
bit-exact oracle of _kernels._batch_evaluate.  Its own pins are the SPEC
examples (tests/test_newton_cpu.py) and a finite-difference Hessian check.
"""
from __future__ import annotations

import numpy as np

from . import pyoracle as O


def _evaluate(pts, psi, dom_args, tol, grid, smf):
    o = O.evaluate(pts, psi, dom_args, tol, grid, ball_aware=True, want_m2=False, smf=smf)
    return o


def hessian_ell(pts, psi, o, tau_psi, smf):
    """Row-wise H = -grad^2 K from cell i's facet list."""
    n = len(pts)
    fc = np.minimum(o["fcount"], smf)
    cols = np.full((n, smf), -1, np.int64)
    vals = np.zeros((n, smf))
    diag = np.zeros(n)
    mask = (np.arange(smf)[None, :] < fc[:, None]) & (o["ftag"] >= 0)
    j = np.where(mask, o["ftag"], 0)
    D = np.sqrt(((pts[j] - pts[:, None, :]) ** 2).sum(-1))
    w = np.where(mask, 0.5 * o["farea"] / np.where(mask, D, 1.0), 0.0)
    cols[mask] = o["ftag"][mask]
    vals[mask] = -w[mask]
    diag = w.sum(1) + 0.5 * o["ksur"] / np.sqrt(np.maximum(psi, tau_psi))
    # An empty cell (no facet, no free surface) has a zero row.
    # gives it "the Hessian diagonal from the tau_psi guard"; the only SPEC value
    # of that diagonal is the free ball's, H_ii = d|V_i|/d psi_i = 2 pi sqrt(psi_i)
    # (SPEC.md:296 example), evaluated at max(psi_i, tau_psi).  Cold-start and
    # accepted states never have empty cells (init_weights / the KMT floor), so
    # this only affects rows the damping then rejects.
    bad = ~(diag > 0.0)
    diag[bad] = 2.0 * np.pi * np.sqrt(np.maximum(psi[bad], tau_psi))
    return cols, vals, diag


def spmv(cols, vals, diag, x):
    xs = np.where(cols >= 0, x[np.maximum(cols, 0)], 0.0)
    return diag * x + (vals * xs).sum(1)


def pcg(cols, vals, diag, b, rtol, max_iter=10000):
    """Jacobi PCG (cg_solve): x0 = 0, preconditioner D^-1,
    stop when ||H x - b|| = ||r|| <= tol ||b|| (the SPEC's post-condition, with
    the recursively updated residual) or max_iter."""
    x = np.zeros_like(b)
    r = b.copy()
    z = r / diag
    p = z.copy()
    rz = float(r @ z)
    bb = float(b @ b)
    if not bb > 0.0:
        return x, 0
    it = 0
    while True:
        Ap = spmv(cols, vals, diag, p)
        pAp = float(p @ Ap)
        alpha = rz / pAp if pAp != 0.0 else 0.0
        x += alpha * p
        r -= alpha * Ap
        z = r / diag
        rz_new = float(r @ z)
        rr = float(r @ r)
        beta = rz_new / rz if rz != 0.0 else 0.0
        rz = rz_new
        it += 1
        if np.sqrt(rr) <= rtol * np.sqrt(bb) or it >= max_iter or rz_new != rz_new:
            return x, it
        p = z + beta * p


def newton_solve(pts, nu, dom_args, tol, domain_diag, psi_init=None, eps_vol=0.01,
                 max_newton=100, smf=32):
    pts = np.ascontiguousarray(pts, np.float64)
    nu = np.asarray(nu, np.float64)
    grid = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    tau = 1e-12 * domain_diag ** 2
    stats = dict(iterations=0, evaluations=0, cg_iterations=0, damping_halvings=0,
                 init_doublings=0, status=0, cg_per_iter=[], worst_history=[])
    if psi_init is None:
        kappa = 1.0
        while True:
            psi = kappa * (3.0 * nu / (4.0 * np.pi)) ** (2.0 / 3.0)
            o = _evaluate(pts, psi, dom_args, tol, grid, smf)
            stats["evaluations"] += 1
            if o["vol"].min() > 0.0:
                break
            kappa *= 2.0
            stats["init_doublings"] += 1
            if kappa > 1024.0:
                stats["status"] = 3
                return psi, stats
    else:
        psi = np.array(psi_init, np.float64)
        o = _evaluate(pts, psi, dom_args, tol, grid, smf)
        stats["evaluations"] += 1
        # warm start with per-cell rescue (SPEC.md init_weights): empty cells get
        # psi_i <- max(psi_i, kappa (3 nu_i / 4 pi)^(2/3)), kappa doubling
        if not o["vol"].min() > 0.0:
            # an empty cell first takes the weight of its nearest other site
            from scipy.spatial import cKDTree

            e = np.nonzero(~(o["vol"] > 0.0))[0]
            _, nn = cKDTree(pts).query(pts[e], k=2)
            j = np.where(nn[:, 0] == e, nn[:, 1], nn[:, 0])
            psi[e] = np.maximum(psi[e], psi[j])
            stats["init_doublings"] += 1
            o = _evaluate(pts, psi, dom_args, tol, grid, smf)
            stats["evaluations"] += 1
        kappa = 1.0
        while not o["vol"].min() > 0.0:
            if kappa > 1024.0:
                stats["status"] = 3
                return psi, stats
            e = ~(o["vol"] > 0.0)
            psi[e] = np.maximum(psi[e], kappa * (3.0 * nu[e] / (4.0 * np.pi)) ** (2.0 / 3.0))
            stats["init_doublings"] += 1
            o = _evaluate(pts, psi, dom_args, tol, grid, smf)
            stats["evaluations"] += 1
            kappa *= 2.0
    floor_v = 0.5 * min(nu.min(), o["vol"].min())
    worst = float(np.max(np.abs(o["vol"] - nu) / nu))
    stats["worst_initial"] = worst
    stats["worst_history"].append(worst)
    for _ in range(max_newton):
        if worst <= eps_vol:
            break
        g = nu - o["vol"]
        cols, vals, diag = hessian_ell(pts, psi, o, tau, smf)
        rtol = 1e-4 if worst < 10 * eps_vol else 1e-3
        u, cg = pcg(cols, vals, diag, g, rtol)
        stats["cg_iterations"] += cg
        stats["cg_per_iter"].append(cg)
        alpha = 1.0
        ok = False
        while alpha >= 2.0 ** -20:
            pt = psi + alpha * u
            ot = _evaluate(pts, pt, dom_args, tol, grid, smf)
            stats["evaluations"] += 1
            if ot["vol"].min() >= floor_v:
                ok = True
                break
            alpha *= 0.5
            stats["damping_halvings"] += 1
        if not ok:
            stats["status"] = 2
            break
        psi, o = pt, ot
        stats["iterations"] += 1
        worst = float(np.max(np.abs(o["vol"] - nu) / nu))
        stats["worst_history"].append(worst)
    stats["worst_final"] = worst
    if stats["status"] == 0 and worst > eps_vol:
        stats["status"] = 1
    stats["last_eval"] = o
    return psi, stats
