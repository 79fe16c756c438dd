"""CPU restatement of the spec-only Newton solve (oracle/newton_ref.py):
pinned on the SPEC examples, on the survey's prototype
counts for C1 (4 iterations / 5 evaluations / 65 CG, per
iteration 15, 17, 15, 18) and on a finite-difference Hessian check
(1e-4 relative)."""
import numpy as np
import pytest

from oracle import newton_ref as NR
from oracle import pyoracle as O
from paper_2601_05765_b200 import geom, laguerre, scenes

DOM = geom.box_domain([0, 0, 0], [1, 1, 1])
DPK = laguerre.domain_pack(DOM)


def solve(pts, nu, **kw):
    return NR.newton_solve(pts, nu, DPK.args(), DPK.tol, DOM.diagonal(), **kw)


def test_single_ball_one_iteration():
    nu = np.array([(4 / 3) * np.pi * 1e-3])
    psi, st = solve(np.array([[0.5, 0.5, 0.5]]), nu, psi_init=np.array([0.009]))
    assert st["status"] == 0 and st["iterations"] <= 1
    assert abs(psi[0] - 1e-2) < 2e-4


def test_symmetric_sites_equal_weights():
    c = np.array([[x, y, z] for x in (0.25, 0.75) for y in (0.25, 0.75) for z in (0.25, 0.75)])
    psi, st = solve(c, np.full(8, 0.1))
    assert st["status"] == 0
    assert np.ptp(psi) <= 1e-12 * psi.max()


def test_random_2000_converges():
    rng = np.random.default_rng(5)
    pts = rng.random((2000, 3))
    nu = np.full(2000, 0.3 / 2000)
    psi, st = solve(pts, nu)
    assert st["status"] == 0 and st["iterations"] <= 100
    v = st["last_eval"]["vol"]
    assert np.max(np.abs(v - nu) / nu) <= 0.01


def test_c1_matches_survey_prototype():
    s = scenes.c1_random()
    psi, st = solve(s.pts, s.nu)
    assert (st["iterations"], st["evaluations"], st["cg_iterations"]) == (4, 5, 65)
    assert st["cg_per_iter"] == [15, 17, 15, 18]
    assert abs(st["worst_initial"] - 0.846) < 1e-3 and st["worst_final"] < 1e-4


def test_hessian_matches_finite_differences():
    rng = np.random.default_rng(11)
    pts = rng.random((20, 3))
    psi = np.full(20, 0.04) * (1 + 0.3 * rng.random(20))
    grid = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    o = O.evaluate(pts, psi, DPK.args(), DPK.tol, grid, smf=32)
    cols, vals, diag = NR.hessian_ell(pts, psi, o, 1e-12 * 3, 32)
    H = np.diag(diag)
    for i in range(20):
        for k in range(32):
            if cols[i, k] >= 0:
                H[i, cols[i, k]] += vals[i, k]
    worst = 0.0
    for j in range(20):
        h = 1e-6 * psi[j]
        pp, pm = psi.copy(), psi.copy()
        pp[j] += h
        pm[j] -= h
        vp = O.evaluate(pts, pp, DPK.args(), DPK.tol, grid, smf=32)["vol"]
        vm = O.evaluate(pts, pm, DPK.args(), DPK.tol, grid, smf=32)["vol"]
        col = (vp - vm) / (2 * h)  # d|V_i|/dpsi_j = H_ij (H = -grad^2 K)
        for i in range(20):
            if abs(H[i, j]) > 1e-8:
                worst = max(worst, abs(col[i] - H[i, j]) / abs(H[i, j]))
    assert worst < 1e-4
