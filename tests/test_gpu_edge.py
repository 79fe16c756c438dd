"""Edge cases through the reference-signature drop-in, against the CPU oracle:
no sites, one site, coincident sites (the reference's heavier-weight / lower-
index rule), zero weights, a site on the domain boundary, and facet lists
longer than the caller's stride (smf overflow flag)."""
import numpy as np
import pytest

from conftest import OUT_KEYS

pytestmark = pytest.mark.gpu


def _both(pts, psi, smf=32, ball_aware=True):
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import _kernels, geom, laguerre

    pts = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 3))
    psi = np.ascontiguousarray(np.asarray(psi, dtype=np.float64))
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    n = len(pts)
    dev = O.alloc_outputs(n, smf)
    gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
    dpsi = float(psi.max() - psi.min()) if n else 0.0
    err = _kernels._batch_evaluate(pts, psi, *dpk.args(), *gargs, dpk.tol, dpsi, ball_aware, True, smf,
                                   *[dev[k] for k in O.OUT_ORDER])
    g = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    ref = O.evaluate(pts, psi, dpk.args(), dpk.tol, g, ball_aware=ball_aware, smf=smf) if n else None
    return err, dev, ref


def _same(dev, ref, err):
    assert err == ref["err"]
    for k in ("status", "fcount", "ftag"):
        assert np.array_equal(dev[k], ref[k]), k
    for k in ("vol", "ksur", "farea"):
        assert np.allclose(dev[k], ref[k], rtol=1e-9, atol=1e-15), k


def test_no_sites():
    err, dev, _ = _both(np.zeros((0, 3)), np.zeros(0))
    assert err == 0 and all(dev[k].size == 0 for k in OUT_KEYS)


def test_one_site_is_a_full_ball():
    err, dev, ref = _both([[0.5, 0.5, 0.5]], [0.01])
    _same(dev, ref, err)
    assert dev["status"][0] == 1 and abs(dev["vol"][0] - 4 / 3 * np.pi * 0.1 ** 3) < 1e-15


def test_coincident_sites_and_zero_weights():
    rng = np.random.default_rng(5)
    pts = rng.random((400, 3))
    pts[10] = pts[11]          # coincident, equal weights: lower index wins
    pts[20] = pts[21]          # coincident, heavier second site wins
    psi = np.full(400, 0.06 ** 2)
    psi[21] *= 1.5
    psi[30:35] = 0.0           # empty balls
    err, dev, ref = _both(pts, psi)
    _same(dev, ref, err)
    assert dev["status"][11] == 0 and dev["status"][20] == 0 and (dev["status"][30:35] == 0).all()


def test_site_on_the_boundary_and_full_mode():
    rng = np.random.default_rng(6)
    pts = rng.random((300, 3))
    pts[0] = [0.0, 0.5, 0.5]
    pts[1] = [1.0, 1.0, 0.3]
    psi = np.full(300, 0.08 ** 2)
    for ba in (True, False):
        err, dev, ref = _both(pts, psi, ball_aware=ba)
        _same(dev, ref, err)


def test_facet_list_longer_than_stride():
    rng = np.random.default_rng(7)
    pts = rng.random((2000, 3))
    psi = np.full(2000, 0.09 ** 2)
    err, dev, ref = _both(pts, psi, smf=4)
    _same(dev, ref, err)
    assert err & 1  # FLAG_OVERFLOW: some cell has more restricted facets than the stride
