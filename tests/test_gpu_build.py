"""Unrestricted Laguerre cells on the device: the
reference's `_kernels._batch_build` drop-in and `laguerre.build_diagram_packed`
against the reference's own outputs (tests/golden, ball-aware and full
security-radius mode): every array bit-exact."""
import numpy as np
import pytest

from conftest import golden_domain

pytestmark = pytest.mark.gpu

KEYS = ("status", "nv", "nf", "nl", "verts", "planes", "tags", "lp", "lv")


@pytest.mark.parametrize("mode", ["ba", "full"])
def test_dropin_batch_build_matches_reference(golden, mode):
    from paper_2601_05765_b200 import _kernels

    pts, psi = golden["bb_pts"], golden["bb_psi"]
    n = len(pts)
    smv, smf, sml = (golden[f"bb_{mode}_verts"].shape[1], golden[f"bb_{mode}_planes"].shape[1],
                     golden[f"bb_{mode}_lv"].shape[1])
    arrs = [np.zeros(n, np.int64) for _ in range(4)] + [
        np.zeros((n, smv, 3)), np.zeros((n, smf, 4)), np.zeros((n, smf), np.int64),
        np.zeros((n, smf + 1), np.int64), np.zeros((n, sml), np.int64)]
    gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
    err = _kernels._batch_build(pts, psi, *golden_domain(golden), *gargs, float(golden["dom_unit_tol"]),
                                float(psi.max() - psi.min()), mode == "ba", smv, smf, sml, *arrs)
    assert err == 0
    for k, a in zip(KEYS, arrs):
        assert np.array_equal(a, golden[f"bb_{mode}_{k}"]), k


@pytest.mark.parametrize("mode", ["ba", "full"])
def test_build_diagram_packed_matches_reference(golden, mode):
    from paper_2601_05765_b200 import geom, laguerre

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    d = laguerre.build_diagram_packed((golden["bb_pts"], golden["bb_psi"]), dom, ball_aware=(mode == "ba"))
    for k in KEYS:
        assert np.array_equal(getattr(d, k), golden[f"bb_{mode}_{k}"]), k
    if mode == "full":  # full security radius: the cells partition the domain
        cells = laguerre.build_diagram((golden["bb_pts"], golden["bb_psi"]), dom)
        vol = sum(geom.cell_volume_convex(c) for c in cells if c is not None)
        assert abs(vol - 1.0) < 1e-9


@pytest.mark.parametrize("mode", ["ba", "full"])
def test_single_cell_build_matches_reference(golden, mode):
    """laguerre.build_cell (reference laguerre.py:148-183): the cell of one
    site, from the sites near it, equals the reference's packed cell of the
    whole-diagram build bit for bit (vertices, planes, tags, loops)."""
    from paper_2601_05765_b200 import geom, laguerre

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    pts, psi = golden["bb_pts"], golden["bb_psi"]
    st = golden[f"bb_{mode}_status"]
    rng = np.random.default_rng(5)
    picks = list(rng.choice(len(pts), 12, replace=False)) + [int(np.argmax(psi)), int(np.argmin(psi))]
    for i in picks:
        c = laguerre.build_cell(int(i), (pts, psi), dom, ball_aware=(mode == "ba"))
        if st[i] == 1:
            assert c is None
            continue
        g = {k: golden[f"bb_{mode}_{k}"][i] for k in KEYS}
        want = geom.unpack_cell(g["verts"], np.array([g["nv"], g["nf"], g["nl"]]), g["planes"], g["tags"],
                                g["lp"], g["lv"])
        assert np.array_equal(c.vertices, want.vertices)
        assert len(c.facets) == len(want.facets)
        for fc, fw in zip(c.facets, want.facets):
            assert fc.tag == fw.tag
            assert np.array_equal(fc.plane.n, fw.plane.n) and fc.plane.d == fw.plane.d
            assert np.array_equal(fc.loop, fw.loop)
    with pytest.raises(IndexError):
        laguerre.build_cell(len(pts), (pts, psi), dom)


def test_full_mode_heavy_weights_match_oracle(golden):
    """Full mode with a few huge weights (the n - 1-candidate pathology of
    SURVEY §8(f) row 2): the device's heavy-site phase gives the reference's
    packed cells bit for bit (oracle = the bit-identical C restatement), and
    in a fraction of the time the global security radius would take."""
    import os
    import sys
    import time

    import torch

    from conftest import ROOT
    from paper_2601_05765_b200 import _kernels

    sys.path.insert(0, ROOT)
    from oracle import pyoracle as O

    rng = np.random.default_rng(21)
    n = 4000
    pts = rng.random((n, 3))
    psi = np.full(n, (0.6 * (1.0 / n) ** (1.0 / 3.0)) ** 2)
    psi[[5, 1234, 2999]] = (0.3, 0.12, 0.05)
    dpsi = float(psi.max() - psi.min())
    dom, tol = golden_domain(golden), float(golden["dom_unit_tol"])
    smv, smf, sml = 512, 160, 2048  # the reference's capacities: the heavy sites' cells are large

    def arrays():
        return [np.zeros(n, np.int64) for _ in range(4)] + [
            np.zeros((n, smv, 3)), np.zeros((n, smf, 4)), np.zeros((n, smf), np.int64),
            np.zeros((n, smf + 1), np.int64), np.zeros((n, sml), np.int64)]

    ref = arrays()
    g = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    err_ref = O.batch_build(pts, psi, *dom, *g.kernel_args(), tol, dpsi, False, smv, smf, sml, *ref)
    gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
    times = {}
    for mode in ("heavy", "global"):
        if mode == "global":
            os.environ["PF_NO_HEAVY"] = "1"
        try:
            dev = arrays()
            for rep in range(2):  # second call timed
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                assert _kernels._batch_build(pts, psi, *dom, *gargs, tol, dpsi, False, smv, smf, sml, *dev) == err_ref
                torch.cuda.synchronize()
                times[mode] = time.perf_counter() - t0
        finally:
            os.environ.pop("PF_NO_HEAVY", None)
        for k, a, b in zip(KEYS, dev, ref):
            assert np.array_equal(a, b), (mode, k)
    assert times["heavy"] < times["global"]
