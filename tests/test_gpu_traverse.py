"""Cell-to-cell traversal (SPEC.md renderer `traverse`, §6) against
brute force: the pieces partition the ray's chord of the domain, each lies in
its power cell, the fluid pieces are the ray inside the union of the balls
(the fluid = union of V_i ∩ B_i), and SurfaceOnly stops at the first exit
through a sphere.  SPEC examples: an axis ray through a 2-cell domain gives 2
spans summing to the chord."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _chord(o, d):
    """[t0, t1] of the ray in the unit box."""
    with np.errstate(divide="ignore", invalid="ignore"):
        ta, tb = (0.0 - o) / d, (1.0 - o) / d
    lo, hi = np.minimum(ta, tb), np.maximum(ta, tb)
    return max(0.0, float(np.max(lo))), float(np.min(hi))


def _union_intervals(o, d, pts, psi, t0, t1):
    w = o[None, :] - pts
    b = w @ d
    c = np.sum(w * w, axis=1) - psi
    disc = b * b - c
    iv = []
    for k in np.nonzero((disc > 0) & (psi > 0))[0]:
        s = np.sqrt(disc[k])
        a, e = max(-b[k] - s, t0), min(-b[k] + s, t1)
        if a < e:
            iv.append((a, e))
    iv.sort()
    out = []
    for a, e in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([a, e])
    return out


def test_two_cell_axis_ray():
    from paper_2601_05765_b200 import render

    pts = np.array([[0.25, 0.5, 0.5], [0.75, 0.5, 0.5]])
    psi = np.array([0.01, 0.04])
    tr = render.traverse(pts, psi, [[-1.0, 0.5, 0.5]], [[1.0, 0.0, 0.0]])
    assert tr.status[0] == 0
    path = tr.path(0)
    spans = {}
    for cell, a, b, _ in path:
        spans.setdefault(cell, []).append((a, b))
    assert list(spans) == [0, 1]  # two cells, in order
    assert abs(path[0][1] - 1.0) < 1e-12 and abs(path[-1][2] - 2.0) < 1e-12  # the chord [1, 2]
    assert sum(b - a for _, a, b, _ in path) == pytest.approx(1.0, abs=1e-12)
    # the power bisector of the two sites: x = 0.5 + (psi_0 - psi_1) / (2 * 0.5) = 0.47
    assert spans[0][-1][1] == pytest.approx(1.47, abs=1e-12)
    # fluid: the two balls' chords, [0.15, 0.35] and [0.55, 0.95] along x
    assert tr.fluid_length()[0] == pytest.approx(0.2 + 0.4, abs=1e-12)


def test_random_rays_against_brute_force():
    from paper_2601_05765_b200 import render

    rng = np.random.default_rng(3)
    n = 600
    pts = rng.random((n, 3))
    psi = (rng.uniform(0.3, 1.2, n) * (1.0 / n) ** (1.0 / 3.0)) ** 2
    m = 300
    o = rng.uniform(-0.5, 1.5, (m, 3))
    tgt = rng.random((m, 3))
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    tr = render.traverse(pts, psi, o, d)
    sur = render.traverse(pts, psi, o, d, mode="surface")
    for r in range(m):
        t0, t1 = _chord(o[r], d[r])
        assert tr.status[r] == 0
        path = tr.path(r)
        assert path[0][1] == pytest.approx(t0, abs=1e-9) and path[-1][2] == pytest.approx(t1, abs=1e-9)
        for (c0, a0, b0, f0), (c1, a1, b1, f1) in zip(path, path[1:]):
            assert b0 == a1  # consecutive pieces share their end points
        assert sum(b - a for _, a, b, _ in path) == pytest.approx(t1 - t0, abs=1e-8)
        for cell, a, b, fl in path:
            x = o[r] + 0.5 * (a + b) * d[r]
            pd = np.sum((x - pts) ** 2, axis=1) - psi
            if b - a > 1e-9:
                assert pd[cell] <= pd.min() + 1e-12, "piece outside its power cell"
                assert fl == (pd[cell] < 0.0) or abs(pd[cell]) < 1e-12
        union = _union_intervals(o[r], d[r], pts, psi, t0, t1)
        assert tr.fluid_length()[r] == pytest.approx(sum(e - a for a, e in union), abs=1e-9)
        # SurfaceOnly: up to the first exit through a sphere patch
        sp = sur.path(r)
        if union and union[0][1] < t1 - 1e-9:
            assert sp[-1][3] and sp[-1][2] == pytest.approx(union[0][1], abs=1e-9)
        elif not union:
            assert sp[-1][2] == pytest.approx(t1, abs=1e-9)


def test_ray_missing_the_domain():
    from paper_2601_05765_b200 import render

    pts = np.array([[0.5, 0.5, 0.5]])
    tr = render.traverse(pts, np.array([0.01]), [[2.0, 2.0, 2.0]], [[1.0, 0.0, 0.0]])
    assert tr.status[0] == 1 and tr.count[0] == 0
