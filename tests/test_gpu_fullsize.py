"""Parity at the BASELINE.json sizes (C3 500k chocs, C4 2M droplet, C5 1M
two-fluid): the device evaluates every cell; the CPU oracle re-evaluates a
random sample of them (cells are independent, so a sample is an exact check
of those cells).  Size-independent properties are checked on all cells:
facet adjacency symmetric (i sees j <=> j sees i), facet areas equal from
both sides, run-to-run determinism.

Adjacency (status, fcount, ordered ftag) is bit-exact on every sampled cell.
Values agree to 1e-9 relative except on the cells of DESIGN.md §5.1 (the
reference's degenerate-arc / spurious-entry cases, where the device follows
the geometry and the oracle keeps the reference's wrong values): at most
0.05% of the sample."""
import numpy as np
import pytest

from conftest import OUT_KEYS

pytestmark = pytest.mark.gpu

REL = 1e-9


def _scene(kind):
    from paper_2601_05765_b200 import scenes

    if kind == "C3":
        sc = scenes.c3_chocs()
        return sc, sc.psi_cold()
    if kind in ("C3c", "C5c"):  # converged weights: large local weight spread (per-cell slack, mid tier)
        import torch

        from paper_2601_05765_b200 import geom, solver

        sc = scenes.c3_chocs() if kind == "C3c" else scenes.c5_two_fluid()
        res = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"),
                                  geom.box_domain([0, 0, 0], [1, 1, 1]))
        return sc, res.psi.cpu().numpy()
    if kind == "C4":
        sc = scenes.c4_droplet()
        return sc, np.full(sc.n, (0.85 * sc.meta["h"]) ** 2)
    sc = scenes.c5_two_fluid()
    h = sc.meta["h"]
    return sc, np.where(sc.nu > h ** 3 * 1.5, (1.7 * h) ** 2, (0.85 * h) ** 2)


@pytest.mark.parametrize("kind", ["C3", "C3c", "C4", "C5", "C5c"])
def test_full_size_sample_matches_oracle(kind):
    import torch

    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre, restricted

    sc, psi = _scene(kind)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    d = restricted.evaluate(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(psi, device="cuda"),
                            dom, smf=32)
    o = {k: getattr(d, k).cpu().numpy() for k in OUT_KEYS}
    rng = np.random.default_rng(1)
    cells = np.sort(rng.choice(sc.n, size=20_000, replace=False)).astype(np.int64)
    g = O.SpatialGrid(sc.pts, [0, 0, 0], [1, 1, 1], 1.0)
    r = O.evaluate(sc.pts, psi, dpk.args(), dpk.tol, g, smf=32, i0=0, i1=len(cells), cells=cells)
    for k in ("status", "fcount", "ftag"):
        assert np.array_equal(o[k][cells], r[k][cells]), k
    sph = 4 * np.pi * float(psi.max())
    dv = np.abs(o["vol"][cells] - r["vol"][cells]) / np.maximum(np.abs(r["vol"][cells]), sph ** 1.5 * 1e-6)
    da = np.max(np.abs(o["farea"][cells] - r["farea"][cells]) / sph, axis=1)
    bad = (dv > REL) | (da > REL)
    assert bad.sum() <= max(1, int(5e-4 * len(cells))), (kind, int(bad.sum()), float(dv.max()))
    ok = ~bad
    assert float(np.max(np.abs(o["ksur"][cells][ok] - r["ksur"][cells][ok]) / sph)) <= REL


@pytest.mark.parametrize("kind", ["C4"])
def test_full_size_symmetry_and_determinism(kind):
    import torch

    from paper_2601_05765_b200 import geom, restricted

    sc, psi = _scene(kind)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    tp, tw = torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(psi, device="cuda")
    a = restricted.evaluate(tp, tw, dom)
    b = restricted.evaluate(tp, tw, dom)
    for k in OUT_KEYS:
        assert torch.equal(getattr(a, k), getattr(b, k)), k
    n = sc.n
    ft, fa, fc = a.ftag.cpu().numpy(), a.farea.cpu().numpy(), a.fcount.cpu().numpy()
    used = (np.arange(ft.shape[1])[None, :] < fc[:, None]) & (ft >= 0)
    I = np.nonzero(used)[0].astype(np.int64)
    J = ft[used].astype(np.int64)
    A = fa[used]
    k1 = I * n + J
    o1 = np.argsort(k1)
    k1s = k1[o1]
    k2 = J * n + I
    pos = np.searchsorted(k1s, k2)
    pos = np.minimum(pos, len(k1s) - 1)
    found = k1s[pos] == k2
    sph = 4 * np.pi * float(psi.max())
    # every facet (i, j) has its twin (j, i), except slivers at the tolerance
    # (one side restricted to area 0 by the reference's tolerance predicates)
    lone = A[~found] / sph
    assert (~found).sum() <= 1e-6 * len(A) and (lone.max() if lone.size else 0.0) < 1e-7, \
        (int((~found).sum()), float(lone.max()) if lone.size else 0.0)
    twin = A[o1[pos]][found]
    # two-sided areas agree to < 1e-7 of the sphere area except on tolerance-level
    # slivers, where the reference is itself asymmetric (C4, oracle: pair
    # 1557572/1563799 has 3.678e-9 vs 3.096e-9, 5e-6 of the sphere area)
    dif = np.abs(A[found] - twin) / sph
    assert int((dif > 1e-7).sum()) <= 1e-6 * len(dif) and float(np.max(dif)) < 1e-4, \
        (float(np.max(dif)), int((dif > 1e-7).sum()))
