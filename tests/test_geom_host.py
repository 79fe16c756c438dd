"""Host geometry (domain packing) equals the reference's, and SPEC known answers."""
import numpy as np

from conftest import golden_domain
from oracle import pyoracle as O
from paper_2601_05765_b200 import geom, laguerre


def test_domain_pack_bitwise(golden):
    for which, lo, hi in (("unit", [0, 0, 0], [1, 1, 1]), ("aniso", [-0.3, 0.1, 0.2], [0.7, 0.4, 2.5])):
        dp = laguerre.domain_pack(geom.box_domain(lo, hi))
        for a, b in zip(dp.args(), golden_domain(golden, which)):
            assert np.array_equal(a, b)
        assert dp.tol == float(golden[f"dom_{which}_tol"])


def _clip(cell, n, d, tag=-1):
    va, ca, pa, ta, lpa, lva = geom.pack_cell(cell)
    out = [np.empty_like(a) for a in (va, ca, pa, ta, lpa, lva)]
    tol = geom.DEFAULT_REL_TOL * max(cell.diagonal(), 1.0)
    st = O.clip_into(va, ca, pa, ta, lpa, lva, *out, n[0], n[1], n[2], d, tag, tol)
    return st, (geom.unpack_cell(*out) if st == 0 else None)


def test_spec_clip_examples(golden):
    cube = geom.box_domain([0, 0, 0], [1, 1, 1])
    assert cube.n_vertices == 8 and cube.n_facets == 6 and cube.n_edges() == 12
    st, half = _clip(cube, [1.0, 0, 0], 0.5)
    assert st == 0 and abs(geom.cell_volume_convex(half) - 0.5) < 1e-15
    assert geom.cell_volume_convex(half) == float(golden["spec_half_volume"])
    st, _ = _clip(cube, [1.0, 0, 0], 2.0)
    assert st == 1  # plane outside the cell: untouched
    nrm = np.array([1.0, 1.0, 1.0]) / np.sqrt(3.0)
    st, corner = _clip(cube, nrm, 2.5 / np.sqrt(3.0))
    assert st == 0 and corner.n_facets == int(golden["spec_corner_nfacets"]) == 7
    assert abs(geom.cell_volume_convex(corner) - (1 - 0.5 ** 3 / 6)) < 1e-12
    corner.validate()
    # idempotence (SPEC geom invariants)
    st2, _ = _clip(corner, nrm, 2.5 / np.sqrt(3.0))
    assert st2 == 1


def test_spec_polygon_integrals():
    # full circle r=2 -> 4 pi; half disk r=1 -> pi/2 with centroid 4/(3 pi)
    A, *_ = O.piece_integrals(np.array([[2.0, 0, 0, 0, 0, 0, 0, 2.0, 0, 0]]), 1)
    assert abs(A - 4 * np.pi) < 1e-12
    rows = np.array([[0.0, 1, 0, -1, 0, 0, 0, 0, 0, 0], [1.0, 0, 0, 0, 0, 0, 0, 1.0, np.pi, 2 * np.pi]])
    A, Mx, My, Ip = O.piece_integrals(rows, 2)
    assert abs(A - np.pi / 2) < 1e-12 and abs(My / A + 4 / (3 * np.pi)) < 1e-12


def test_tetra_and_box_volume():
    planes = [geom.Plane([-1.0, 0, 0], 0.0), geom.Plane([0, -1.0, 0], 0.0),
              geom.Plane([0, 0, -1.0], 0.0), geom.Plane([1.0, 1.0, 1.0], 1.0)]
    tet = geom.init_cell_from_domain(planes)
    assert tet.n_vertices == 4 and abs(geom.cell_volume_convex(tet) - 1 / 6) < 1e-15
