"""Cells where the reference's restriction emits a degenerate arc (end points
within tolerance, clockwise by rounding) whose sweep wraps to ~2 pi.  The
reference's volume for these cells is off by ~20%; Monte-Carlo (800k samples)
gives the true volume.  The device algorithm (run here through the host warp
emulator) corrects exactly these arcs and lands on the Monte-Carlo volume,
while facet adjacency stays identical to the reference.

Fixture: tests/golden/degenerate_arcs.npz (make_degenerate.py)."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT
from oracle import pyoracle as O
from paper_2601_05765_b200 import geom, laguerre

sys.path.insert(0, os.path.join(ROOT, "tests", "emu"))
import pyemu  # noqa: E402

FIX = os.path.join(ROOT, "tests", "golden", "degenerate_arcs.npz")
DOM = geom.box_domain([0, 0, 0], [1, 1, 1])
DPK = laguerre.domain_pack(DOM)


def _cells():
    g = np.load(FIX)
    return [int(c) for c in g["cells"]]


@pytest.mark.parametrize("cell", _cells())
def test_degenerate_arc_cells(cell):
    g = np.load(FIX)
    pts, psi, loc = g[f"c{cell}_pts"], g[f"c{cell}_psi"], int(g[f"c{cell}_local"])
    dpsi = float(g["dpsi"])
    # the oracle reproduces the reference's (wrong) volume bit for bit
    grid = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    o = O.evaluate(pts, psi, DPK.args(), DPK.tol, grid, smf=32, i0=0, i1=1, cells=np.array([loc]),
                   dpsi=dpsi)
    assert o["vol"][loc] == float(g[f"c{cell}_ref_vol"])
    mc, se = float(g[f"c{cell}_mc_vol"]), float(g[f"c{cell}_mc_se"])
    assert abs(o["vol"][loc] - mc) > 20 * se  # the reference is provably off
    gn = np.array([128, 128, 128])
    e = pyemu.evaluate(pts, psi, DPK.args(), DPK.tol, np.zeros(3), gn.astype(float), gn, dpsi,
                       smf=32, tier=0, seed=3)
    assert abs(e["vol"][loc] - mc) < 4 * se, (e["vol"][loc], mc, se)
    # adjacency unchanged
    assert e["fcount"][loc] == o["fcount"][loc]
    assert np.array_equal(e["ftag"][loc], o["ftag"][loc])


@pytest.mark.parametrize("cell", _cells())
def test_degenerate_arc_cells_parity_mode(cell):
    """Parity mode reproduces the reference's outcome on the same cells: the
    spurious entry and the wrapped arc are kept, and the volume, free surface
    and facet areas equal the reference's to 1e-9."""
    g = np.load(FIX)
    pts, psi, loc = g[f"c{cell}_pts"], g[f"c{cell}_psi"], int(g[f"c{cell}_local"])
    dpsi = float(g["dpsi"])
    grid = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    o = O.evaluate(pts, psi, DPK.args(), DPK.tol, grid, smf=32, i0=0, i1=1, cells=np.array([loc]),
                   dpsi=dpsi)
    gn = np.array([128, 128, 128])
    e = pyemu.evaluate(pts, psi, DPK.args(), DPK.tol, np.zeros(3), gn.astype(float), gn, dpsi,
                       smf=32, tier=0, seed=3, parity_mode=True)
    assert e["fcount"][loc] == o["fcount"][loc]
    assert np.array_equal(e["ftag"][loc], o["ftag"][loc])
    assert e["status"][loc] == o["status"][loc]
    sph = 4 * np.pi * psi[loc]
    assert abs(e["vol"][loc] - o["vol"][loc]) <= 1e-9 * abs(o["vol"][loc])
    assert abs(e["ksur"][loc] - o["ksur"][loc]) <= 1e-9 * sph
    assert float(np.max(np.abs(e["farea"][loc] - o["farea"][loc]))) <= 1e-9 * sph
