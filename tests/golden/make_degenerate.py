"""Extract small neighbourhoods around cells where the reference's restriction
produces a degenerate arc (an exit/entry pair within tolerance whose sweep
wraps to ~2 pi), for tests/test_degenerate_arcs.py.

Provenance: C4 (2M droplet, paper_2601_05765_b200.scenes.c4_droplet) weights
after 6 iterations of the CPU Newton restatement (oracle/newton_ref.py,
cold start) -- the state in which the SPEC Newton stalls because these cells'
volumes are wrong (SURVEY/DESIGN: "degenerate arcs").  Usage:

    python tests/golden/make_degenerate.py /path/to/c4_psi.npy
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as O  # noqa: E402
from paper_2601_05765_b200 import geom, laguerre, scenes  # noqa: E402

CELLS = [712342, 1287224, 1466507, 820715]


def mc_volume(pts, psi, i, rng, m=800_000):
    p, r = pts[i], np.sqrt(psi[i])
    x = p + rng.uniform(-r, r, (m, 3))
    x = x[((x - p) ** 2).sum(1) <= psi[i]]
    nb = np.nonzero(((pts - p) ** 2).sum(1) < (3 * r + 0.02) ** 2)[0]
    pw = ((x[:, None, :] - pts[nb][None]) ** 2).sum(2) - psi[nb][None]
    own = (nb[np.argmin(pw, 1)] == i) & np.all((x >= 0) & (x <= 1), 1)
    f = own.mean()
    vb = 4 / 3 * np.pi * r ** 3
    return f * vb, np.sqrt(f * (1 - f) / len(x)) * vb


def main(psi_path):
    s = scenes.c4_droplet()
    psi = np.load(psi_path)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    dpsi = O.dpsi_max(psi)
    g = O.SpatialGrid(s.pts, [0, 0, 0], [1, 1, 1], 1.0)
    rng = np.random.default_rng(0)
    out = {"dpsi": np.array(dpsi), "cells": np.array(CELLS)}
    for c in CELLS:
        o = O.evaluate(s.pts, psi, dpk.args(), dpk.tol, g, smf=32, i0=0, i1=1,
                       cells=np.array([c]), dpsi=dpsi)
        near = np.nonzero(((s.pts - s.pts[c]) ** 2).sum(1) < 0.012 ** 2)[0]
        loc = int(np.nonzero(near == c)[0][0])
        vmc, se = mc_volume(s.pts, psi, c, rng)
        out[f"c{c}_pts"] = s.pts[near]
        out[f"c{c}_psi"] = psi[near]
        out[f"c{c}_local"] = np.array(loc)
        out[f"c{c}_ref_vol"] = np.array(o["vol"][c])
        out[f"c{c}_ref_err"] = np.array(o["err"])
        out[f"c{c}_mc_vol"] = np.array(vmc)
        out[f"c{c}_mc_se"] = np.array(se)
        out[f"c{c}_nu"] = np.array(s.nu[c])
        print(c, len(near), "ref vol/nu", o["vol"][c] / s.nu[c], "mc", vmc / s.nu[c], "+-", se / s.nu[c],
              "flags", o["err"])
    np.savez_compressed(os.path.join(HERE, "degenerate_arcs.npz"), **out)


if __name__ == "__main__":
    main(sys.argv[1])
