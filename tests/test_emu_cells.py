"""The device cell algorithm (csrc/pf_cell.cuh), compiled for the host under
the lock-step warp emulator (tests/emu, test infrastructure), against the
reference's golden outputs: the warp-cooperative build is bit-exact and the
evaluation agrees to 1e-12.  Runs on CPU, no GPU needed."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, golden_domain, golden_scene

sys.path.insert(0, os.path.join(ROOT, "tests", "emu"))
import pyemu  # noqa: E402

NAMES = ["sparse", "sparse_varpsi", "sparse_full", "dense", "twofluid", "lattice_ties"]
EXACT = ("status", "fcount", "ftag", "fh", "fnrm")
CLOSE = ("vol", "ksur", "farea", "m2")  # relative 1e-10 (bar: 1e-9)
POS = ("cent", "fcent", "ipt")  # absolute 1e-10 in the unit domain


def grid_for(pts, psi, dpsi):
    br = np.sqrt(np.maximum(psi, 0)) + np.sqrt(np.maximum(psi, 0) + dpsi)
    H = max(float(np.mean(br)) * 0.5, 1e-6)
    gn = np.clip(np.ceil(1.0 / H).astype(int), 1, 256)
    return np.zeros(3), np.full(3, float(gn)), np.full(3, gn)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("tier", [0, 1, 2])
def test_emulated_kernel_vs_reference(golden, name, tier):
    s = golden_scene(golden, name)
    lo, ih, gn = grid_for(s["pts"], s["psi"], float(s["dpsi"]))
    e = pyemu.evaluate(s["pts"], s["psi"], golden_domain(golden), float(golden["dom_unit_tol"]),
                       lo, ih, gn, float(s["dpsi"]), ball_aware=bool(s["ball_aware"]),
                       smf=int(golden["ev_smf"]), t_init=0.05 ** 2, tier=tier, seed=17 + tier)
    assert e["err"] == int(s["err"]), "flag word / emulator divergence"
    for k in EXACT:
        assert np.array_equal(e[k], s[k]), k
    psi_max = float(np.max(s["psi"]))
    floor = {"vol": psi_max ** 1.5 * 1e-3, "ksur": psi_max * 1e-3, "farea": psi_max * 1e-3,
             "m2": psi_max ** 2.5 * 1e-3}
    for k in CLOSE:
        rel = np.abs(e[k] - s[k]) / np.maximum(np.abs(s[k]), floor[k])
        assert float(np.max(rel)) <= 1e-10, k
    for k in POS:
        assert float(np.max(np.abs(e[k] - s[k]))) <= 1e-10, k
