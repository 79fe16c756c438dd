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


@pytest.mark.parametrize("nheavy", [1, 3, 12])
def test_full_mode_heavy_site_phase_vs_reference(golden, nheavy):
    """Full (non-ball-aware) mode with one huge weight: the reference's global
    security radius makes every cell walk (almost) all n - 1 sites.  The
    device's heavy-site phase (build_cell) stops the
    ordinary stream at the ordinary sites' radius and takes the heavy site at
    its turn: the cells are the reference's bit for bit, for a fraction of the
    processed candidates."""
    sys.path.insert(0, ROOT)
    from oracle import pyoracle as O

    rng = np.random.default_rng(9)
    n = 300
    pts = rng.random((n, 3))
    psi = np.full(n, (0.6 * (1.0 / n) ** (1.0 / 3.0)) ** 2)
    # huge weights (ball radius up to 0.63 in the unit box); 12 > the device's
    # list of 8: the rest bound the ordinary sites' slack
    psi[17 + 11 * np.arange(nheavy)] = np.linspace(0.4, 0.1, nheavy)
    psi[40] = 0.5 * psi[0]
    dpsi = float(psi.max() - psi.min())
    dom, tol, smf = golden_domain(golden), float(golden["dom_unit_tol"]), int(golden["ev_smf"])
    ref = {k: np.zeros(s, t) for k, s, t in (
        ("status", n, np.int64), ("vol", n, np.float64), ("ksur", n, np.float64), ("cent", (n, 3), np.float64),
        ("ipt", (n, 3), np.float64), ("m2", n, np.float64), ("fcount", n, np.int64), ("ftag", (n, smf), np.int64),
        ("farea", (n, smf), np.float64), ("fh", (n, smf), np.float64), ("fnrm", (n, smf, 3), np.float64),
        ("fcent", (n, smf, 3), np.float64))}
    clips = np.zeros(n, np.int64)
    g = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    O.batch_evaluate(pts, psi, *dom, *g.kernel_args(), tol, dpsi, False, True, smf,
                     *[ref[k] for k in ("status", "vol", "ksur", "cent", "ipt", "m2", "fcount", "ftag", "farea",
                                        "fh", "fnrm", "fcent")], clip_count=clips)
    lo, ih, gn = grid_for(pts, psi, dpsi)
    e = pyemu.evaluate(pts, psi, dom, tol, lo, ih, gn, dpsi, ball_aware=False, smf=smf, t_init=0.05 ** 2,
                       tier=0, seed=5, parity_mode=True)
    for k in EXACT:
        assert np.array_equal(e[k], ref[k]), k
    psi_max = float(np.max(psi))  # relative to the value, floored as in the golden test above
    floor = {"vol": psi_max ** 1.5 * 1e-3, "ksur": psi_max * 1e-3, "farea": psi_max * 1e-3,
             "m2": psi_max ** 2.5 * 1e-3}
    for k in CLOSE:
        rel = np.abs(e[k] - ref[k]) / np.maximum(np.abs(ref[k]), floor[k])
        assert float(np.max(rel)) <= 1e-10, k
    print("processed candidates per cell: reference", np.mean(clips), "device", np.mean(e["census"]))
    if nheavy <= 8:
        assert np.mean(clips) > 0.35 * (n - 1)  # the pathology: the reference visits a large part of all sites
        assert np.mean(e["census"]) < 0.3 * np.mean(clips)  # the device: the cutting neighbourhood + heavy sites
