"""The CPU oracle (oracle/potflow_oracle.c) is pinned against outputs of the
reference itself (tests/golden/reference_kernels.npz, made by
tests/golden/make_golden.py): every output bit-identical."""
import numpy as np
import pytest

from conftest import OUT_KEYS, golden_domain, golden_scene
from oracle import pyoracle as O

NAMES = ["sparse", "sparse_varpsi", "sparse_full", "dense", "twofluid", "lattice_ties"]


@pytest.mark.parametrize("name", NAMES)
def test_batch_evaluate_bitwise(golden, name):
    s = golden_scene(golden, name)
    dom = golden_domain(golden)
    smf = int(golden["ev_smf"])
    g = O.SpatialGrid(s["pts"], [0, 0, 0], [1, 1, 1], float(golden["dom_unit_vol"]))
    o = O.evaluate(s["pts"], s["psi"], dom, float(golden["dom_unit_tol"]), g,
                   ball_aware=bool(s["ball_aware"]), want_m2=True, smf=smf, dpsi=float(s["dpsi"]))
    assert o["err"] == int(s["err"])
    for k in OUT_KEYS:
        assert np.array_equal(o[k], s[k]), k


def test_grid_matches_reference(golden):
    s = golden_scene(golden, "sparse")
    g = O.SpatialGrid(s["pts"], [0, 0, 0], [1, 1, 1], float(golden["dom_unit_vol"]))
    assert np.array_equal(g.dims, golden["grid_dims"])
    assert np.array_equal(g.bucket_start, golden["grid_bucket_start"])
    assert np.array_equal(g.bucket_sites, golden["grid_bucket_sites"])


def test_knn_matches_reference(golden):
    s = golden_scene(golden, "sparse")
    g = O.SpatialGrid(s["pts"], [0, 0, 0], [1, 1, 1], float(golden["dom_unit_vol"]))
    for q, k, ref in zip(golden["knn_q"], golden["knn_k"], golden["knn_idx"]):
        out = np.empty(int(k), np.int64)
        got = O.knn_kernel(g.points, *g.kernel_args(), *q, int(k), out)
        assert got == k
        assert np.array_equal(out, ref[:k])


@pytest.mark.parametrize("mode", ["ba", "full"])
def test_batch_build_matches_reference(golden, mode):
    pts, psi = golden["bb_pts"], golden["bb_psi"]
    n = len(pts)
    dom = golden_domain(golden)
    g = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], float(golden["dom_unit_vol"]))
    smv, smf, sml = golden[f"bb_{mode}_verts"].shape[1], golden[f"bb_{mode}_planes"].shape[1], \
        golden[f"bb_{mode}_lv"].shape[1]
    arrs = [np.zeros(n, np.int64) for _ in range(4)] + [
        np.zeros((n, smv, 3)), np.zeros((n, smf, 4)), np.zeros((n, smf), np.int64),
        np.zeros((n, smf + 1), np.int64), np.zeros((n, sml), np.int64)]
    err = O.batch_build(pts, psi, *dom, *g.kernel_args(), float(golden["dom_unit_tol"]),
                        O.dpsi_max(psi), mode == "ba", smv, smf, sml, *arrs)
    assert err == 0
    for k, a in zip(("status", "nv", "nf", "nl", "verts", "planes", "tags", "lp", "lv"), arrs):
        assert np.array_equal(a, golden[f"bb_{mode}_{k}"]), k
