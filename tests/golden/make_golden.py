"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It copies /root/reference/pkg to a scratch directory (numba's cache must not
write into the read-only tree), imports ``potflow`` from there and records
inputs and outputs of the reference's own kernels:

* ``_batch_evaluate`` (_kernels.py:1362-1478) on six small scenes
* ``_batch_build``    (_kernels.py:1481-1559) in ball-aware and full mode
* ``_knn`` / ``laguerre.knn`` (_kernels.py:1562-1620) on random queries
* ``SpatialGrid``     (laguerre.py:45-87) bucket CSR
* ``domain_pack``     (laguerre.py:113-139) of two boxes
* SPEC known-answer values computed through the reference API (SPEC.md examples)

The fixtures travel with the repo (tests/golden/*.npz); nothing at test time
reads /root/reference.
"""
from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"


def import_reference():
    tmp = tempfile.mkdtemp(prefix="potflow_ref_")
    shutil.copytree(REF, os.path.join(tmp, "pkg"))
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tmp, "nbcache"))
    sys.path.insert(0, os.path.join(tmp, "pkg", "src"))
    import potflow  # noqa: F401
    from potflow import _kernels, geom, laguerre

    return geom, laguerre, _kernels


def lattice(m, lo, h, rng, jitter=0.05):
    ax = [lo[a] + (np.arange(m[a]) + 0.5) * h for a in range(3)]
    P = np.stack(np.meshgrid(*ax, indexing="ij"), -1).reshape(-1, 3)
    return P + rng.uniform(-jitter * h, jitter * h, P.shape) if jitter else P


def scenes():
    rng = np.random.default_rng(12345)
    n = 1500
    pts = rng.random((n, 3))
    psi = np.full(n, (3 * (0.3 / n) / (4 * np.pi)) ** (2 / 3))
    yield "sparse", pts, psi, True
    yield "sparse_varpsi", pts, psi * (1 + 0.6 * rng.random(n)), True
    yield "sparse_full", pts[:400], psi[:400] * 3.0, False
    m = 10
    h = 0.5 / m
    r7 = np.random.default_rng(7)
    P = lattice((m, m, m), (0, 0, 0), h, r7)
    yield "dense", P, (0.8 * h + 0.1 * h * r7.random(len(P))) ** 2, True
    hA = 0.5 / 10
    A = lattice((10, 10, 5), (0, 0, 0), hA, r7)
    B = lattice((5, 5, 3), (0, 0, 0.25), 2 * hA, r7)
    P2 = np.concatenate([A, B])
    psi2 = np.concatenate([np.full(len(A), (0.85 * hA) ** 2), np.full(len(B), (1.7 * hA) ** 2)])
    yield "twofluid", P2, psi2, True
    P3 = lattice((6, 6, 6), (0.2, 0.2, 0.2), 0.1, r7, jitter=0.0)
    yield "lattice_ties", P3, np.full(len(P3), 0.085 ** 2), True


def main():
    geom, laguerre, K = import_reference()
    out = {}
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dp = laguerre.domain_pack(dom)
    for k, a in zip(("dv", "dc", "dp", "dt", "dlp", "dlv"), dp.args()):
        out[f"dom_unit_{k}"] = a
    out["dom_unit_tol"] = np.array(dp.tol)
    out["dom_unit_vol"] = np.array(dp.volume)
    dom2 = geom.box_domain([-0.3, 0.1, 0.2], [0.7, 0.4, 2.5])
    dp2 = laguerre.domain_pack(dom2)
    for k, a in zip(("dv", "dc", "dp", "dt", "dlp", "dlv"), dp2.args()):
        out[f"dom_aniso_{k}"] = a
    out["dom_aniso_tol"] = np.array(dp2.tol)
    dp = laguerre.domain_pack(dom)
    smf = 16
    names = []
    for name, pts, psi, ba in scenes():
        pts = np.ascontiguousarray(pts)
        n = len(pts)
        g = laguerre.SpatialGrid(pts, dom)
        o = dict(status=np.zeros(n, np.int64), vol=np.zeros(n), ksur=np.zeros(n),
                 cent=np.zeros((n, 3)), ipt=np.zeros((n, 3)), m2=np.zeros(n),
                 fcount=np.zeros(n, np.int64), ftag=np.zeros((n, smf), np.int64),
                 farea=np.zeros((n, smf)), fh=np.zeros((n, smf)),
                 fnrm=np.zeros((n, smf, 3)), fcent=np.zeros((n, smf, 3)))
        dpsi = laguerre._dpsi_max(psi)
        err = K._batch_evaluate(pts, psi, *dp.args(), *g.kernel_args(), dp.tol, dpsi, ba, True,
                                smf, *o.values())
        out[f"ev_{name}_pts"] = pts
        out[f"ev_{name}_psi"] = psi
        out[f"ev_{name}_ball_aware"] = np.array(ba)
        out[f"ev_{name}_dpsi"] = np.array(dpsi)
        out[f"ev_{name}_err"] = np.array(err)
        for k, v in o.items():
            out[f"ev_{name}_{k}"] = v
        names.append(name)
        print(name, n, "err", err, "fcount mean", o["fcount"].mean())
    out["ev_names"] = np.array(names)
    out["ev_smf"] = np.array(smf)
    # grid + knn on the sparse scene
    rng = np.random.default_rng(1)
    pts = out["ev_sparse_pts"]
    g = laguerre.SpatialGrid(pts, dom)
    out["grid_bucket_start"] = g.bucket_start
    out["grid_bucket_sites"] = g.bucket_sites
    out["grid_dims"] = g.dims
    q = rng.random((40, 3))
    ks = rng.integers(1, 30, 40)
    knn = np.full((40, 30), -1, np.int64)
    for t in range(40):
        r = laguerre.knn(g, q[t], int(ks[t]))
        knn[t, :len(r)] = r
    out["knn_q"] = q
    out["knn_k"] = ks
    out["knn_idx"] = knn
    # batch_build (unrestricted cells), both modes, on a small cloud
    pts_b = np.ascontiguousarray(np.random.default_rng(3).random((300, 3)))
    psi_b = np.random.default_rng(4).random(300) * 1e-3
    out["bb_pts"] = pts_b
    out["bb_psi"] = psi_b
    for ba in (True, False):
        bd = laguerre.build_diagram_packed((pts_b, psi_b), dom, ball_aware=ba)
        tagk = "ba" if ba else "full"
        for k in ("status", "nv", "nf", "nl", "verts", "planes", "tags", "lp", "lv"):
            out[f"bb_{tagk}_{k}"] = getattr(bd, k)
    # SPEC known answers through the reference API (SPEC.md examples)
    cube = dom
    half = geom.clip_cell(cube, geom.Plane(np.array([1.0, 0, 0]), 0.5))
    corner = geom.clip_cell(cube, geom.Plane(np.array([1.0, 1.0, 1.0]), 2.5))
    out["spec_half_volume"] = np.array(geom.cell_volume_convex(half))
    out["spec_corner_volume"] = np.array(geom.cell_volume_convex(corner))
    out["spec_corner_nfacets"] = np.array(corner.n_facets)
    np.savez_compressed(os.path.join(HERE, "reference_kernels.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_kernels.npz"),
          os.path.getsize(os.path.join(HERE, "reference_kernels.npz")) // 1024, "KiB")


if __name__ == "__main__":
    main()
