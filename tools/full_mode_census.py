"""Unrestricted diagram (full security-radius mode, _batch_build) on whole
scenes: the device's packed cells against the CPU oracle (bit-identical to
the numba reference), every array bit for bit -- with the heavy-site phase
 active -- plus a scene with a few huge weights.
usage: full_mode_census.py KIND [KIND ...]   KIND: c2c c5c heavy"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import _kernels, geom, laguerre
    from parity_census import scene_psi

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
    keys = ("status", "nv", "nf", "nl", "verts", "planes", "tags", "lp", "lv")
    for kind in sys.argv[1:]:
        if kind == "heavy":
            rng = np.random.default_rng(21)
            n = 100000  # the oracle (the reference's global security radius) visits ~n/4 sites per cell
            pts = rng.random((n, 3))
            psi = np.full(n, (0.6 * (1.0 / n) ** (1.0 / 3.0)) ** 2)
            psi[[5, 1234, 2999, 77777]] = (0.3, 0.12, 0.05, 0.02)
            what = "100k random sites, 4 huge weights"
        else:
            sc, psi, what = scene_psi(kind)
            pts = np.ascontiguousarray(sc.pts)
            n = sc.n
        dpsi = float(psi.max() - psi.min())
        smv, smf, sml = 512, 160, 2048  # the reference's capacities (~4.5 KB per cell per array set)

        def arrays():
            return [np.zeros(n, np.int64) for _ in range(4)] + [
                np.zeros((n, smv, 3)), np.zeros((n, smf, 4)), np.zeros((n, smf), np.int64),
                np.zeros((n, smf + 1), np.int64), np.zeros((n, sml), np.int64)]

        dev = arrays()
        t0 = time.perf_counter()
        e_dev = _kernels._batch_build(pts, psi, *dpk.args(), *gargs, dpk.tol, dpsi, False, smv, smf, sml, *dev)
        t_dev = time.perf_counter() - t0
        ref = arrays()
        g = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], dpk.volume)
        t0 = time.perf_counter()
        e_ref = O.batch_build(pts, psi, *dpk.args(), *g.kernel_args(), dpk.tol, dpsi, False, smv, smf, sml, *ref)
        t_ref = time.perf_counter() - t0
        bad = {k: int(np.sum(np.any((a != b).reshape(n, -1), axis=1))) for k, a, b in zip(keys, dev, ref)}
        print(f"{kind} n={n} ({what}): flags device {e_dev} oracle {e_ref}; cells differing per array {bad}; "
              f"device {t_dev:.2f} s (incl. host copies), oracle {t_ref:.1f} s ({os.cpu_count()} threads)", flush=True)


if __name__ == "__main__":
    main()
