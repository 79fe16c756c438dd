"""Whole-scene parity census vs the CPU oracle (bit-identical to the numba
reference): every cell of a configuration, device vs oracle, in parity mode
and/or the robust default.

usage: parity_census.py CFG [CFG ...] [--mode parity|robust|both] [--mc]

CFG: c1 c2 c3 c4 c5 (cold-start / fixed weights) or c1c c2c c3c c4c c5c (the
config's Newton-converged weights: the committed fixture tests/golden/psi_<C>.npz
when present -- the bench workload -- else a device solve).  Prints one line
per (config, mode): adjacency mismatches (status, fcount, ordered ftag) and
cells whose volume / free surface / facet areas differ by > 1e-9 relative.
In robust mode the differing cells are arbitrated (twin-facet symmetry; with
--mc a Monte-Carlo volume)."""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def scene_psi(which):
    import torch

    from paper_2601_05765_b200 import geom, scenes, solver

    cfg = which[:2].upper()
    sc = scenes.make(cfg)
    if which.endswith("c"):
        fx = os.path.join(ROOT, "tests", "golden", f"psi_{cfg}.npz")
        if os.path.exists(fx):
            return sc, np.load(fx)["psi"].astype(np.float64), "fixture " + os.path.relpath(fx, ROOT)
        res = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"),
                                  geom.box_domain([0, 0, 0], [1, 1, 1]))
        return sc, res.psi.cpu().numpy(), "device Newton solve"
    if cfg in ("C2", "C4"):
        return sc, np.full(sc.n, (0.85 * sc.meta["h"]) ** 2), "(0.85 h)^2"
    if cfg == "C5":
        h = sc.meta["h"]
        return sc, np.where(sc.nu > h ** 3 * 1.5, (1.7 * h) ** 2, (0.85 * h) ** 2), "(0.85 h)^2 / (1.7 h)^2"
    return sc, sc.psi_cold(), "cold start"


def compare(o, r, psi):
    adj = np.all(o["ftag"] == r["ftag"], axis=1) & (o["fcount"] == r["fcount"]) & (o["status"] == r["status"])
    sph = 4 * np.pi * psi
    dv = np.abs(o["vol"] - r["vol"]) / np.maximum(np.abs(r["vol"]), sph ** 1.5 * 1e-6)
    dk = np.abs(o["ksur"] - r["ksur"]) / sph
    da = np.max(np.abs(o["farea"] - r["farea"]), axis=1) / sph
    bad = (dv > 1e-9) | (dk > 1e-9) | (da > 1e-9)
    return adj, bad, dv, dk, da


def arbitrate(sc, psi, o, r, b, dv, mc):
    sph = 4 * np.pi * psi

    def twin_area(src, j, i):
        row = src["ftag"][j][: src["fcount"][j]].tolist()
        return src["farea"][j][row.index(i)] if i in row else 0.0

    dev_better = ora_better = ties = 0
    for i in b:
        for s in range(r["fcount"][i]):
            j = int(r["ftag"][i, s])
            if j < 0 or abs(o["farea"][i, s] - r["farea"][i, s]) <= 1e-9 * sph[i]:
                continue
            td, to = twin_area(o, j, i), twin_area(r, j, i)
            ed, eo = abs(o["farea"][i, s] - td), abs(r["farea"][i, s] - to)
            if ed < 0.5 * eo:
                dev_better += 1
            elif eo < 0.5 * ed:
                ora_better += 1
            else:
                ties += 1
    print(f"    facets differing: device closer to its twin {dev_better}, reference closer {ora_better}, "
          f"undecided {ties}")
    if not mc:
        return
    from scipy.spatial import cKDTree

    big = b[dv[b] > 1e-3][:40]
    if len(big):
        C = float(psi.max()) * 1.0001
        lift = np.concatenate([sc.pts, np.sqrt(np.maximum(C - psi, 0.0))[:, None]], 1)
        tree = cKDTree(lift)
        rng = np.random.default_rng(0)
        dev_ok = ora_ok = 0
        for i in big:
            R = np.sqrt(psi[i]); N = 200_000
            u = rng.normal(size=(N, 3)); u /= np.linalg.norm(u, axis=1)[:, None]
            x = sc.pts[i] + u * (R * rng.random(N) ** (1 / 3))[:, None]
            x = x[np.all((x >= 0) & (x <= 1), axis=1)]
            _, nn = tree.query(np.concatenate([x, np.zeros((len(x), 1))], 1))
            p = np.mean(nn == i) * len(x) / N
            vmc = (4 / 3) * np.pi * R ** 3 * p
            sd = (4 / 3) * np.pi * R ** 3 * np.sqrt(max(p * (1 - p), 1e-12) / N)
            dev_ok += abs(o["vol"][i] - vmc) / sd < 4
            ora_ok += abs(r["vol"][i] - vmc) / sd < 4
        print(f"    Monte-Carlo (2e5 samples) on {len(big)} cells differing > 1e-3: device within 4 sigma {dev_ok}, "
              f"reference within 4 sigma {ora_ok}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", nargs="+")
    ap.add_argument("--mode", default="both", choices=["parity", "robust", "both"])
    ap.add_argument("--mc", action="store_true")
    a = ap.parse_args()
    import torch

    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre, restricted

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    modes = ["parity", "robust"] if a.mode == "both" else [a.mode]
    for which in a.which:
        sc, psi, src = scene_psi(which)
        t0 = time.perf_counter()
        g = O.SpatialGrid(sc.pts, [0, 0, 0], [1, 1, 1], 1.0)
        r = O.evaluate(sc.pts, psi, dpk.args(), dpk.tol, g, smf=32)
        t_cpu = time.perf_counter() - t0
        for mode in modes:
            d = restricted.evaluate(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(psi, device="cuda"),
                                    dom, smf=32, parity_mode=mode == "parity")
            o = {k: getattr(d, k).cpu().numpy() for k in ("status", "fcount", "ftag", "vol", "ksur", "farea")}
            adj, bad, dv, dk, da = compare(o, r, psi)
            print(f"{which} [{mode}] n={sc.n} psi={src}: adjacency mismatches={int((~adj).sum())} "
                  f"value mismatches(>1e-9)={int(bad.sum())} ({100 * bad.mean():.4f}%)  max vol rel {dv.max():.3e}  "
                  f"max ksur/sph {dk.max():.3e}  max farea/sph {da.max():.3e}  (oracle {t_cpu:.1f} s, "
                  f"{O.num_threads()} threads)", flush=True)
            b = np.nonzero(bad)[0]
            if mode == "robust" and len(b):
                arbitrate(sc, psi, o, r, b, dv, a.mc)


if __name__ == "__main__":
    main()
