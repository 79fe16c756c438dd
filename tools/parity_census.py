"""Whole-scene parity census vs the CPU oracle (dev tool): how many cells
differ beyond 1e-9 and what they look like.  usage: parity_census.py c4|c3|c3c|c5|c5c|c2|c1c"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O
from paper_2601_05765_b200 import geom, laguerre, restricted, scenes
which = sys.argv[1] if len(sys.argv) > 1 else "c4"
if which == "c4":
    sc = scenes.c4_droplet(); psi = np.full(sc.n, (0.85 * sc.meta["h"]) ** 2)
elif which == "c2":
    sc = scenes.c2_dam_break(); psi = np.full(sc.n, (0.85 * sc.meta["h"]) ** 2)
elif which == "c3":
    sc = scenes.c3_chocs(); psi = sc.psi_cold()
elif which == "c1c":  # C1 10k random at its converged weights
    from paper_2601_05765_b200 import solver
    sc = scenes.c1_random()
    psi = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"),
                              geom.box_domain([0, 0, 0], [1, 1, 1])).psi.cpu().numpy()
elif which == "c5c":  # C5 two-fluid at its converged weights
    from paper_2601_05765_b200 import solver
    sc = scenes.c5_two_fluid()
    psi = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"),
                              geom.box_domain([0, 0, 0], [1, 1, 1])).psi.cpu().numpy()
elif which == "c3c":  # C3 at its converged weights (large local weight spread)
    from paper_2601_05765_b200 import solver
    sc = scenes.c3_chocs()
    psi = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"),
                              geom.box_domain([0, 0, 0], [1, 1, 1])).psi.cpu().numpy()
else:
    sc = scenes.c5_two_fluid(); h = sc.meta["h"]; psi = np.where(sc.nu > h ** 3 * 1.5, (1.7 * h) ** 2, (0.85 * h) ** 2)
dom = geom.box_domain([0, 0, 0], [1, 1, 1]); dpk = laguerre.domain_pack(dom)
d = restricted.evaluate(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(psi, device="cuda"), dom, smf=32)
o = {k: getattr(d, k).cpu().numpy() for k in ("status", "fcount", "ftag", "vol", "ksur", "farea")}
g = O.SpatialGrid(sc.pts, [0, 0, 0], [1, 1, 1], 1.0)
r = O.evaluate(sc.pts, psi, dpk.args(), dpk.tol, g, smf=32)
n = sc.n
adj = np.all(o["ftag"] == r["ftag"], axis=1) & (o["fcount"] == r["fcount"]) & (o["status"] == r["status"])
sph = 4 * np.pi * psi
dv = np.abs(o["vol"] - r["vol"]) / np.maximum(np.abs(r["vol"]), sph ** 1.5 * 1e-6)
dk = np.abs(o["ksur"] - r["ksur"]) / sph
da = np.max(np.abs(o["farea"] - r["farea"]), axis=1) / sph
bad = (dv > 1e-9) | (dk > 1e-9) | (da > 1e-9)
print(f"{which}: n={n} adjacency mismatches={int((~adj).sum())} value mismatches(>1e-9)={int(bad.sum())} "
      f"({100 * bad.mean():.4f}%)  max vol rel {dv.max():.3e}  max ksur/sph {dk.max():.3e}  max farea/sph {da.max():.3e}")
# smallest restricted facet of each mismatching cell (tolerance-level slivers?)
small = np.where((np.arange(32)[None, :] < r["fcount"][:, None]) & (r["farea"] > 0), r["farea"], np.inf).min(1) / sph
b = np.nonzero(bad)[0]
if len(b):
    print("  mismatching cells: smallest facet / sphere area: median %.2e max %.2e; vol rel median %.2e; >1e-6: %d" % (
        np.median(small[b]), small[b].max(), np.median(dv[b]), int((dv[b] > 1e-6).sum())))
    print("  all cells: fraction with a facet < 1e-4 of the sphere area: %.4f" % float((small < 1e-4).mean()))

# --- which side is right on the mismatching cells? --------------------------
# (1) two-sided consistency: a restricted facet is the same planar region seen
# from both cells (on the power bisector |x-p_i|^2-psi_i = |x-p_j|^2-psi_j),
# so |B_ij| must equal |B_ji|; compare each side's value with its twin.
if len(b):
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
            if ed < 0.5 * eo: dev_better += 1
            elif eo < 0.5 * ed: ora_better += 1
            else: ties += 1
    print(f"  facets differing: device closer to its twin {dev_better}, reference closer {ora_better}, undecided {ties}")
    # (2) Monte-Carlo volume of the cells that differ by > 1e-3
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
            q = np.concatenate([x, np.zeros((len(x), 1))], 1)
            _, nn = tree.query(q)  # power-nearest site = nearest lifted point
            vmc = (4 / 3) * np.pi * R ** 3 * np.mean(nn == i) * len(x) / N
            sd = (4 / 3) * np.pi * R ** 3 * np.sqrt(max(np.mean(nn == i) * (1 - np.mean(nn == i)), 1e-12) / N)
            zd, zo = abs(o["vol"][i] - vmc) / sd, abs(r["vol"][i] - vmc) / sd
            dev_ok += zd < 4; ora_ok += zo < 4
        print(f"  Monte-Carlo (2e5 samples) on {len(big)} cells differing > 1e-3: device within 4 sigma {dev_ok}, reference within 4 sigma {ora_ok}")
