"""Facet pairs whose areas differ from the two sides (dev tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O
from paper_2601_05765_b200 import geom, laguerre, restricted, scenes
sc = scenes.c4_droplet(); psi = np.full(sc.n, (0.85 * sc.meta["h"]) ** 2)
dom = geom.box_domain([0, 0, 0], [1, 1, 1]); dpk = laguerre.domain_pack(dom)
a = restricted.evaluate(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(psi, device="cuda"), dom)
n = sc.n
ft, fa, fc = a.ftag.cpu().numpy(), a.farea.cpu().numpy(), a.fcount.cpu().numpy()
used = (np.arange(32)[None, :] < fc[:, None]) & (ft >= 0)
I = np.nonzero(used)[0]; J = ft[used]; A = fa[used]
k1 = I * n + J; o1 = np.argsort(k1); k1s = k1[o1]; k2 = J * n + I
pos = np.minimum(np.searchsorted(k1s, k2), len(k1s) - 1); found = k1s[pos] == k2
sph = 4 * np.pi * psi.max()
dif = np.where(found, np.abs(A - A[o1[pos]]) / sph, 0)
bad = np.nonzero(dif > 1e-7)[0]
cells = np.unique(np.concatenate([I[bad], J[bad]])).astype(np.int64)
g = O.SpatialGrid(sc.pts, [0, 0, 0], [1, 1, 1], 1.0)
r = O.evaluate(sc.pts, psi, dpk.args(), dpk.tol, g, smf=32, i0=0, i1=len(cells), cells=cells)
def area(src_t, src_a, i, j):
    row = list(src_t[i]); return src_a[i][row.index(j)] if j in row else None
for b in bad:
    i, j = int(I[b]), int(J[b])
    print(f"pair {i}-{j}: device {area(ft, fa, i, j):.6e} / {area(ft, fa, j, i):.6e}   oracle {area(r['ftag'], r['farea'], i, j)} / {area(r['ftag'], r['farea'], j, i)}  vol dev {a.vol[i].item():.6e},{a.vol[j].item():.6e} ora {r['vol'][i]:.6e},{r['vol'][j]:.6e}")
