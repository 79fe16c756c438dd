"""First on-device parity + timing probe (dev tool)."""
import sys, time, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import geom, laguerre, restricted, scenes
from oracle import pyoracle as O

dom = geom.box_domain([0, 0, 0], [1, 1, 1])
dpk = laguerre.domain_pack(dom)
print(torch.cuda.get_device_name(0), flush=True)

def compare(name, pts, psi, ba=True, smf=32, oracle=True):
    pts = np.ascontiguousarray(pts); psi = np.ascontiguousarray(psi)
    n = len(pts)
    tp = torch.as_tensor(pts, device="cuda"); tw = torch.as_tensor(psi, device="cuda")
    torch.cuda.synchronize()
    t0 = time.time()
    r = restricted.evaluate(tp, tw, dom, ball_aware=ba, smf=smf)
    torch.cuda.synchronize()
    t1 = time.time()
    ts = []
    for it in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); restricted.evaluate(tp, tw, dom, ball_aware=ba, smf=smf); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    msg = f"{name}: n={n} gpu first {1e3*(t1-t0):.1f} ms, steady {min(ts):.2f} ms ({n/min(ts)*1e3/1e6:.2f} Mcells/s) flags={r.flags} retry={restricted.retry_count()}"
    if oracle:
        g = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
        t2 = time.time()
        o = O.evaluate(pts, psi, dpk.args(), dpk.tol, g, ball_aware=ba, smf=smf)
        t3 = time.time()
        msg += f" | oracle {1e3*(t3-t2):.0f} ms ({O.num_threads()} thr) err={o['err']}"
        G = {k: getattr(r, k if k not in ('farea','fh','fcent') else k).cpu().numpy() for k in ('status','vol','ksur','cent','ipt','m2','fcount','ftag','farea','fh','fnrm','fcent')}
        exact = {k: np.array_equal(G[k], o[k]) for k in ('status','fcount','ftag')}
        bitw = {k: np.array_equal(G[k], o[k]) for k in ('vol','ksur','cent','farea','fh','fnrm','fcent','ipt','m2')}
        def rel(a, b):
            d = np.abs(a - b); s = np.maximum(np.abs(b), 1e-300)
            return float(np.max(d / s)) if d.size else 0.0
        msg += f"\n   exact={exact}\n   bitwise={bitw}\n   vol rel {rel(G['vol'],o['vol']):.2e} ksur rel {rel(G['ksur'],o['ksur']):.2e} farea max abs/psi {np.max(np.abs(G['farea']-o['farea']))/psi.max():.2e} cent abs {np.max(np.abs(G['cent']-o['cent'])):.2e}"
        if not all(exact.values()):
            bad = np.nonzero((G['ftag'] != o['ftag']).any(1) | (G['status'] != o['status']))[0]
            msg += f"\n   mismatching cells: {len(bad)} e.g. {bad[:5]}"
            for i in bad[:3]:
                msg += f"\n    cell {i}: gpu st={G['status'][i]} fc={G['fcount'][i]} tags={G['ftag'][i,:G['fcount'][i]]} | ora st={o['status'][i]} fc={o['fcount'][i]} tags={o['ftag'][i,:o['fcount'][i]]}"
    print(msg, flush=True)

s = scenes.c1_random()
compare("C1 10k cold", s.pts, s.psi_cold())
compare("C1 10k cold full-mode", s.pts[:3000], s.psi_cold()[:3000] * 2, ba=False)
m = 20; h = 0.5 / m
rng = np.random.default_rng(7)
P = scenes._lattice((m, m, m), (0, 0, 0), h, rng)
compare("dense 8k", P, np.full(len(P), (0.85 * h) ** 2))
compare("dense 8k var", P, (0.8 * h + 0.1 * h * rng.random(len(P))) ** 2)
s2 = scenes.c2_dam_break()
h2 = s2.meta["h"]
compare("C2 97k psi=(0.85h)^2", s2.pts, np.full(s2.n, (0.85 * h2) ** 2))
s5 = scenes.c5_two_fluid(n_target=20000)
hA = s5.meta["h"]
compare("C5 20k twofluid", s5.pts, np.where(s5.nu > hA**3 * 1.5, (1.7 * hA) ** 2, (0.85 * hA) ** 2))
s1m = scenes.c1_random(n=1_000_000)
compare("C1 1M cold", s1m.pts, s1m.psi_cold(), oracle=True)
s4 = scenes.c4_droplet()
h4 = s4.meta["h"]
compare("C4 2M (0.85h)^2", s4.pts, np.full(s4.n, (0.85 * h4) ** 2), oracle=True)
