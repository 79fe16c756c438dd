"""Newton convergence diagnostics at several scales (dev tool)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PF_NEWTON_VERBOSE"] = "1"
from paper_2601_05765_b200 import geom, restricted, scenes, solver
dom = geom.box_domain([0, 0, 0], [1, 1, 1])
for nt in [int(x) for x in sys.argv[1:]] or [150_000]:
    sc = scenes.c4_droplet(n_target=nt)
    t = time.time()
    res = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"), dom,
                              max_newton=12)
    torch.cuda.synchronize()
    print("n", sc.n, "time", time.time() - t, res.stats, flush=True)
    psi = res.psi
    print("psi nan", int(torch.isnan(psi).sum()), "psi<=0", int((psi <= 0).sum()), flush=True)
    d = restricted.evaluate(torch.as_tensor(sc.pts, device="cuda"), psi, dom)
    vol = d.vol.cpu().numpy()
    rel = np.abs(vol - sc.nu) / sc.nu
    w = np.argsort(-rel)[:8]
    print("flags", d.flags, "worst cells", rel[w], sc.pts[w].tolist(), d.status.cpu().numpy()[w], d.fcount.cpu().numpy()[w], flush=True)
