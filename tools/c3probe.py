import sys; sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_05765_b200 import geom, solver, scenes, restricted
sc = scenes.c3_chocs(); dom = geom.box_domain([0,0,0],[1,1,1])
res = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"), dom)
psi = res.psi.cpu().numpy(); r0 = (3*sc.nu[0]/(4*np.pi))**(1/3)
print("r0", r0, "sqrt psi min/median/max", np.sqrt(psi.min()), np.sqrt(np.median(psi)), np.sqrt(psi.max()), "dpsi/r0^2", (psi.max()-psi.min())/r0**2)
print("br global / r0:", (np.sqrt(np.median(psi)) + np.sqrt(np.median(psi) + psi.max()-psi.min()))/r0)
import time
for i in range(2):
    torch.cuda.synchronize(); t=time.time(); d = restricted.evaluate(res.psi, res.psi, dom) if False else restricted.evaluate(torch.as_tensor(sc.pts, device="cuda"), res.psi, dom); torch.cuda.synchronize(); print("eval ms", 1e3*(time.time()-t), "retries", restricted.retry_count())
cen = restricted.census(sc.n).cpu().numpy(); print("processed candidates mean/p99/max", cen.mean(), np.percentile(cen, 99), cen.max())
print("psi quantiles (sqrt/r0):", np.quantile(np.sqrt(psi)/r0, [0.5, 0.9, 0.99, 0.999, 1.0]))
