"""Mean census counters (CEN_*) of one evaluation (dev tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import _lib, geom, laguerre, restricted, scenes
which = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = scenes.make(which.upper())
dom = geom.box_domain([0, 0, 0], [1, 1, 1]); dpk = laguerre.domain_pack(dom)
c = _lib.ctx(); laguerre.upload_domain(c, *dpk.args(), dpk.tol)
n = s.n
pts = torch.as_tensor(s.pts, device="cuda")
if which in ("c2", "c4"):
    psi = torch.full((n,), (0.85 * s.meta["h"]) ** 2, dtype=torch.float64, device="cuda")
else:  # converged weights
    from paper_2601_05765_b200 import solver
    psi = solver.newton_solve(pts, torch.as_tensor(s.nu, device="cuda"), dom).psi
outs = restricted.alloc(n, 32)
cen = torch.zeros((n, 16), dtype=torch.int32, device="cuda")
L = _lib.lib()
err = L.pf_batch_evaluate_ex(c, n, _lib.ptr(pts), _lib.ptr(psi), float(dpk.tol), -1.0, 1, 1, 32, *[_lib.ptr(t) for t in outs], None, 0, None, _lib.ptr(cen), 1, _lib.stream_ptr())
torch.cuda.synchronize()
names = ["clips", "tests", "newv", "nfv", "rfar", "cuts", "loop", "cross", "rfac", "rfac_nf", "seg", "arc", "bpts", "proj", "fullc", "gathers"]
m = cen.double().mean(0).cpu().numpy()
print(which, {k: round(float(v), 2) for k, v in zip(names, m)})
cl = cen[:, 0].double(); cu = cen[:, 5].double()
print("untouched-ish clips per cell", float((cl - cu).mean()))
for k, nm in ((0, "clips"), (5, "cuts"), (15, "gathers")):
    v = cen[:, k].double().cpu().numpy()
    print(nm, "p50/p90/p99/max", np.percentile(v, [50, 90, 99]).round(1), v.max())
