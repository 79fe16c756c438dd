"""Mean census counters (CEN_*) of one evaluation (dev tool)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import _lib, geom, laguerre, restricted, scenes
which = sys.argv[1] if len(sys.argv) > 1 else "c2"
s = scenes.c2_dam_break() if which == "c2" else scenes.c4_droplet()
h = s.meta["h"]
dom = geom.box_domain([0, 0, 0], [1, 1, 1]); dpk = laguerre.domain_pack(dom)
c = _lib.ctx(); laguerre.upload_domain(c, *dpk.args(), dpk.tol)
n = s.n
pts = torch.as_tensor(s.pts, device="cuda"); psi = torch.full((n,), (0.85 * h) ** 2, dtype=torch.float64, device="cuda")
outs = restricted.alloc(n, 32)
cen = torch.zeros((n, 16), dtype=torch.int32, device="cuda")
L = _lib.lib()
err = L.pf_batch_evaluate_ex(c, n, _lib.ptr(pts), _lib.ptr(psi), float(dpk.tol), -1.0, 1, 1, 32, *[_lib.ptr(t) for t in outs], None, 0, None, _lib.ptr(cen), 1, _lib.stream_ptr())
torch.cuda.synchronize()
names = ["clips", "tests", "newv", "nfv", "rfar", "cuts", "loop", "cross", "rfac", "rfac_nf", "seg", "arc", "bpts", "proj", "fullc"]
m = cen.double().mean(0).cpu().numpy()
print(which, {k: round(float(v), 2) for k, v in zip(names, m)})
cl = cen[:, 0].double(); cu = cen[:, 5].double()
print("untouched-ish clips per cell", float((cl - cu).mean()))
