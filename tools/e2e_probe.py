"""Time the host-array drop-in with different chunk counts (dev tool)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import _kernels, geom, laguerre, scenes
from oracle import pyoracle as O

s = scenes.c4_droplet()
h = s.meta["h"]
psi = np.full(s.n, (0.85 * h) ** 2)
dom = geom.box_domain([0, 0, 0], [1, 1, 1]); dpk = laguerre.domain_pack(dom)
pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
host = {k: pin(v) for k, v in O.alloc_outputs(s.n, 32).items()}
print("pinned:", torch.from_numpy(host["ftag"]).is_pinned(), flush=True)
pts, w = pin(s.pts), pin(psi)
gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
dpsi = 0.0
for K in (8, 16, 32):
    os.environ["PF_E2E_CHUNKS"] = str(K)
    ts = []
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        _kernels._batch_evaluate(pts, w, *dpk.args(), *gargs, dpk.tol, dpsi, True, True, 32, *[host[k] for k in O.OUT_ORDER])
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(K, [f"{1e3*t:.1f}" for t in ts], flush=True)
