"""Run one scene's evaluation a few times (for ncu captures)."""
import sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import geom, restricted, scenes
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dom = geom.box_domain([0, 0, 0], [1, 1, 1])
if name == "C2":
    s = scenes.c2_dam_break(); psi = np.full(s.n, (0.85 * s.meta["h"]) ** 2)
elif name == "C1":
    s = scenes.c1_random(); psi = s.psi_cold()
elif name == "C1M":
    s = scenes.c1_random(n=1_000_000); psi = s.psi_cold()
elif name == "C4":
    s = scenes.c4_droplet(); psi = np.full(s.n, (0.85 * s.meta["h"]) ** 2)
tp = torch.as_tensor(s.pts, device="cuda"); tw = torch.as_tensor(psi, device="cuda")
for r in range(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); d = restricted.evaluate(tp, tw, dom); e1.record(); torch.cuda.synchronize()
    print(name, s.n, "eval ms", e0.elapsed_time(e1), "retry", restricted.retry_count(), flush=True)
