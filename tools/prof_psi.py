"""Evaluations of a scene at its converged weights (dev tool; for ncu).  usage: prof_psi.py C3 [reps]"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import geom, restricted, scenes, solver
sc = scenes.make(sys.argv[1]); reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dom = geom.box_domain([0, 0, 0], [1, 1, 1])
pts = torch.as_tensor(sc.pts, device="cuda")
res = solver.newton_solve(pts, torch.as_tensor(sc.nu, device="cuda"), dom)
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); restricted.evaluate(pts, res.psi, dom); e1.record(); torch.cuda.synchronize()
    print(sys.argv[1], f"{e0.elapsed_time(e1):.2f} ms", "retries", restricted.retry_count(), flush=True)
