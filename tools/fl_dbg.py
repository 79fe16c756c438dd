import os, sys, time, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2601_05765_b200 import fluid, geom, scenes
sc = scenes.make(sys.argv[1])
dom = geom.box_domain([0, 0, 0], [1, 1, 1])
st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
prm = fluid.SimParams(dt=sc.meta.get("dt", 1e-3), eps=sc.meta.get("eps", 5e-3), max_newton=int(sys.argv[3]))
for k in range(int(sys.argv[2])):
    t0 = time.time(); d = fluid.step(st, prm, dom); torch.cuda.synchronize()
    print(k, f"{time.time()-t0:.2f}s", d, flush=True)
