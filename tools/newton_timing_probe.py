import sys, time; sys.path.insert(0, "/root/repo")
import torch, bench
from paper_2601_05765_b200 import geom, scenes
sc = scenes.c4_droplet(); dom = geom.box_domain([0,0,0],[1,1,1])
for k in range(5):
    t = time.perf_counter(); _, ms, st = bench.converged_psi(sc, dom); print(k, round(ms,1), round(1e3*(time.perf_counter()-t),1), st["cg_iterations"], flush=True)
