"""Profiling driver (dev tool): a few evaluations of one scene, for ncu.

usage: python tools/prof_cells.py [c2|c4] [reps]
"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import geom, restricted, scenes

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dom = geom.box_domain([0, 0, 0], [1, 1, 1])
s = scenes.c2_dam_break() if which == "c2" else scenes.c4_droplet()
h = s.meta["h"]
tp = torch.as_tensor(s.pts, device="cuda")
tw = torch.full((s.n,), (0.85 * h) ** 2, dtype=torch.float64, device="cuda")
for _ in range(reps):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); r = restricted.evaluate(tp, tw, dom, smf=32); e1.record()
    torch.cuda.synchronize()
    print(which, s.n, "cells", f"{e0.elapsed_time(e1):.2f} ms", "flags", r.flags, flush=True)
