"""Wall-clock breakdown of fluid steps at one size (dev tool).  usage: step_probe.py N [steps]"""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import fluid, geom, scenes, solver

n = int(sys.argv[1]); steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sc = scenes.c2_dam_break(m=max(2, int(round(n ** (1.0 / 3.0)))))
dom = geom.box_domain([0, 0, 0], [1, 1, 1])
st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
prm = fluid.SimParams(dt=1e-3, eps=5e-3)
orig = solver.newton_solve
acc = {}
def timed(name, f):
    def w(*a, **k):
        torch.cuda.synchronize(); t = time.perf_counter(); r = f(*a, **k); torch.cuda.synchronize()
        acc[name] = acc.get(name, 0.0) + 1e3 * (time.perf_counter() - t); return r
    return w
solver.newton_solve = timed("newton_solve", orig)
for k in range(steps):
    torch.cuda.synchronize(); t = time.perf_counter()
    d = fluid.step(st, prm, dom)
    torch.cuda.synchronize(); dt = 1e3 * (time.perf_counter() - t)
    print(f"step {k}: {dt:.1f} ms, newton {acc.get('newton_solve', 0):.1f} ms, evaluations {d['evaluations']}, "
          f"iterations {d['iterations']}, cg {d['cg_iterations']}", flush=True)
    acc.clear()
