"""Run the fluid scheme on a BASELINE config and report per-step Newton stats
and device time (dev tool).  usage: fluid_run.py C2|C3 [steps]"""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_05765_b200 import fluid, geom, scenes

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
sc = scenes.make(name)
dom = geom.box_domain([0, 0, 0], [1, 1, 1])
st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
prm = fluid.SimParams(dt=sc.meta.get("dt", 1e-3), eps=sc.meta.get("eps", 5e-3),
                      gravity=tuple(sc.meta.get("g", (0.0, 0.0, -9.81))))
torch.cuda.synchronize()
t0 = time.perf_counter()
hist = []
halted = None
for k in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    try:
        d = fluid.step(st, prm, dom)
    except fluid.OtNonConvergence as ex:
        halted = ex.diag
        break
    e1.record(); torch.cuda.synchronize()
    d["ms"] = e0.elapsed_time(e1)
    hist.append(d)
wall = time.perf_counter() - t0
ms = np.array([h["ms"] for h in hist])
print(json.dumps({"config": name, "n": sc.n, "steps": len(hist), "halted": halted, "wall_s": wall,
                  "ms_per_step_mean": float(ms.mean()), "ms_first": float(ms[0]),
                  "ms_per_step_after_first": float(ms[1:].mean()) if steps > 1 else None,
                  "all_converged": all(h["status_name"] == "converged" for h in hist),
                  "newton_iters_mean": float(np.mean([h["iterations"] for h in hist])),
                  "evaluations_total": int(sum(h["evaluations"] for h in hist)),
                  "damping_halvings_total": int(sum(h.get("damping_halvings", 0) for h in hist)),
                  "worst_final_max": float(max(h["worst_final"] for h in hist)),
                  "x_range": [float(st.x.min()), float(st.x.max())]}))
