"""Command-line driver: `simulate` runs
the fluid scheme writing POTF frames and a CSV of per-step statistics (warm
start from a frame), `bench` prints the per-stage timings in the shape of the
paper's Table 1 (Laguerre / Evaluation / Solve / Complete
Step, mean over the steps), `render` writes a frame's fluid surface as PPM.

    python -m paper_2601_05765_b200.cli bench --sizes 10000,50000 --steps 20
    python -m paper_2601_05765_b200.cli simulate --config C2 --steps 100 --out runs/c2

Exit codes: 0 ok, 2 config error, 3 non-convergence (without
--best-effort).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np


def _stage_bind():
    from . import _lib

    L = _lib.lib()
    if not getattr(L, "_stage_bound", False):
        L.pf_stage_timing.argtypes = [C.c_void_p, C.c_int]
        L.pf_stage_times.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L._stage_bound = True
    return L


def timed_step(state, prm, dom):
    """One fluid step with per-stage device times (ms)."""
    import torch

    from . import _lib, fluid

    L = _stage_bind()
    c = _lib.ctx()
    L.pf_stage_timing(c, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d = fluid.step(state, prm, dom)
    e1.record()
    torch.cuda.synchronize()
    b, e, k = C.c_double(), C.c_double(), C.c_int64()
    _lib.check(L.pf_stage_times(c, C.byref(b), C.byref(e), C.byref(k)), "pf_stage_times")
    L.pf_stage_timing(c, 0)
    total = e0.elapsed_time(e1)
    return d, {"laguerre_ms": b.value, "evaluation_ms": e.value,
               "solve_ms": max(total - b.value - e.value, 0.0), "step_ms": total, "evaluations": k.value}


def cmd_bench(a) -> int:
    from . import fluid, geom, scenes

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    rows = []
    for size in [int(s) for s in a.sizes.split(",")]:
        sc = scenes.c2_dam_break(m=max(2, int(round(size ** (1.0 / 3.0)))))
        st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
        prm = fluid.SimParams(dt=1e-3, eps=5e-3)
        acc = []
        for _ in range(a.steps):
            _, t = timed_step(st, prm, dom)
            acc.append(t)
        mean = {k: float(np.mean([t[k] for t in acc])) for k in acc[0]}
        rows.append({"cells": sc.n, **mean})
    print(f"{'cells':>10} {'Laguerre':>10} {'Evaluation':>11} {'Solve':>9} {'Complete Step':>14}   (ms, mean of {a.steps} steps)")
    for r in rows:
        print(f"{r['cells']:>10} {r['laguerre_ms']:>10.3f} {r['evaluation_ms']:>11.3f} {r['solve_ms']:>9.3f} {r['step_ms']:>14.3f}")
    if a.json:
        print(json.dumps(rows))
    return 0


def cmd_simulate(a) -> int:
    from . import fluid, frames, geom, scenes

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    try:
        sc = scenes.make(a.config)
    except KeyError:
        print(f"unknown config {a.config}", file=sys.stderr)
        return 2
    if a.warm_start:
        st = frames.state_from_frame(frames.read_frame(a.warm_start), sc.nu, sc.rho)
    else:
        st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
    prm = fluid.SimParams(dt=sc.meta.get("dt", 1e-3), eps=sc.meta.get("eps", 5e-3), best_effort=a.best_effort)
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "stats.csv"), "w") as csv:
        csv.write("step,worst_rel_error,newton_iters,sum_vol,kinetic_energy,sum_ksur,wall_ms,flagged\n")
        for _ in range(a.steps):
            try:
                d, t = timed_step(st, prm, dom)
            except fluid.OtNonConvergence as ex:
                print(str(ex), file=sys.stderr)
                return 3
            f = frames.frame_from_state(st, d, t["step_ms"])
            m = sc.rho * sc.nu
            ke = 0.5 * float((m[:, None] * f.v ** 2).sum())
            csv.write(f"{f.step},{f.worst_rel_error},{f.newton_iters},{f.vol.sum()},{ke},{f.ksur.sum()},"
                      f"{t['step_ms']},{int(d['status_name'] != 'converged')}\n")
            if f.step % a.frame_stride == 0:
                frames.write_frame(os.path.join(a.out, f"frame_{f.step:06d}.potf"), f)
    return 0


def cmd_render(a) -> int:
    """Render a frame's fluid surface (Raw / Smooth / Depth) to a binary PPM and
    optionally sample its surface to a point cloud."""
    import time

    import torch

    from . import frames, render

    f = frames.read_frame(a.frame)
    cam = render.Camera(eye=tuple(a.eye), look_at=tuple(a.look_at), fov=a.fov, width=a.width, height=a.height)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kw = {"k": a.blend} if a.mode == "smooth" else {}
    img = render.render(f.x, f.psi, cam, a.mode, **kw)
    torch.cuda.synchronize()
    render.write_ppm(a.out, img)
    print(f"rendered {f.n} particles ({a.mode}), {a.width}x{a.height} in "
          f"{1e3 * (time.perf_counter() - t0):.1f} ms -> {a.out}")
    if a.samples > 0:
        x, nrm, _ = render.sample_surface(f.x, f.psi, a.samples)
        render.write_point_cloud(a.cloud, x, nrm)
        print(f"{a.samples} surface samples -> {a.cloud}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="potflow_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="per-stage timings, Table 1 shape")
    b.add_argument("--sizes", default="10000,50000")
    b.add_argument("--steps", type=int, default=20)
    b.add_argument("--json", action="store_true")
    s = sub.add_parser("simulate", help="run the fluid scheme, write frames + stats.csv")
    s.add_argument("--config", default="C2")
    s.add_argument("--steps", type=int, default=100)
    s.add_argument("--out", default="runs/sim")
    s.add_argument("--frame-stride", type=int, default=10)
    s.add_argument("--warm-start", default=None, help="POTF frame to resume from")
    s.add_argument("--best-effort", action="store_true")
    r = sub.add_parser("render", help="render a frame (raw | smooth | depth) to .ppm, optionally a surface point cloud")
    r.add_argument("frame")
    r.add_argument("--out", default="frame.ppm")
    r.add_argument("--eye", type=float, nargs=3, default=[0.5, -1.2, 0.9])
    r.add_argument("--look-at", type=float, nargs=3, default=[0.5, 0.5, 0.2])
    r.add_argument("--fov", type=float, default=0.8)
    r.add_argument("--width", type=int, default=1280)
    r.add_argument("--height", type=int, default=720)
    r.add_argument("--mode", default="raw", choices=["raw", "smooth", "depth"])
    r.add_argument("--blend", type=float, default=None, help="Smooth blend radius k (default 0.5 x mean radius)")
    r.add_argument("--samples", type=int, default=0, help="also write this many surface samples")
    r.add_argument("--cloud", default="surface.xyz", help="point cloud path for --samples")
    a = ap.parse_args(argv)
    return {"bench": cmd_bench, "simulate": cmd_simulate, "render": cmd_render}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
