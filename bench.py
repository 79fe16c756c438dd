#!/usr/bin/env python
"""Benchmark of the partial-OT hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): "generalized Laguerre cells/sec (vol+areas) and ms per
Newton solve at 2M cells".  Workload at N=1: C4, the 2M-cell droplet scene
(paper teaser scale), weights psi at convergence of the
config's first (cold-start) Newton solve, which is computed in the untimed
set-up and itself timed once as ``newton.ms_per_solve``.

One step = one full evaluation of the restricted Laguerre cells (bucket grid
counting sort + dpsi reduction + candidate gather + clip + restriction +
volumes / free-surface / facet areas / centroids), fp64, ball-aware, outputs
in the reference's fixed-stride layout (smf=32) resident in HBM.  L2 is
flushed (a 256 MiB write) before every timed step.  `e2e` repeats the step
through the reference-facing drop-in (`_kernels._batch_evaluate` on host numpy
arrays): host->device copy of (pts, psi) and device->host copy of all twelve
outputs inside the timed region.

N>1 (torchrun): the domain is partitioned into x-slabs; rank r evaluates the
cells it owns using owned + ghost sites (ghost margin = largest ball-aware
search radius, with the global dpsi), so per-cell results are identical to
N=1 and there is no data-path collective during the evaluation.  Total work
is fixed (strong scaling).  `--impl reference` times the CPU oracle port of
the reference kernel (oracle/, bit-identical to the numba reference) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "generalized Laguerre cells/sec (vol+areas)"
UNIT = "cells/s"

# S_cell = sum of census terms x DP-pipe slots (census slot order)
S_WEIGHTS = np.array([29, 3, 16, 19, 6, 8, 6, 74, 70, 15, 160, 170, 60, 37, 20, 0], np.float64)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--smf", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-newton", action="store_true")
    ap.add_argument("--no-hbm", action="store_true")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_scene(name):
    from paper_2601_05765_b200 import scenes

    return scenes.make(name)


def workload_desc(name, sc):
    return {"C1": "C1 10k random seeds (30% fill), unit box",
            "C2": "C2 100k dam break (46^3 jittered lattice)",
            "C3": "C3 500k chocs (ball of radius 1/4)",
            "C4": "C4 2M-cell droplet (pool z<0.08 + drop r=0.12), paper teaser scale",
            "C5": "C5 1M two-fluid (spacing h / 2h)"}[name] + f", n={sc.n}"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"pf_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows]
        mx = float(rows[0][1])
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, nm in enumerate(names):
                if len(r) > 4 + k and "Active" in r[4 + k] and "Not" not in r[4 + k]:
                    reasons.add(nm)
        busy = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def converged_psi(sc, dom):
    import torch

    from paper_2601_05765_b200 import solver

    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"),
                              torch.as_tensor(sc.nu, device="cuda"), dom)
    e1.record()
    torch.cuda.synchronize()
    return res.psi, float(e0.elapsed_time(e1)), res.stats


def all_reduce_host(vals, op="sum"):
    """All-reduce of a few host scalars (through the device for NCCL)."""
    import torch
    import torch.distributed as dist

    gloo = dist.get_backend() == "gloo"
    t = torch.tensor(vals, dtype=torch.float64, device="cpu" if gloo else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return t.cpu()


def dist_newton(sc, dom, ws):
    """Partitioned Newton solve over the ranks (x-slabs, halo exchange per CG
    iteration, all-reduced dots); device time, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2601_05765_b200 import dist_solver

    solver = dist_solver.DistNewton(sc.pts, sc.nu, dom)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = solver.solve()
    e1.record()
    torch.cuda.synchronize()
    ms = all_reduce_host([e0.elapsed_time(e1)], "max")
    parts = [None] * ws
    dist.all_gather_object(parts, (res.owned_global, res.psi_owned))
    psi = np.zeros(sc.n)
    for g, v in parts:
        psi[g] = v
    st = res.stats
    newton = {"ms_per_solve": float(ms[0]), "iterations": st["iterations"], "evaluations": st["evaluations"],
              "cg_iterations": st["cg_iterations"], "worst_initial": st["worst_initial"],
              "worst_final": st["worst_final"], "status": st["status_name"],
              "start": "cold (kappa (3 nu/4 pi)^(2/3))", "eps_vol": 0.01, "n": sc.n,
              "partition": f"{ws} x-slabs, halo {st['halo_entries']} entries/rank, "
                           f"{st['repartitions']} re-partitions"}
    return torch.as_tensor(psi, device="cuda"), newton


def hbm_kernels(sc, dom, psi_g, smf, reps=5, cg_iters=50):
    """Achieved HBM bandwidth of the two memory-bound kernels on this workload
    (SURVEY §8(d) algorithmic bytes): the grid counting sort (68 B/site) and a
    Jacobi-PCG iteration on the Newton Hessian of the converged weights
    (12 nnz + 108 n bytes).  CUDA events on the launching stream."""
    import ctypes

    import torch

    from paper_2601_05765_b200 import _lib, solver

    L = _lib.lib()
    c = _lib.ctx()
    n = sc.n
    pts = torch.as_tensor(sc.pts, device="cuda")
    s = _lib.stream_ptr()
    peak = None
    pp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pp):
        peak = json.load(open(pp)).get("hbm_gbs")
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    # grid counting sort (bucket size from the weights, as every evaluation does)
    _lib.check(L.pf_grid_build(c, n, _lib.ptr(pts), _lib.ptr(psi_g), 0.0, s), "pf_grid_build")
    e0, e1 = ev(), ev()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        _lib.check(L.pf_grid_build(c, n, _lib.ptr(pts), _lib.ptr(psi_g), 0.0, s), "pf_grid_build")
    e1.record()
    torch.cuda.synchronize()
    t_grid = e0.elapsed_time(e1) / reps
    # PCG iterations on the final Hessian of the last Newton solve
    solver._bind()
    _, ksur, fcount, ftag, farea = solver.last_state(n, smf)
    f8, i4 = dict(dtype=torch.float64, device="cuda"), dict(dtype=torch.int32, device="cuda")
    hcnt, hcol = torch.empty(n, **i4), torch.empty((n, smf), **i4)
    hval, diag = torch.empty((n, smf), **f8), torch.empty(n, **f8)
    tau = 1e-12 * dom.diagonal() ** 2
    _lib.check(L.pf_newton_hessian(n, smf, _lib.ptr(pts), _lib.ptr(psi_g), _lib.ptr(fcount), _lib.ptr(ftag),
                                   _lib.ptr(farea), _lib.ptr(ksur), float(tau), _lib.ptr(hcnt), _lib.ptr(hcol),
                                   _lib.ptr(hval), _lib.ptr(diag), s), "pf_newton_hessian")
    b = torch.rand(n, generator=torch.Generator(device="cuda").manual_seed(1), **f8)
    x = torch.empty(n, **f8)
    L.pf_pcg(n, smf, _lib.ptr(hcnt), _lib.ptr(hcol), _lib.ptr(hval), _lib.ptr(diag), _lib.ptr(b), _lib.ptr(x),
             0.0, 8, s)
    torch.cuda.synchronize()
    e0.record()
    it = L.pf_pcg(n, smf, _lib.ptr(hcnt), _lib.ptr(hcol), _lib.ptr(hval), _lib.ptr(diag), _lib.ptr(b),
                  _lib.ptr(x), 0.0, cg_iters, s)
    e1.record()
    torch.cuda.synchronize()
    t_it = e0.elapsed_time(e1) / max(it, 1)
    nnz = int(hcnt.sum())
    gb_grid = 68.0 * n / (t_grid * 1e-3) / 1e9
    gb_cg = (12.0 * nnz + 108.0 * n) / (t_it * 1e-3) / 1e9
    mk = lambda gbs, ms, by, note: {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",  # noqa: E731
                                    "frac": gbs / peak if peak else None, "ms": ms, "algorithmic_bytes": by,
                                    "note": note}
    return {"grid_counting_sort": mk(gb_grid, t_grid, 68 * n, "68 B/site (SURVEY §8(d)); 6 small kernels + 1 host "
                                     "read of the bucket-size sum"),
            "pcg_iteration": mk(gb_cg, t_it, int(12 * nnz + 108 * n),
                                f"12 nnz + 108 n bytes, nnz={nnz}; 5 kernels per iteration (SpMV 8 lanes/row, "
                                "2 single-block reductions, 2 vector updates), host check every 8"),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs"}


def cpu_reference_run(sc, psi, steps, warmup, sample_cells, threads):
    """CPU oracle port of _kernels._batch_evaluate on the host cores."""
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre

    O.set_threads(threads)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    rng = np.random.default_rng(0)
    cells = np.sort(rng.choice(sc.n, size=min(sample_cells, sc.n), replace=False)).astype(np.int64)
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        g = O.SpatialGrid(sc.pts, [0, 0, 0], [1, 1, 1], dpk.volume)
        o = O.evaluate(sc.pts, psi, dpk.args(), dpk.tol, g, ball_aware=True, want_m2=True, smf=32,
                       i0=0, i1=len(cells), cells=cells)
        t1 = time.perf_counter()
        if it >= warmup:
            times.append(t1 - t0)
    return len(cells) / (sum(times) / len(times)), O.num_threads(), o["err"]


def main():
    a = parse()
    ws, rank, local = dist_env()
    if a.impl == "reference":
        if rank != 0:
            return
        sc = make_scene(a.config)
        # converged weights need the device solve; the CPU arm uses the same
        # weights when a GPU is present, else the cold-start weights
        psi = sc.psi_cold()
        try:
            import torch

            if torch.cuda.is_available():
                from paper_2601_05765_b200 import geom

                psi = converged_psi(sc, geom.box_domain([0, 0, 0], [1, 1, 1]))[0].cpu().numpy()
        except Exception:
            pass
        threads = os.cpu_count() or 1
        sample = 400_000 if sc.n > 400_000 else sc.n
        v, cores, err = cpu_reference_run(sc, psi, a.steps, a.warmup, sample, threads)
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": 1e3 * sample / v, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference",
                "config": {"workload": workload_desc(a.config, sc), "ball_aware": True, "smf": 32},
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                 "sample": f"{sample} random cells of the workload per step "
                                           "(full neighbourhoods), grid build included"},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
                "flags": err}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    from paper_2601_05765_b200 import _kernels, _lib, geom, laguerre, restricted

    if ws > 1:
        # PF_DIST_BACKEND=gloo runs several ranks on one device (testing only)
        backend = os.environ.get("PF_DIST_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.cuda.current_device()
    sc = make_scene(a.config)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    L = _lib.lib()
    c = _lib.ctx()
    laguerre.upload_domain(c, *dpk.args(), dpk.tol)

    # ---- set-up (untimed): converged weights from the config's first solve
    newton = None
    if a.no_newton:
        psi_g = torch.as_tensor(sc.psi_cold(), device="cuda")
    elif ws > 1:
        psi_g, newton = dist_newton(sc, dom, ws)
    else:
        psi_g, first_ms, nst = converged_psi(sc, dom)    # first solve of the process (allocations,
        again = [converged_psi(sc, dom)[1] for _ in range(3)]  # module loads); the same cold start x3
        newton_ms = statistics.median(again)
        newton = {"ms_per_solve": newton_ms, "ms_solves": again, "ms_first_solve_in_process": first_ms,
                  "iterations": nst["iterations"],
                  "evaluations": nst["evaluations"], "cg_iterations": nst["cg_iterations"],
                  "worst_initial": nst["worst_initial"], "worst_final": nst["worst_final"],
                  "status": nst["status_name"], "start": "cold (kappa (3 nu/4 pi)^(2/3))",
                  "eps_vol": 0.01, "n": sc.n}
    psi_h = psi_g.cpu().numpy()
    from paper_2601_05765_b200 import partition

    dpsi = partition.global_dpsi(psi_h) if ws > 1 else float(max(psi_h.max() - psi_h.min(), 0.0))

    if ws > 1:
        slab = partition.slab_partition(sc.pts, psi_h, dpsi, ws, rank)
        idx, owned = slab.local_to_global, slab.owned_local
    else:
        idx, owned = np.arange(sc.n), None
    pts_l = torch.as_tensor(np.ascontiguousarray(sc.pts[idx]), device="cuda")
    psi_l = torch.as_tensor(np.ascontiguousarray(psi_h[idx]), device="cuda")
    owned_t = None if owned is None else torch.as_tensor(owned, device="cuda")
    n_l = len(idx)
    n_eval = n_l if owned is None else len(owned)
    smf = a.smf
    outs = restricted.alloc(n_l, smf)
    census = torch.zeros((n_l, 16), dtype=torch.int32, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step(cen=None):
        err = L.pf_batch_evaluate_ex(c, n_l, _lib.ptr(pts_l), _lib.ptr(psi_l), float(dpk.tol), dpsi, 1,
                                     1, smf, *[_lib.ptr(t) for t in outs],
                                     _lib.ptr(owned_t), 0 if owned_t is None else len(owned),
                                     None, _lib.ptr(cen), 1, _lib.stream_ptr())
        return _lib.check(err, "pf_batch_evaluate_ex")

    # census pass (untimed) -> algorithmic FP64 work of this workload
    step(census)
    torch.cuda.synchronize()
    cen = census[owned_t.long()] if owned_t is not None else census
    s_cell = float((cen.double().cpu().numpy() @ S_WEIGHTS).sum())  # DP slots, all owned cells
    mean_clips = float(cen[:, 0].double().mean())

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if os.environ.get("PF_NCU_STEP"):  # one extra untimed step inside a profiler range
        torch.cuda.profiler.start()    # (ncu --profile-from-start off captures just this step)
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()

    # ---- timed region
    fl = 0
    tot_ms = 0.0
    cells_ms = 0.0
    launches0 = L.pf_launch_count()
    with ClockSampler(dev) as clk:
        for _ in range(a.steps):
            flush.fill_(1.0)
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fl |= step()
            e1.record()
            torch.cuda.synchronize()
            tot_ms += e0.elapsed_time(e1)
            import ctypes

            ms = ctypes.c_double(0.0)
            if n_eval > 0:
                _lib.check(L.pf_last_cells_ms(c, ctypes.byref(ms)), "pf_last_cells_ms")
            cells_ms += ms.value
    launches = int(L.pf_launch_count() - launches0)
    t_step = tot_ms / a.steps
    t_cells = cells_ms / a.steps
    if ws > 1:
        tt = all_reduce_host([t_step, t_cells], "max")
        t_step, t_cells = float(tt[0]), float(tt[1])
        s_cell_total = float(all_reduce_host([s_cell], "sum")[0])
    else:
        s_cell_total = s_cell
    value = sc.n / (t_step * 1e-3)

    # ---- end to end through the drop-in numpy API (N=1)
    # (N > 1: every rank calls the drop-in on its slab's host arrays -- owned
    # cells plus ghosts, the ghost results discarded -- max time over ranks)
    e2e = None
    if not a.no_e2e:
        from oracle import pyoracle as O  # only for the output allocator shapes

        host = O.alloc_outputs(n_l, smf)
        pin = lambda x: torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()  # noqa: E731
        pts_p, psi_p = pin(sc.pts[idx]), pin(psi_h[idx])
        host = {k: pin(v) for k, v in host.items()}
        gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
        times = []
        for it in range(2 + a.steps):
            if ws > 1:
                dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _kernels._batch_evaluate(pts_p, psi_p, *dpk.args(), *gargs, dpk.tol, dpsi, True, True, smf,
                                     *[host[k] for k in O.OUT_ORDER])
            torch.cuda.synchronize()
            if it >= 2:
                times.append(time.perf_counter() - t0)
        t_e2e = sum(times) / len(times)
        h2d = pts_p.nbytes + psi_p.nbytes
        d2h = sum(host[k].nbytes for k in O.OUT_ORDER)
        if ws > 1:
            t_e2e = float(all_reduce_host([t_e2e], "max")[0])
            tot = all_reduce_host([h2d, d2h], "sum")
            h2d, d2h = float(tot[0]), float(tot[1])
        e2e = {"value": sc.n / t_e2e, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * t_e2e,
               "api": "paper_2601_05765_b200._kernels._batch_evaluate (numpy, pinned host buffers)"
                      + (f"; {ws} ranks, each on its slab (owned + ghost cells), max over ranks" if ws > 1 else "")}

    # ---- FP64 roofline of the dominant kernel (k_cells_fast + exact tier)
    import ctypes

    peak = ctypes.c_double(0.0)
    _lib.check(L.pf_fp64_peak(ctypes.byref(peak), None), "pf_fp64_peak")
    peak_v = peak.value
    if ws > 1:  # achieved is whole-job (all ranks' cells / max time): compare with the job's peak
        peak_v = float(all_reduce_host([peak_v], "sum")[0])
    achieved = 2.0 * s_cell_total / (t_cells * 1e-3) / 1e12  # slot = FMA-equivalent (2 flop)
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tr = json.load(open(tp)).get(a.config)
            if tr:
                traffic = float(tr["k_cells_build_dram_bytes"] + tr["k_cells_eval_sync_dram_bytes"])
                traffic_src = tr
        except Exception:
            traffic = None
    roofline = {"bound": "fp64", "achieved": achieved, "peak": peak_v, "unit": "TFLOP/s",
                "frac": achieved / peak_v if peak_v > 0 else None, "traffic": traffic,
                "traffic_unit": "bytes per step (DRAM read+write of the cell kernels, ncu)",
                "traffic_detail": traffic_src,
                "kernel": "k_cells_build+k_cells_eval (+k_cells_exact retries)",
                "kernel_ms": t_cells, "kernel_share_of_step": t_cells / t_step,
                "algorithmic": f"census S_cell (SURVEY.md §8(d)) = {s_cell_total / sc.n:.0f} DP slots/cell,"
                               f" x2 flop/slot; mean processed candidates {mean_clips:.1f}/cell",
                "peak_source": "measured in-run by pf_fp64_peak (DFMA chains; MEASURED_PEAKS.json has no FP64 entry)"
                               + (f", summed over the {ws} ranks' GPUs" if ws > 1 else "")}

    # ---- HBM-bound kernels of the path (N=1, converged weights)
    hbm = None
    if ws == 1 and newton is not None and not a.no_hbm:
        hbm = hbm_kernels(sc, dom, psi_g, smf)

    # ---- CPU baseline: oracle port on the host cores (rank 0, N=1)
    cpu = None
    if not a.no_cpu and ws == 1 and rank == 0:
        threads = os.cpu_count() or 1
        sample = 200_000 if sc.n > 200_000 else sc.n
        v, cores, _ = cpu_reference_run(sc, psi_h, 1, 0, sample, threads)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{sample} random cells of the same workload (full neighbourhoods), one pass, "
                         "grid build included; oracle/potflow_oracle.c is bit-identical to the numba reference"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": t_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_desc(a.config, sc), "ball_aware": True, "smf": smf,
                           "psi": "converged (first cold-start Newton solve, eps_vol=1%)"
                           if newton else "cold start",
                           "l2": "256 MiB flush write before every timed step",
                           "parallelism": f"x-slab spatial partition over {ws} GPU(s), ghosts by search radius"
                           if ws > 1 else "1 GPU"},
                "flags": fl, "e2e": e2e, "gpu_launches": launches,
                "roofline": roofline, "roofline_hbm_kernels": hbm, "cpu_baseline": cpu, "newton": newton,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
