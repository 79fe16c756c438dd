#!/usr/bin/env python
"""Benchmark of the partial-OT hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Metric (BASELINE.json): "generalized Laguerre cells/sec (vol+areas) and ms per
Newton solve at 2M cells".  Workload at N=1: C4, the 2M-cell droplet scene
(paper teaser scale), at the weights psi of the config's
first (cold-start) Newton solve -- the committed fixture
tests/golden/psi_C4.npz (tools/make_psi_fixtures.py), read by BOTH arms so
they time bit-identical inputs.  The cold Newton solve itself is timed once
(median of three) as ``newton.ms_per_solve``.

One step = one full evaluation of the restricted Laguerre cells (bucket grid
counting sort + dpsi reduction + candidate gather + clip + restriction +
volumes / free-surface / facet areas / centroids), fp64, ball-aware, in
parity mode (the reference's restriction bit for bit; the
robust default's time is reported beside it), outputs in the reference's
fixed-stride layout (smf=32) resident in HBM.  L2 is flushed (a 256 MiB
write) before every timed step.  `e2e` repeats the step through the
reference-facing drop-in (`_kernels._batch_evaluate` on pageable numpy
arrays, allocated once like a caller's, -> pf_batch_evaluate_host): the
host->device copy of (pts, psi) and the device->host copy of everything the
reference writes are inside the timed region.

N>1 (torchrun): the domain is partitioned into x-slabs; rank r evaluates the
cells it owns using owned + ghost sites (ghost margin = largest ball-aware
search radius, with the global dpsi), so per-cell results are identical to
N=1 and there is no data-path collective during the evaluation.  Total work
is fixed (strong scaling).  `--impl reference` times the CPU port of the
reference kernel (oracle/, bit-identical to the numba reference) on the host
cores over ALL cells of the same workload each step (grid build included),
rank 0 only; it never loads the CUDA library.
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
    ap.add_argument("--mode", default="parity", choices=["parity", "robust"],
                    help="restriction of the timed evaluation (DESIGN.md §5.1)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_scene(name):
    from paper_2601_05765_b200 import scenes

    return scenes.make(name)


def workload_psi(name, sc):
    """(psi f64, description) of the workload: the committed converged weights."""
    fx = os.path.join(ROOT, "tests", "golden", f"psi_{name}.npz")
    if os.path.exists(fx):
        return (np.load(fx)["psi"].astype(np.float64),
                f"converged weights of the config's first cold-start Newton solve (eps_vol 1%), "
                f"fixture tests/golden/psi_{name}.npz (f32-rounded), identical in both arms")
    return None, None


def config_of(a, sc, psi_desc):
    """The workload description, identical in both arms."""
    return {"workload": workload_desc(a.config, sc), "ball_aware": True, "smf": a.smf, "psi": psi_desc,
            "restriction": "parity mode (the reference's restriction bit for bit)" if a.mode == "parity"
            else "robust (DESIGN.md 5.1)",
            "l2": "GPU arm: 256 MiB flush write before every timed step",
            "parallelism": f"x-slab spatial partition over {a.gpus} GPU(s), ghosts by search radius"
            if a.gpus > 1 else "1 GPU"}


# Speed of the CPU baseline (the C port) against the real numba reference on the
# same workload and threads, measured in the build container where the reference
# exists (tools/port_vs_numba.py -> profiles/port_vs_numba.json; C4, 8 threads:
# numba 59.0 s, port 29.0 s, all outputs bit-identical)
try:
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "port_vs_numba.json")) as _f:
        _pvn = json.load(_f)
    PORT_VS_NUMBA = {"factor": round(_pvn["port_vs_numba"], 3), "config": _pvn["config"], "threads": _pvn["threads"],
                     "numba_s": round(_pvn["numba_s"], 2), "port_s": round(_pvn["port_s"], 2),
                     "outputs_identical": _pvn["outputs_identical"],
                     "source": "profiles/port_vs_numba.json (tools/port_vs_numba.py, build container)"}
except (OSError, ValueError, KeyError):
    PORT_VS_NUMBA = None


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

    from paper_2601_05765_b200 import dist_solver, partition

    # exchange data plane: every rank starts from the sites of its own slab
    # (ghosts and the CG halo plan come from all-to-alls, halo.SlabComm)
    rank = dist.get_rank()
    cuts = partition.slab_cuts(sc.pts[:, 0], ws)
    gid = np.nonzero(partition.slab_owner(sc.pts[:, 0], ws, cuts=cuts) == rank)[0]
    dev = "cuda"
    solver = dist_solver.DistNewtonLocal(torch.as_tensor(gid, device=dev), torch.as_tensor(sc.pts[gid], device=dev),
                                         torch.as_tensor(sc.nu[gid], device=dev), dom, cuts)
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
              "partition": f"{ws} x-slabs (owned sites per rank, ghosts by all-to-all), halo "
                           f"{st['halo_entries']} entries/rank, {st['repartitions']} re-partitions"}
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
    # exact k-nearest sites of every site (k = 16, the _knn drop-in's kernel)
    knn = torch.empty((n, 16), dtype=torch.int64, device="cuda")
    L.pf_knn(c, n, _lib.ptr(pts), n, _lib.ptr(pts), 16, _lib.ptr(knn), 0, s)
    torch.cuda.synchronize()
    e0.record()
    L.pf_knn(c, n, _lib.ptr(pts), n, _lib.ptr(pts), 16, _lib.ptr(knn), 0, s)
    e1.record()
    torch.cuda.synchronize()
    t_knn = e0.elapsed_time(e1)
    gb_grid = 68.0 * n / (t_grid * 1e-3) / 1e9
    gb_cg = (12.0 * nnz + 108.0 * n) / (t_it * 1e-3) / 1e9
    gb_knn = 152.0 * n / (t_knn * 1e-3) / 1e9
    mk = lambda gbs, ms, by, note: {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s",  # noqa: E731
                                    "frac": gbs / peak if peak else None, "ms": ms, "algorithmic_bytes": by,
                                    "note": note}
    return {"grid_counting_sort": mk(gb_grid, t_grid, 68 * n, "68 B/site (SURVEY §8(d)); 6 small kernels + 1 host "
                                     "read of the bucket-size sum"),
            "pcg_iteration": mk(gb_cg, t_it, int(12 * nnz + 108 * n),
                                f"12 nnz + 108 n bytes, nnz={nnz}; one cooperative kernel on a SELL-32 copy of the "
                                f"Hessian (2 grid barriers per iteration), {it} iterations per call incl. the "
                                "SELL repack and the final host read"),
            "knn": mk(gb_knn, t_knn, 152 * n, "every site's 16 nearest sites: 24 B query + 128 B result per site "
                      "(candidate positions are L2-resident); warp per query, shell gather + rank sort"),
            "peak_source": "MEASURED_PEAKS.json hbm_gbs"}


def cpu_reference_run(sc, psi, steps, warmup, threads, cells=None):
    """CPU port of _kernels._batch_evaluate (oracle/, bit-identical to the
    numba reference) on the host cores: per step the reference's own
    SpatialGrid (numpy stable argsort, laguerre.py:52-80), _dpsi_max and the
    batch kernel over every cell (or the `cells` sample).  Outputs are
    allocated once, as a caller would."""
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre

    O.set_threads(threads)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    outs = O.alloc_outputs(sc.n, 32)
    m = sc.n if cells is None else len(cells)
    times, err = [], 0
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        g = O.SpatialGrid(sc.pts, [0, 0, 0], [1, 1, 1], dpk.volume)
        err = O.batch_evaluate(sc.pts, psi, *dpk.args(), *g.kernel_args(), dpk.tol, O.dpsi_max(psi), True, True,
                               32, *[outs[k] for k in O.OUT_ORDER], i0=0, i1=0 if cells is None else m,
                               cells=cells)
        t1 = time.perf_counter()
        if it >= warmup:
            times.append(t1 - t0)
    return m / (sum(times) / len(times)), O.num_threads(), err, times


def cpu_newton_run(cfg, threads):
    """CPU Newton restatement (oracle/newton_ref.py: SPEC.md:286-335 over the
    oracle) from the cold start: (ms, stats)."""
    from oracle import newton_ref
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre

    O.set_threads(threads)
    sc = make_scene(cfg)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    t0 = time.perf_counter()
    _, st = newton_ref.newton_solve(sc.pts, sc.nu, dpk.args(), dpk.tol, dom.diagonal())
    return 1e3 * (time.perf_counter() - t0), st


def main():
    a = parse()
    ws, rank, local = dist_env()
    if a.impl == "reference":
        if rank != 0:
            return
        sc = make_scene(a.config)
        psi, desc = workload_psi(a.config, sc)
        if psi is None:
            psi, desc = sc.psi_cold(), "cold start (no converged-weight fixture)"
        threads = os.cpu_count() or 1
        v, cores, err, times = cpu_reference_run(sc, psi, a.steps, a.warmup, threads)
        line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference", "config": config_of(a, sc, desc),
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                                 "sample": f"all {sc.n} cells of the workload every step, grid build + dpsi "
                                           "included (oracle/potflow_oracle.c: the reference kernel restated in "
                                           "C, bit-identical to the numba reference, tests/test_oracle_golden.py)",
                                 "port_vs_numba": PORT_VS_NUMBA},
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

    _lib.set_parity_mode(a.mode == "parity")
    psi_fix, psi_desc = workload_psi(a.config, sc)

    # ---- set-up (untimed): the config's first (cold-start) Newton solve, timed
    newton = None
    psi_g = None
    if a.no_newton:
        pass
    elif ws > 1:
        psi_g, newton = dist_newton(sc, dom, ws)
    else:
        with _lib.parity(False):  # the robust restriction (parity mode stalls on C4)
            psi_g, first_ms, nst = converged_psi(sc, dom)    # first solve of the process (allocations,
            again = [converged_psi(sc, dom)[1] for _ in range(3)]  # module loads); the same cold start x3
        newton_ms = statistics.median(again)
        newton = {"ms_per_solve": newton_ms, "ms_solves": again, "ms_first_solve_in_process": first_ms,
                  "iterations": nst["iterations"],
                  "evaluations": nst["evaluations"], "cg_iterations": nst["cg_iterations"],
                  "worst_initial": nst["worst_initial"], "worst_final": nst["worst_final"],
                  "status": nst["status_name"], "start": "cold (kappa (3 nu/4 pi)^(2/3))",
                  "restriction": "robust", "eps_vol": 0.01, "n": sc.n}
    if psi_fix is not None:
        psi_h = psi_fix
        if psi_g is not None and newton is not None:  # the fixture is this solve's result (f32-rounded)
            newton["fixture_max_rel_diff"] = float(np.max(np.abs(psi_g.cpu().numpy() - psi_fix) / psi_fix))
    elif psi_g is not None:
        psi_h, psi_desc = psi_g.cpu().numpy(), "converged weights of this run's cold-start Newton solve"
    else:
        psi_h, psi_desc = sc.psi_cold(), "cold start"
    psi_g = torch.as_tensor(psi_h, device="cuda")
    from paper_2601_05765_b200 import partition

    dpsi = partition.global_dpsi(psi_h) if ws > 1 else float(max(psi_h.max() - psi_h.min(), 0.0))

    if ws > 1:
        # exchange data plane: owned sites of this rank's slab, ghosts from the
        # other ranks' owned sites within this rank's search radius (all-to-all)
        from paper_2601_05765_b200 import dist_solver, halo

        cuts = partition.slab_cuts(sc.pts[:, 0], ws)
        gid = np.nonzero(partition.slab_owner(sc.pts[:, 0], ws, cuts=cuts) == rank)[0]
        sl = halo.SlabComm(cuts, dist_solver.Comm())
        loc = sl.ghosts(torch.as_tensor(gid, device="cuda"), {"pts": torch.as_tensor(sc.pts[gid], device="cuda")},
                        halo.ghost_margin(psi_h[gid], dpsi, 1.0))
        idx, owned = loc.gid.cpu().numpy(), loc.owned.cpu().numpy().astype(np.int32)
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
    # N=1: the device dpsi reduction runs inside every step (dpsi < 0); N>1: the
    # all-reduced global value (a slab's own max - min is not the reference's)
    dpsi_step = dpsi if ws > 1 else -1.0

    def step(cen=None):
        err = L.pf_batch_evaluate_ex(c, n_l, _lib.ptr(pts_l), _lib.ptr(psi_l), float(dpk.tol), dpsi_step, 1,
                                     1, smf, *[_lib.ptr(t) for t in outs],
                                     _lib.ptr(owned_t), 0 if owned_t is None else len(owned),
                                     None, _lib.ptr(cen), 1, _lib.stream_ptr())
        return _lib.check(err, "pf_batch_evaluate_ex")

    # census pass (untimed) -> algorithmic FP64 work of this workload
    step(census)
    torch.cuda.synchronize()
    cen = census[owned_t.long()] if owned_t is not None else census
    s_cell = float((cen.double().cpu().numpy() @ S_WEIGHTS).sum())  # DP slots, all owned cells
    cen_mean = cen.double().mean(0).cpu().numpy()
    mean_clips = float(cen_mean[0])
    s_build = float(cen_mean[:6] @ S_WEIGHTS[:6])
    s_eval = float(cen_mean[6:] @ S_WEIGHTS[6:])

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if os.environ.get("PF_NCU_STEP"):  # one extra untimed step inside a profiler range
        torch.cuda.profiler.start()    # (ncu --profile-from-start off captures just this step)
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()

    import ctypes

    def timed(nsteps, clk_on=True):
        fl, tot_ms, cells_ms, build_ms = 0, 0.0, 0.0, 0.0
        _lib.check(L.pf_stage_timing(c, 1), "pf_stage_timing")
        for _ in range(nsteps):
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
            ms = ctypes.c_double(0.0)
            if n_eval > 0:
                _lib.check(L.pf_last_cells_ms(c, ctypes.byref(ms)), "pf_last_cells_ms")
            cells_ms += ms.value
        b, e, ne = ctypes.c_double(0), ctypes.c_double(0), ctypes.c_int64(0)
        _lib.check(L.pf_stage_times(c, ctypes.byref(b), ctypes.byref(e), ctypes.byref(ne)), "pf_stage_times")
        _lib.check(L.pf_stage_timing(c, 0), "pf_stage_timing")
        nst = max(ne.value, 1)
        return fl, tot_ms / nsteps, cells_ms / nsteps, b.value / nst, e.value / nst

    # ---- timed region
    launches0 = L.pf_launch_count()
    with ClockSampler(dev) as clk:
        fl, t_step, t_cells, t_build, t_evalk = timed(a.steps)
    launches = int(L.pf_launch_count() - launches0)
    # the robust restriction's time on the same workload (same contract, not the headline)
    with _lib.parity(a.mode != "parity"):
        _, t_other, _, _, _ = timed(max(3, min(a.steps, 5)))
    if ws > 1:
        tt = all_reduce_host([t_step, t_cells, t_build, t_evalk, t_other], "max")
        t_step, t_cells, t_build, t_evalk, t_other = (float(x) for x in tt)
        s_cell_total = float(all_reduce_host([s_cell], "sum")[0])
    else:
        s_cell_total = s_cell
    value = sc.n / (t_step * 1e-3)

    # ---- end to end through the drop-in numpy API: pageable caller arrays
    # (N > 1: every rank calls the drop-in on its slab's host arrays -- owned
    # cells plus ghosts, the ghost results discarded -- max time over ranks)
    e2e = None
    if not a.no_e2e:
        gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
        order = ("status", "vol", "ksur", "cent", "ipt", "m2", "fcount", "ftag", "farea", "fh", "fnrm", "fcent")

        def host_outputs(pinned):
            shp = {"status": ((n_l,), np.int64), "vol": ((n_l,), np.float64), "ksur": ((n_l,), np.float64),
                   "cent": ((n_l, 3), np.float64), "ipt": ((n_l, 3), np.float64), "m2": ((n_l,), np.float64),
                   "fcount": ((n_l,), np.int64), "ftag": ((n_l, smf), np.int64), "farea": ((n_l, smf), np.float64),
                   "fh": ((n_l, smf), np.float64), "fnrm": ((n_l, smf, 3), np.float64),
                   "fcent": ((n_l, smf, 3), np.float64)}
            if not pinned:
                return {k: np.zeros(*shp[k]) for k in order}
            return {k: torch.zeros(shp[k][0], dtype=torch.from_numpy(np.zeros(1, shp[k][1])).dtype).pin_memory()
                    .numpy() for k in order}

        def run_e2e(pinned, nsteps):
            host = host_outputs(pinned)  # allocated once, like a caller's arrays
            pts_h = np.ascontiguousarray(sc.pts[idx])
            psi_hh = np.ascontiguousarray(psi_h[idx])
            if pinned:
                pts_h = torch.from_numpy(pts_h).pin_memory().numpy()
                psi_hh = torch.from_numpy(psi_hh).pin_memory().numpy()
            times = []
            for it in range(2 + nsteps):
                if ws > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _kernels._batch_evaluate(pts_h, psi_hh, *dpk.args(), *gargs, dpk.tol, dpsi_step, True, True, smf,
                                         *[host[k] for k in order])
                if it >= 2:
                    times.append(time.perf_counter() - t0)
            t = sum(times) / len(times)
            h2d, d2h = _kernels.last_copy_bytes
            if ws > 1:
                t = float(all_reduce_host([t], "max")[0])
                tot = all_reduce_host([h2d, d2h], "sum")
                h2d, d2h = float(tot[0]), float(tot[1])
            return t, int(h2d), int(d2h), host

        t_e2e, h2d, d2h, host = run_e2e(False, a.steps)
        e2e = {"value": sc.n / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * t_e2e,
               "api": "paper_2601_05765_b200._kernels._batch_evaluate on pageable numpy arrays (np.zeros outputs "
                      "allocated once) -> C ABI pf_batch_evaluate_host; copies counted by the library: (pts, psi) "
                      "in, per cell 96 B + per restricted facet 72 B out (everything the reference writes)"
                      + (f"; {ws} ranks, each on its slab (owned + ghost cells), max over ranks" if ws > 1 else "")}
        # the drop-in's host outputs equal the device-resident step's (same cells, same kernels)
        if ws == 1:
            step()  # the device-resident step in the same restriction mode
            torch.cuda.synchronize()
            fc_dev = outs[6].cpu().numpy()
            e2e["matches_device_step"] = bool(np.array_equal(host["fcount"], fc_dev)
                                              and np.array_equal(host["vol"], outs[1].cpu().numpy()))
        del host
        t_pin, _, _, _ = run_e2e(True, max(3, min(a.steps, 5)))
        e2e["pinned"] = {"value": sc.n / t_pin, "ms_per_step": 1e3 * t_pin,
                         "note": "same call with page-locked caller arrays"}

    # ---- FP64 roofline of the dominant kernels (k_cells_build + k_cells_eval_sync + tiers)
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
                "kernel": "k_cells_build+k_cells_eval_sync (+mid/exact tiers)",
                "kernel_ms": t_cells, "kernel_share_of_step": t_cells / t_step,
                "split": {"build_ms": t_build, "eval_ms": t_evalk,
                          "build_slots_per_cell": s_build, "eval_slots_per_cell": s_eval,
                          "build_frac": 2.0 * s_build * sc.n / (t_build * 1e-3) / 1e12 / peak_v if t_build > 0 else None,
                          "eval_frac": 2.0 * s_eval * sc.n / (t_evalk * 1e-3) / 1e12 / peak_v if t_evalk > 0 else None},
                "algorithmic": f"census S_cell (SURVEY.md §8(d)) = {s_cell_total / sc.n:.0f} DP slots/cell "
                               f"(build {s_build:.0f} + evaluation {s_eval:.0f}), x2 flop/slot; mean processed "
                               f"candidates {mean_clips:.1f}/cell",
                "census_per_cell": {k: round(float(v), 2) for k, v in zip(
                    ("clips", "vertex_tests", "new_vertices", "new_facet_vertices", "rfar_updates", "cuts",
                     "loop_entries", "sphere_crossings", "restricted_facets", "restricted_facets_x_nf",
                     "segment_pieces", "arc_pieces", "boundary_points", "projected_points", "full_circles",
                     "candidate_shells"), cen_mean)},
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
        v, cores, _, tt = cpu_reference_run(sc, psi_h, 1, 0, threads)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"all {sc.n} cells of the same workload, one pass ({tt[0]:.1f} s), grid build + dpsi "
                         "included; oracle/potflow_oracle.c is bit-identical to the numba reference",
               "port_vs_numba": PORT_VS_NUMBA}
        # Newton: the CPU restatement (SPEC.md:286-335 over the oracle) converges on C2
        # (the reference-faithful restriction stalls on C4); the device on C2 beside it
        try:
            ms_cpu, st = cpu_newton_run("C2", threads)
            sc2 = make_scene("C2")
            with _lib.parity(True):
                _, ms_dev, st2 = converged_psi(sc2, dom)
                ms_dev = statistics.median([converged_psi(sc2, dom)[1] for _ in range(3)])
            cpu["newton"] = {"config": "C2 97k dam break, cold start, eps_vol 1%", "cpu_ms": ms_cpu,
                             "cpu_iterations": st["iterations"], "cpu_evaluations": st["evaluations"],
                             "cpu_cg_iterations": st["cg_iterations"], "device_ms": ms_dev,
                             "device_iterations": st2["iterations"], "device_evaluations": st2["evaluations"],
                             "device_cg_iterations": st2["cg_iterations"],
                             "device_restriction": "parity mode", "cores": threads}
        except Exception as ex:  # report, never fail the bench line
            cpu["newton"] = {"error": repr(ex)[:200]}

    if rank == 0:
        cfg = config_of(a, sc, psi_desc)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": t_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": cfg, "flags": fl, "e2e": e2e, "gpu_launches": launches,
                "other_restriction_ms_per_step": {("robust" if a.mode == "parity" else "parity"): t_other},
                "roofline": roofline, "roofline_hbm_kernels": hbm, "cpu_baseline": cpu, "newton": newton,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
