"""Partitioned Newton on the device (pf_dist.cu through dist_solver.CudaOps):
one rank against the single-device pf_newton_solve, and two ranks sharing
cuda:0 over gloo (halo exchange staged through the host) against the same."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _scene():
    import sys

    sys.path.insert(0, ROOT)
    from paper_2601_05765_b200 import scenes

    return scenes.c2_dam_break(m=16)


def _single():
    from paper_2601_05765_b200 import geom, solver

    sc = _scene()
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    res = solver.newton_solve(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(sc.nu, device="cuda"), dom)
    return sc, res.psi.cpu().numpy(), res.stats


def test_one_rank_matches_device_solver():
    from paper_2601_05765_b200 import dist_solver, geom

    sc, psi_ref, st = _single()
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    res = dist_solver.DistNewton(sc.pts, sc.nu, dom).solve()
    s = res.stats
    assert s["status"] == 0
    assert s["iterations"] == st["iterations"] and s["evaluations"] == st["evaluations"]
    assert abs(s["cg_iterations"] - st["cg_iterations"]) <= 2
    psi = np.empty(sc.n)
    psi[res.owned_global] = res.psi_owned
    assert np.max(np.abs(psi - psi_ref) / psi_ref) < 1e-6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2601_05765_b200 import dist_solver, geom

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sc = _scene()
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    res = dist_solver.DistNewton(sc.pts, sc.nu, dom, axis_lo=0.0, axis_hi=0.5, slack=1.2).solve()
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), psi=res.psi_owned, gid=res.owned_global,
             **{k: v for k, v in res.stats.items() if isinstance(v, (int, float))})
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_on_one_device_match_device_solver(tmp_path):
    sc, psi_ref, st = _single()
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    psi = np.full(sc.n, np.nan)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        psi[d["gid"]] = d["psi"]
        assert int(d["status"]) == 0
        assert int(d["iterations"]) == st["iterations"]
        assert int(d["evaluations"]) == st["evaluations"]
    assert np.isfinite(psi).all()
    assert np.max(np.abs(psi - psi_ref) / psi_ref) < 1e-6


def _eval_worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_2601_05765_b200 import _lib, geom, laguerre, partition, restricted, scenes

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sc = scenes.c2_dam_break(m=20)
    psi = np.full(sc.n, (0.85 * sc.meta["h"]) ** 2)
    dpsi = partition.global_dpsi(psi[rank::world])
    slab = partition.slab_partition(sc.pts, psi, dpsi, world, rank)
    l2g, own = slab.local_to_global, slab.owned_local
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    c = _lib.ctx()
    laguerre.upload_domain(c, *dpk.args(), dpk.tol)
    pts = torch.as_tensor(np.ascontiguousarray(sc.pts[l2g]), device="cuda")
    w = torch.as_tensor(np.ascontiguousarray(psi[l2g]), device="cuda")
    outs = restricted.alloc(len(l2g), 32)
    cells = torch.as_tensor(own, device="cuda")
    err = _lib.lib().pf_batch_evaluate_ex(c, len(l2g), _lib.ptr(pts), _lib.ptr(w), float(dpk.tol), dpsi, 1, 1, 32,
                                          *[_lib.ptr(t) for t in outs], _lib.ptr(cells), len(own), None, None, 1,
                                          _lib.stream_ptr())
    _lib.check(err, "pf_batch_evaluate_ex")
    o = {k: t.cpu().numpy()[own] for k, t in zip(("status", "vol", "ksur", "cent", "ipt", "m2", "fcount", "ftag",
                                                   "farea", "fh", "fnrm", "fcent"), outs)}
    o["ftag"] = partition.to_global(slab, o["ftag"], o["fcount"])
    np.savez(os.path.join(out_dir, f"e{rank}.npz"), gid=l2g[own], **o)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_device_evaluation_is_bitwise_single_device(tmp_path):
    """Spatial partition of the evaluation: per-cell results of 2
    ranks (owned + ghost sites, all-reduced dpsi) equal the 1-GPU ones bitwise."""
    from paper_2601_05765_b200 import geom, restricted, scenes

    mp.start_processes(_eval_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    sc = scenes.c2_dam_break(m=20)
    psi = np.full(sc.n, (0.85 * sc.meta["h"]) ** 2)
    d = restricted.evaluate(torch.as_tensor(sc.pts, device="cuda"), torch.as_tensor(psi, device="cuda"),
                            geom.box_domain([0, 0, 0], [1, 1, 1]))
    seen = np.zeros(sc.n, bool)
    for r in range(2):
        e = np.load(tmp_path / f"e{r}.npz")
        gid = e["gid"]
        assert not seen[gid].any()
        seen[gid] = True
        for k in ("status", "vol", "ksur", "cent", "fcount", "ftag", "farea", "fh", "fnrm"):
            assert np.array_equal(e[k], getattr(d, k).cpu().numpy()[gid]), k
    assert seen.all()
