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
