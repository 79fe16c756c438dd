"""Partitioned Newton solve over 2 gloo ranks on CPU: halo
exchange of the CG direction and of the Newton step, all-reduced dots and
statistics, re-partition when the weights outgrow the ghost layer.  Compared
with the single-rank CPU restatement (oracle/newton_ref.py) on the same
scene: same Newton iterations and evaluations, weights equal to the solver
tolerance.  The cell evaluator is the CPU oracle (tests/dist_numpy_ops.py);
the device path runs the same orchestration over pf_dist.cu."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    import sys

    sys.path.insert(0, ROOT)
    from paper_2601_05765_b200 import scenes

    return scenes.c2_dam_break(m=12)


def _worker(rank, world, port, out_dir, slack):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from dist_numpy_ops import NumpyOps
    from paper_2601_05765_b200 import dist_solver, geom, laguerre

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = _scene()
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    tau = 1e-12 * dom.diagonal() ** 2
    solver = dist_solver.DistNewton(
        sc.pts, sc.nu, dom, slack=slack, axis_lo=0.0, axis_hi=0.5,
        ops_factory=lambda p, n, r: NumpyOps(p, n, r, dpk.args(), dpk.tol, 32, tau))
    res = solver.solve()
    np.savez(os.path.join(out_dir, f"r{rank}_{slack}.npz"), psi=res.psi_owned, gid=res.owned_global,
             **{k: v for k, v in res.stats.items() if isinstance(v, (int, float))})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("slack", [1.0, 2.0])
def test_two_rank_newton_matches_single_rank(tmp_path, slack):
    from oracle import newton_ref
    from paper_2601_05765_b200 import geom, laguerre

    world, port = 2, _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path), slack), nprocs=world, join=True,
                       start_method="spawn")
    sc = _scene()
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    psi_ref, st = newton_ref.newton_solve(sc.pts, sc.nu, dpk.args(), dpk.tol, dom.diagonal())
    psi = np.full(sc.n, np.nan)
    stats = []
    for r in range(world):
        d = np.load(tmp_path / f"r{r}_{slack}.npz")
        psi[d["gid"]] = d["psi"]
        stats.append(d)
    assert np.isfinite(psi).all()
    for d in stats:
        assert int(d["status"]) == 0
        assert int(d["iterations"]) == st["iterations"]
        assert int(d["evaluations"]) == st["evaluations"]
        assert abs(int(d["cg_iterations"]) - st["cg_iterations"]) <= 2
    if slack == 1.0:
        assert int(stats[0]["repartitions"]) >= 1  # the weights outgrow a tight ghost layer
    assert np.max(np.abs(psi - psi_ref) / psi_ref) < 1e-6
