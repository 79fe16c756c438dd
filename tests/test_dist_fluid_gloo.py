"""Distributed fluid steps on the exchange data plane (paper_2601_05765_b200/
dist_fluid.py) over 2 gloo ranks on CPU against the same steps on one rank:
advection, migration across the slab cut (particles are given an x velocity
so that they cross it), Newton with ghosts exchanged from owned particles
only, spring + gravity.  Cells by the CPU oracle, per-particle updates by a
numpy restatement of the kernels (tests/dist_numpy_ops.py)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import ROOT

STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, out):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch

    from dist_numpy_ops import NumpyOps, NumpyParticleOps
    from paper_2601_05765_b200 import dist_fluid, fluid, geom, laguerre, partition, scenes

    sc = scenes.c2_dam_break(m=10)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    tau = 1e-12 * dom.diagonal() ** 2
    fac = lambda p, n, r: NumpyOps(p, n, r, dpk.args(), dpk.tol, 32, tau)  # noqa: E731
    v = np.zeros_like(sc.pts)
    v[:, 0] = 5.0  # the block moves right: the column next to x = 0.25 crosses the cut
    rho = np.full(sc.n, 1000.0)
    cuts = np.array([0.25]) if world == 2 else np.zeros(0)
    gid = np.nonzero(partition.slab_owner(sc.pts[:, 0], world, cuts=cuts) == rank)[0]
    params = fluid.SimParams(dt=2e-3, eps=5e-3)
    df = dist_fluid.DistFluid(torch.as_tensor(gid), sc.pts[gid], v[gid], sc.nu[gid], rho[gid], dom, cuts,
                              params, ops_factory=fac, particle_ops=NumpyParticleOps(), slack=1.5)
    moved = 0
    for _ in range(STEPS):
        before = set(df.gid.tolist())
        df.step()
        moved += len(set(df.gid.tolist()) - before)
    np.savez(out, gid=df.gid.numpy(), x=df.x.numpy(), v=df.v.numpy(), psi=df.psi.numpy(), moved=moved,
             it=[h["iterations"] for h in df.history], ev=[h["evaluations"] for h in df.history])


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _run(rank, world, os.path.join(out_dir, f"r{rank}.npz"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_fluid_steps_match_one_rank(tmp_path):
    import sys

    sys.path.insert(0, ROOT)
    _run(0, 1, str(tmp_path / "single.npz"))
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    s = np.load(tmp_path / "single.npz")
    n = len(s["gid"])
    x, v, psi = np.full((n, 3), np.nan), np.full((n, 3), np.nan), np.full(n, np.nan)
    moved = 0
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        x[d["gid"]], v[d["gid"]], psi[d["gid"]] = d["x"], d["v"], d["psi"]
        moved += int(d["moved"])
        assert list(d["it"]) == list(s["it"]) and list(d["ev"]) == list(s["ev"])
    assert moved > 0, "no particle crossed the slab cut"
    assert np.isfinite(x).all()
    # the two runs differ only by the CG dot-product summation order
    assert np.max(np.abs(x - s["x"])) < 1e-9
    assert np.max(np.abs(v - s["v"])) < 1e-5
    assert np.max(np.abs(psi - s["psi"]) / s["psi"]) < 1e-6
