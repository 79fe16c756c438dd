"""The exchange data plane on the device (halo.py, DistNewtonLocal, DistFluid
over dist_solver.CudaOps / the pf_fluid_* kernels):

* two ranks sharing cuda:0 over gloo (the exchanges staged through the host)
  against one rank -- Newton from owned sites only, then fluid steps with
  migration across the slab cut;
* the same over NCCL on two GPUs when the box has them (skipped otherwise:
  the pool's boxes have one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu
STEPS = 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world, out, device):
    import sys

    sys.path.insert(0, ROOT)
    from paper_2601_05765_b200 import dist_fluid, dist_solver, fluid, geom, partition, scenes

    sc = scenes.c2_dam_break(m=16)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    cuts = np.array([0.25]) if world == 2 else np.zeros(0)
    gid = np.nonzero(partition.slab_owner(sc.pts[:, 0], world, cuts=cuts) == rank)[0]
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=device)  # noqa: E731
    # Newton from owned sites only
    res = dist_solver.DistNewtonLocal(t(gid), t(sc.pts[gid]), t(sc.nu[gid]), dom, cuts, slack=1.2).solve()
    # fluid steps (the block moves right across the cut)
    v = np.zeros_like(sc.pts)
    v[:, 0] = 5.0
    df = dist_fluid.DistFluid(t(gid), sc.pts[gid], v[gid], sc.nu[gid], np.full(sc.n, 1000.0)[gid], dom, cuts,
                              fluid.SimParams(dt=2e-3, eps=5e-3), slack=1.5)
    for _ in range(STEPS):
        df.step()
    np.savez(out, ngid=res.owned_global, npsi=res.psi_owned, nit=res.stats["iterations"],
             nev=res.stats["evaluations"], gid=df.gid.cpu().numpy(), x=df.x.cpu().numpy(),
             v=df.v.cpu().numpy(), psi=df.psi.cpu().numpy(), it=[h["iterations"] for h in df.history])


def _worker(rank, world, port, out_dir, backend):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = rank if backend == "nccl" else 0
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    _run(rank, world, os.path.join(out_dir, f"r{rank}.npz"), "cuda")
    dist.barrier()
    dist.destroy_process_group()


def _check(tmp_path, single):
    s = np.load(single)
    n = len(s["ngid"])
    npsi, x, v, psi = np.full(n, np.nan), np.full((n, 3), np.nan), np.full((n, 3), np.nan), np.full(n, np.nan)
    for r in range(2):
        d = np.load(tmp_path / f"r{r}.npz")
        npsi[d["ngid"]] = d["npsi"]
        x[d["gid"]], v[d["gid"]], psi[d["gid"]] = d["x"], d["v"], d["psi"]
        assert int(d["nit"]) == int(s["nit"]) and int(d["nev"]) == int(s["nev"])
        assert list(d["it"]) == list(s["it"])
    assert np.isfinite(npsi).all() and np.isfinite(x).all()
    assert np.max(np.abs(npsi - s["npsi"]) / s["npsi"]) < 1e-6
    assert np.max(np.abs(x - s["x"])) < 1e-9
    assert np.max(np.abs(v - s["v"])) < 1e-5
    assert np.max(np.abs(psi - s["psi"]) / s["psi"]) < 1e-6


def test_two_ranks_one_device_gloo(tmp_path):
    _run(0, 1, str(tmp_path / "single.npz"), "cuda")
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), "gloo"), nprocs=2, join=True,
                       start_method="spawn")
    _check(tmp_path, tmp_path / "single.npz")


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="NCCL data plane needs 2 GPUs (the pool's boxes have 1)")
def test_two_gpus_nccl(tmp_path):
    _run(0, 1, str(tmp_path / "single.npz"), "cuda")
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), "nccl"), nprocs=2, join=True,
                       start_method="spawn")
    _check(tmp_path, tmp_path / "single.npz")


def _worker_one_nccl(rank, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PF_DIST_FORCE_COLLECTIVES="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    _run(0, 1, out, "cuda")
    dist.barrier()
    dist.destroy_process_group()


def test_one_rank_nccl_collectives(tmp_path):
    """The data plane's collectives (all_to_all_single of counts and rows for
    the ghosts and the migration, the all-reduces of the Newton / PCG scalars)
    over NCCL on the box's one GPU (PF_DIST_FORCE_COLLECTIVES: issued even
    with one rank): same Newton and fluid results as without torch.distributed."""
    _run(0, 1, str(tmp_path / "single.npz"), "cuda")
    mp.start_processes(_worker_one_nccl, args=(_free_port(), str(tmp_path / "nccl.npz")), nprocs=1, join=True,
                       start_method="spawn")
    s, d = np.load(tmp_path / "single.npz"), np.load(tmp_path / "nccl.npz")
    assert int(d["nit"]) == int(s["nit"]) and int(d["nev"]) == int(s["nev"])
    assert list(d["it"]) == list(s["it"])
    for k in ("npsi", "x", "v", "psi"):
        assert np.array_equal(d[k], s[k]), k
