"""Multi-rank spatial decomposition on CPU (world_size 2, gloo): every rank
evaluates its x-slab with owned + ghost sites and the all-reduced dpsi; the
gathered per-cell results are bit-identical to the single-rank evaluation.
The cell evaluator here is the CPU oracle (no GPU in this container); the
device path consumes the same `partition.slab_partition` output."""
import os
import socket

import numpy as np
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

    sc = scenes.c2_dam_break(m=14)
    rng = np.random.default_rng(3)
    psi = (0.8 * sc.meta["h"] + 0.1 * sc.meta["h"] * rng.random(sc.n)) ** 2
    return sc.pts, psi


def _worker(rank, world, port, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre, partition

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    pts, psi = _scene()
    # each rank contributes only its own half of the weights to the dpsi reduction
    mine = (pts[:, 0] < 0.25) if rank == 0 else (pts[:, 0] >= 0.25)
    dpsi = partition.global_dpsi(psi[mine])
    slab = partition.slab_partition(pts, psi, dpsi, world, rank, 0.0, 0.5)
    lp, lw = pts[slab.local_to_global], psi[slab.local_to_global]
    dpk = laguerre.domain_pack(geom.box_domain([0, 0, 0], [1, 1, 1]))
    g = O.SpatialGrid(lp, [0, 0, 0], [1, 1, 1], 1.0)
    own = slab.owned_local.astype(np.int64)
    o = O.evaluate(lp, lw, dpk.args(), dpk.tol, g, smf=32, dpsi=dpsi, i0=0, i1=len(own), cells=own)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), gid=slab.local_to_global[own], vol=o["vol"][own],
             ksur=o["ksur"][own], fcount=o["fcount"][own],
             ftag=partition.to_global(slab, o["ftag"][own], o["fcount"][own]), farea=o["farea"][own],
             status=o["status"][own], dpsi=dpsi, n_local=slab.n_local)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_slabs_match_single_rank(tmp_path):
    from oracle import pyoracle as O
    from paper_2601_05765_b200 import geom, laguerre

    world, port = 2, _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    pts, psi = _scene()
    dpk = laguerre.domain_pack(geom.box_domain([0, 0, 0], [1, 1, 1]))
    g = O.SpatialGrid(pts, [0, 0, 0], [1, 1, 1], 1.0)
    ref = O.evaluate(pts, psi, dpk.args(), dpk.tol, g, smf=32)
    seen = np.zeros(len(pts), bool)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert float(d["dpsi"]) == O.dpsi_max(psi)
        assert int(d["n_local"]) < len(pts)  # ghosts are a proper subset
        gid = d["gid"]
        assert not seen[gid].any()
        seen[gid] = True
        for k in ("vol", "ksur", "fcount", "ftag", "farea", "status"):
            assert np.array_equal(d[k], ref[k][gid]), k
    assert seen.all()
