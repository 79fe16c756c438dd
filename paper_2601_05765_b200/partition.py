"""Spatial decomposition of the cell evaluation across ranks.

Rank r owns the sites of an x-slab and holds, as ghosts, every site within the
largest ball-aware search radius of its owned cells,

    W_r = max_{i owned} sqrt(psi_i) + sqrt(psi_i + dpsi),   dpsi = global max - min

(the reference's stop radius, _kernels.py:1239-1248), so each owned cell sees
exactly the candidates it sees on one GPU.  The local site array keeps the
global index order (owned and ghosts merged, sorted), so the (d^2, j)
tie-break order is unchanged and per-cell outputs are bit-identical to the
single-GPU run: the evaluation needs no collective beyond the scalar dpsi
all-reduce.  Facet tags come back as local indices; `to_global` maps them.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Slab:
    rank: int
    world: int
    lo: float
    hi: float
    local_to_global: np.ndarray  # int64 [n_local], increasing
    owned_local: np.ndarray      # int32 [n_owned] local indices of owned sites
    ghost_margin: float

    @property
    def n_local(self) -> int:
        return len(self.local_to_global)


def global_dpsi(psi_local: np.ndarray, group=None) -> float:
    """max(psi) - min(psi) over all ranks (one all-reduce of two scalars)."""
    import torch
    import torch.distributed as dist

    lo = float(psi_local.min()) if len(psi_local) else np.inf
    hi = float(psi_local.max()) if len(psi_local) else -np.inf
    if dist.is_available() and dist.is_initialized():
        dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor([-lo, hi], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        lo, hi = -float(t[0]), float(t[1])
    return max(hi - lo, 0.0) if np.isfinite(hi) else 0.0


def slab_cuts(x: np.ndarray, world: int, lo: float | None = None, hi: float | None = None) -> np.ndarray:
    """Interior slab boundaries along x: equal-width over [lo, hi] when given,
    else at the x-quantiles of the sites (equal cell counts per rank)."""
    if world <= 1:
        return np.zeros(0)
    if lo is not None and hi is not None:
        return lo + (hi - lo) * np.arange(1, world) / world
    return np.quantile(np.asarray(x, dtype=np.float64), np.arange(1, world) / world)


def slab_owner(x: np.ndarray, world: int, lo: float | None = None, hi: float | None = None,
               cuts: np.ndarray | None = None) -> np.ndarray:
    """Rank owning each x coordinate (slab k = [cuts[k-1], cuts[k]))."""
    if cuts is None:
        cuts = slab_cuts(x, world, lo, hi)
    return np.searchsorted(cuts, np.asarray(x), side="right").astype(np.int64)


def search_radius(psi: np.ndarray, dpsi: float) -> np.ndarray:
    """Ball-aware stop radius sqrt(psi) + sqrt(psi + dpsi) (_kernels.py:1239-1248)."""
    p = np.maximum(np.asarray(psi, dtype=np.float64), 0.0)
    return np.sqrt(p) + np.sqrt(p + dpsi)


def slab_partition(pts: np.ndarray, psi: np.ndarray, dpsi: float, world: int, rank: int,
                   lo: float | None = None, hi: float | None = None, slack: float = 1.0) -> Slab:
    """x-slab r of [lo, hi] with its ghost sites (pts / psi are the global arrays).

    ``slack`` > 1 widens the ghost margin beyond the current search radius so a
    Newton solve (whose weights grow) can keep the partition for several
    iterations; `DistNewton` checks the margin before every evaluation."""
    x = pts[:, 0]
    cuts = slab_cuts(x, world, lo, hi)
    a = float(cuts[rank - 1]) if rank > 0 else -np.inf
    b = float(cuts[rank]) if rank < world - 1 else np.inf
    own = slab_owner(x, world, cuts=cuts) == rank
    br = search_radius(psi, dpsi)
    margin = float(br[own].max()) * (1.0 + 1e-9) * slack if own.any() else 0.0
    keep = own | ((x >= a - margin) & (x <= b + margin))
    idx = np.nonzero(keep)[0].astype(np.int64)
    owned_local = np.nonzero(own[idx])[0].astype(np.int32)
    return Slab(rank, world, a, b, idx, owned_local, margin)


def to_global(slab: Slab, ftag_local: np.ndarray, fcount: np.ndarray) -> np.ndarray:
    """Map the used site tags (>= 0, slot < fcount) to global indices."""
    out = np.array(ftag_local, copy=True)
    used = np.arange(out.shape[1])[None, :] < np.asarray(fcount)[:, None]
    m = used & (out >= 0)
    out[m] = slab.local_to_global[out[m]]
    return out


@dataclass
class HaloPlan:
    """Who sends which owned entries to whom.  For every peer q: ``send[q]``
    are local indices of this rank's owned sites that are ghosts of q, and
    ``recv[q]`` the local indices of this rank's ghosts owned by q; both are in
    global index order, so the two sides of a message agree entry by entry."""
    send: dict
    recv: dict

    def volume(self) -> int:
        return int(sum(len(v) for v in self.send.values()))


def halo_plan(pts: np.ndarray, psi: np.ndarray, dpsi: float, world: int, rank: int,
              lo: float | None = None, hi: float | None = None, slack: float = 1.0):
    """(slab of this rank, halo plan).  Every rank derives every other rank's
    ghost set from the replicated global arrays, so no negotiation is needed."""
    slabs = [slab_partition(pts, psi, dpsi, world, q, lo, hi, slack) for q in range(world)]
    me = slabs[rank]
    owner = slab_owner(pts[:, 0], world, lo, hi)
    send, recv = {}, {}
    for q in range(world):
        if q == rank:
            continue
        ghosts_q = slabs[q].local_to_global
        ghosts_q = ghosts_q[owner[ghosts_q] == rank]           # q's ghosts that I own (sorted)
        if len(ghosts_q):
            send[q] = np.searchsorted(me.local_to_global, ghosts_q).astype(np.int64)
        mine_from_q = me.local_to_global[owner[me.local_to_global] == q]  # my ghosts owned by q
        if len(mine_from_q):
            recv[q] = np.searchsorted(me.local_to_global, mine_from_q).astype(np.int64)
    return me, HaloPlan(send, recv)
