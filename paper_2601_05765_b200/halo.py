"""Distributed particle data plane of the x-slab decomposition.

Every rank holds only the particles it owns (global id, position, weight,
volume, ...) as device tensors; nothing is replicated.  Two exchanges move them:

* ``migrate`` -- after advection, particles whose x left the rank's slab go to
  the owning rank (one all-to-all of counts, one of packed rows);
* ``ghosts`` -- every rank q announces its ghost margin m_q (the largest
  ball-aware search radius of its owned cells, ``partition.search_radius``,
  times a slack); every rank sends each q its owned particles with x in
  [a_q - m_q, b_q + m_q] (again two all-to-alls).  The receiver merges owned
  and ghost rows in global-id order, so the (d^2, j) tie-break order of the
  cell kernels is the global one and per-cell results equal the single-GPU
  ones; the halo plan of the CG exchange falls out of the same message (what
  was sent to q / received from q, in global-id order on both sides).

The local set equals ``partition.halo_plan``'s (which derives it from
replicated global arrays) entry for entry: tests/test_halo_gloo.py.  The
collectives are ``torch.distributed`` all_to_all_single on the tensors'
device (NCCL over NVLink on GPUs; gloo stages CUDA tensors through the host).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .partition import HaloPlan, search_radius


@dataclass
class LocalSet:
    gid: "torch.Tensor"          # int64 [n_local], increasing
    fields: dict                 # name -> tensor [n_local, ...] in gid order
    owned: "torch.Tensor"        # int64 [n_owned] local indices of owned rows (increasing)
    plan: HaloPlan               # send / recv local indices per peer (numpy, gid order)
    margins: np.ndarray          # ghost margin of every rank
    lo: float
    hi: float

    @property
    def n_local(self) -> int:
        return int(self.gid.numel())


class SlabComm:
    """x-slabs with fixed interior cuts (``partition.slab_cuts``); ``comm`` is a
    ``dist_solver.Comm`` (rank, world, torch.distributed group)."""

    def __init__(self, cuts, comm):
        import torch

        self.torch = torch
        self.cuts = np.asarray(cuts, dtype=np.float64)
        self.comm = comm
        self.rank, self.world = comm.rank, comm.world

    def bounds(self, q: int):
        a = float(self.cuts[q - 1]) if q > 0 else -np.inf
        b = float(self.cuts[q]) if q < self.world - 1 else np.inf
        return a, b

    def owner(self, x):
        t = self.torch
        cuts = t.as_tensor(self.cuts, dtype=t.float64, device=x.device)
        return t.searchsorted(cuts, x.contiguous(), right=True)

    # --- packing -------------------------------------------------------------
    @staticmethod
    def _layout(fields: dict):
        return [(k, 1 if v.dim() == 1 else int(v.shape[1])) for k, v in fields.items()]

    def _pack(self, gid, fields, rows):
        t = self.torch
        cols = [gid.index_select(0, rows).to(t.float64)[:, None]]  # gid < 2^53: exact in f64
        for k, v in fields.items():
            r = v.index_select(0, rows).to(t.float64)
            cols.append(r[:, None] if r.dim() == 1 else r)
        return t.cat(cols, 1)

    def _unpack(self, mat, layout, like: dict):
        t = self.torch
        gid = mat[:, 0].to(t.int64)
        out, c = {}, 1
        for k, wdt in layout:
            v = mat[:, c:c + wdt]
            out[k] = (v[:, 0] if like[k].dim() == 1 else v).to(like[k].dtype).contiguous()
            c += wdt
        return gid, out

    def _alltoall(self, parts: list, width: int, device):
        """Exchange one row block per peer; returns (received rows stacked in
        source-rank order, rows received from each source)."""
        t = self.torch
        if not self.comm.active():
            return parts[self.rank], [int(parts[self.rank].shape[0]) if q == self.rank else 0
                                      for q in range(self.world)]
        d = self.comm.dist
        stage = self.comm.gloo and device.type == "cuda"
        dev = t.device("cpu") if stage else device
        cnt_s = t.tensor([int(p.shape[0]) for p in parts], dtype=t.int64, device=dev)
        cnt_r = t.empty_like(cnt_s)
        d.all_to_all_single(cnt_r, cnt_s, group=self.comm.group)
        cr = [int(v) for v in cnt_r.cpu()]
        send = t.cat([p.to(dev) for p in parts], 0).reshape(-1).contiguous()
        recv = t.empty(sum(cr) * width, dtype=t.float64, device=dev)
        d.all_to_all_single(recv, send, output_split_sizes=[c * width for c in cr],
                            input_split_sizes=[int(p.shape[0]) * width for p in parts], group=self.comm.group)
        return recv.reshape(-1, width).to(device), cr

    # --- exchanges -----------------------------------------------------------
    def migrate(self, gid, fields: dict):
        """Re-own particles by their x (fields['pts'][:, 0]); returns (gid,
        fields) of the particles this rank owns afterwards, in gid order."""
        t = self.torch
        own = self.owner(fields["pts"][:, 0])
        layout = self._layout(fields)
        width = 1 + sum(w for _, w in layout)
        parts = []
        for q in range(self.world):
            rows = t.nonzero(own == q).flatten() if q != self.rank else \
                t.zeros(0, dtype=t.int64, device=gid.device)
            parts.append(self._pack(gid, fields, rows))
        keep = t.nonzero(own == self.rank).flatten()
        got, _ = self._alltoall(parts, width, gid.device)
        rg, rf = self._unpack(got, layout, fields) if self.comm.active() else \
            (gid[:0], {k: v[:0] for k, v in fields.items()})
        g2 = t.cat([gid.index_select(0, keep), rg])
        order = t.argsort(g2)
        out = {k: t.cat([v.index_select(0, keep), rf[k]]).index_select(0, order).contiguous()
               for k, v in fields.items()}
        return g2.index_select(0, order).contiguous(), out

    def margins(self, margin_mine: float) -> np.ndarray:
        t = self.torch
        if not self.comm.active():
            return np.array([margin_mine])
        dev = "cuda" if (not self.comm.gloo and t.cuda.is_available()) else "cpu"
        m = t.zeros(self.world, dtype=t.float64, device=dev)
        m[self.rank] = margin_mine
        self.comm.all_reduce(m, "sum")
        return m.cpu().numpy()

    def ghosts(self, gid, fields: dict, margin_mine: float) -> LocalSet:
        """Owned rows (gid order, all inside this slab) + the ghost rows every
        other rank's owned particles contribute within this rank's margin."""
        t = self.torch
        dev = gid.device
        m = self.margins(margin_mine)
        x = fields["pts"][:, 0]
        layout = self._layout(fields)
        width = 1 + sum(w for _, w in layout)
        parts, sel = [], {}
        for q in range(self.world):
            if q == self.rank:
                rows = t.zeros(0, dtype=t.int64, device=dev)
            else:
                a, b = self.bounds(q)
                rows = t.nonzero((x >= a - m[q]) & (x <= b + m[q])).flatten()
                sel[q] = rows
            parts.append(self._pack(gid, fields, rows))
        got, cr = self._alltoall(parts, width, dev)
        no = int(gid.numel())
        if self.comm.active():
            rg, rf = self._unpack(got, layout, fields)
        else:
            rg, rf = gid[:0], {k: v[:0] for k, v in fields.items()}
        g2 = t.cat([gid, rg])
        order = t.argsort(g2)
        inv = t.empty_like(order)
        inv[order] = t.arange(order.numel(), device=dev)
        loc = {k: t.cat([v, rf[k]]).index_select(0, order).contiguous() for k, v in fields.items()}
        send = {q: inv.index_select(0, rows).cpu().numpy() for q, rows in sel.items() if rows.numel()}
        recv, off = {}, no
        for q in range(self.world):
            if q != self.rank and cr[q]:
                recv[q] = inv[off:off + cr[q]].cpu().numpy()
            off += cr[q] if q != self.rank else 0
        a, b = self.bounds(self.rank)
        return LocalSet(g2.index_select(0, order).contiguous(), loc, inv[:no].contiguous(),
                        HaloPlan(send, recv), m, a, b)


def ghost_margin(psi_owned: np.ndarray, dpsi: float, slack: float) -> float:
    """This rank's ghost margin: its largest ball-aware search radius (+1e-9,
    times the slack), as partition.slab_partition sizes it."""
    if len(psi_owned) == 0:
        return 0.0
    return float(search_radius(psi_owned, dpsi).max()) * (1.0 + 1e-9) * slack
