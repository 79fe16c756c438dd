"""Laguerre-diagram plumbing on the B200: domain pack, bucket grid, kNN.

Mirrors the reference's ``potflow.laguerre`` host API
(/root/reference/pkg/src/potflow/laguerre.py) with the per-site work moved to
the device:

* ``Site`` / ``sites_to_arrays``     laguerre.py:20-42   (host, unchanged semantics)
* ``SpatialGrid``                    laguerre.py:45-87   counting sort on the GPU (pf_grid_build)
* ``knn``                            laguerre.py:90-96   batched warp-per-query kernel (pf_knn)
* ``bisector_plane``                 laguerre.py:99-110
* ``domain_pack`` / ``_DomainPack``  laguerre.py:113-139
* ``_dpsi_max``                      laguerre.py:142-145 (device min/max reduction)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geom import DEFAULT_REL_TOL, ConvexCell, Plane, cell_volume_convex, pack_cell


@dataclass
class Site:
    p: np.ndarray
    psi: float = 0.0
    nu: float = 1.0
    phase: int = 0

    def __post_init__(self):
        self.p = np.asarray(self.p, dtype=np.float64)
        if self.psi < 0.0:
            raise ValueError("site weight must be non-negative")
        if self.nu <= 0.0:
            raise ValueError("prescribed volume must be positive")


def sites_to_arrays(sites: list):
    pts = np.array([s.p for s in sites], dtype=np.float64).reshape(-1, 3)
    return (pts, np.array([s.psi for s in sites], dtype=np.float64),
            np.array([s.nu for s in sites], dtype=np.float64),
            np.array([s.phase for s in sites], dtype=np.int64))


def bisector_plane(p_i, psi_i, p_j, psi_j) -> Plane:
    """Power bisector of (p_i, psi_i), (p_j, psi_j), cell i inside (laguerre.py:99-110)."""
    p_i = np.asarray(p_i, dtype=np.float64)
    p_j = np.asarray(p_j, dtype=np.float64)
    diff = p_j - p_i
    D2 = float(diff @ diff)
    if D2 == 0.0:
        raise ValueError("coincident sites have no bisector")
    D = np.sqrt(D2)
    n = diff / D
    return Plane(n, float(n @ p_i) + 0.5 * (D2 + psi_i - psi_j) / D)


class _DomainPack:
    """Packed domain + tolerance + volume (laguerre.py:113-129)."""

    def __init__(self, domain: ConvexCell):
        self.cell = domain
        self.verts, self.cnt, self.planes, self.tags, self.lp, self.lv = pack_cell(domain)
        self.tol = DEFAULT_REL_TOL * domain.diagonal()
        self.volume = cell_volume_convex(domain)

    def args(self):
        return (self.verts, self.cnt, self.planes, self.tags, self.lp, self.lv)


_pack_cache: dict[int, _DomainPack] = {}


def domain_pack(domain: ConvexCell) -> _DomainPack:
    dp = _pack_cache.get(id(domain))
    if dp is None or dp.cell is not domain:
        dp = _DomainPack(domain)
        _pack_cache.clear()
        _pack_cache[id(domain)] = dp
    return dp


# which packed domain is resident in each device context
_resident: dict[int, tuple] = {}


def upload_domain(ctx, dv, dc, dp, dt, dlp, dlv, tol: float) -> None:
    """Make the packed domain resident in the device context (pf_set_domain)."""
    arrs = [np.ascontiguousarray(np.asarray(a), dtype=t) for a, t in
            ((dv, np.float64), (dc, np.int64), (dp, np.float64), (dt, np.int64),
             (dlp, np.int64), (dlv, np.int64))]
    nv, nf, nl = (int(x) for x in arrs[1][:3])
    key = (float(tol), arrs[0][:nv].tobytes(), arrs[2][:nf].tobytes(), arrs[3][:nf].tobytes(),
           arrs[4][:nf + 1].tobytes(), arrs[5][:nl].tobytes())
    if _resident.get(ctx.value) == key:
        return
    _lib.check(_lib.lib().pf_set_domain(ctx, *[a.ctypes.data for a in arrs], float(tol)),
               "pf_set_domain")
    _resident[ctx.value] = key


def _dev(x, dtype):
    import torch

    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            x = x.cuda()
        return x.to(dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def _dpsi_max(psi) -> float:
    """max(psi) - min(psi), >= 0 (laguerre.py:142-145), reduced on the device."""
    import torch

    t = _dev(psi, torch.float64)
    if t.numel() == 0:
        return 0.0
    out = C.c_double(0.0)
    _lib.check(_lib.lib().pf_dpsi_max(_lib.ctx(), t.numel(), _lib.ptr(t), C.byref(out),
                                      _lib.stream_ptr()), "pf_dpsi_max")
    return float(out.value)


class SpatialGrid:
    """Uniform bucket grid over the domain bounding box, built on the GPU.

    ``target_cell_size=None`` reproduces the reference's bucket edge
    (|domain|/n)^(1/3) with dims clipped to [1, 128] (laguerre.py:59-64), so
    ``bucket_start`` / ``bucket_sites`` / ``kernel_args()`` equal the
    reference's arrays (sites ordered by bucket, then index, as numpy's stable
    argsort gives).  The evaluation kernels build their own, finer grid.
    """

    def __init__(self, points, domain: ConvexCell, target_cell_size: float | None = None):
        import torch

        pts = _dev(points, torch.float64).reshape(-1, 3)
        n = pts.shape[0]
        lo, hi = domain.bbox()
        extent = np.maximum(hi - lo, 1e-300)
        if target_cell_size is None:
            target_cell_size = (cell_volume_convex(domain) / max(n, 1)) ** (1.0 / 3.0)
        dims = np.clip(np.ceil(extent / max(target_cell_size, 1e-300)).astype(np.int64), 1, 128)
        h = extent / dims
        self.lo = lo.copy()
        self.dims = dims
        self.h = h
        self.inv_h = 1.0 / h
        self.h_min = float(h.min())
        self.points = pts
        dpk = domain_pack(domain)
        c = _lib.ctx()
        upload_domain(c, *dpk.args(), dpk.tol)
        gdims = (C.c_int * 3)(*[int(x) for x in dims])
        _lib.check(_lib.lib().pf_grid_build_dims(c, n, _lib.ptr(pts), gdims, _lib.stream_ptr()),
                   "pf_grid_build_dims")
        ncell = int(dims.prod())
        self.bucket_start = torch.empty(ncell + 1, dtype=torch.int64, device="cuda")
        self.bucket_sites = torch.empty(n, dtype=torch.int64, device="cuda")
        _lib.check(_lib.lib().pf_grid_export(c, _lib.ptr(self.bucket_start),
                                             _lib.ptr(self.bucket_sites), _lib.stream_ptr()),
                   "pf_grid_export")

    def kernel_args(self):
        return (self.bucket_start, self.bucket_sites,
                float(self.lo[0]), float(self.lo[1]), float(self.lo[2]),
                float(self.inv_h[0]), float(self.inv_h[1]), float(self.inv_h[2]),
                int(self.dims[0]), int(self.dims[1]), int(self.dims[2]), self.h_min)


def knn_batch(points, queries, k: int, domain: ConvexCell):
    """k nearest sites of every query, ordered by (distance, index); int64 [nq, min(k, n)]."""
    import torch

    pts = _dev(points, torch.float64).reshape(-1, 3)
    q = _dev(queries, torch.float64).reshape(-1, 3)
    n = pts.shape[0]
    kk = min(int(k), n)
    out = torch.empty((q.shape[0], max(kk, 0)), dtype=torch.int64, device="cuda")
    if kk <= 0 or q.shape[0] == 0:
        return out
    c = _lib.ctx()
    dpk = domain_pack(domain)
    upload_domain(c, *dpk.args(), dpk.tol)
    got = _lib.check(_lib.lib().pf_knn(c, n, _lib.ptr(pts), q.shape[0], _lib.ptr(q), kk,
                                       _lib.ptr(out), 1, _lib.stream_ptr()), "pf_knn")
    return out[:, :got]


def knn(grid: SpatialGrid, q, k: int, domain: ConvexCell | None = None) -> np.ndarray:
    """Indices of the k nearest sites to q by increasing distance (laguerre.py:90-96)."""
    if domain is None:
        lo = grid.lo
        hi = grid.lo + grid.h * grid.dims
        from .geom import box_domain

        domain = box_domain(lo, hi)
    return knn_batch(grid.points, np.asarray(q, dtype=np.float64).reshape(1, 3), k,
                     domain)[0].cpu().numpy()


def build_cell(i: int, sites, domain: ConvexCell, grid=None, ball_aware: bool = False):
    """Laguerre cell of site i inside the domain; None when the cell is empty
    (reference laguerre.py:148-183, same arguments and errors).

    The device builds the cell from the sites within a radius r of p_i, in
    their global index order (so the (d^2, j) candidate order and the
    coincident-site rule are the reference's) with the GLOBAL weight range
    max psi - min psi, the reference's security-radius slack.  The result is the
    reference's cell once r covers every site the build can process: the
    ball-aware radius sqrt(psi_i) + sqrt(psi_i + dpsi) in ball-aware mode; in
    full mode the subset cell's own security radius rfar + sqrt(rfar^2 +
    dpsi) (beyond it no site can cut), else r grows and the cell is rebuilt.
    ``grid`` is accepted for signature compatibility."""
    from . import _kernels as _k
    from .geom import unpack_cell

    if isinstance(sites, (list, tuple)) and len(sites) and isinstance(sites[0], Site):
        pts, psi, _, _ = sites_to_arrays(sites)
    else:
        pts, psi = sites
        pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
        psi = np.asarray(psi, dtype=np.float64)
    n = len(pts)
    i = int(i)
    if not 0 <= i < n:
        raise IndexError(f"site index {i} out of range for {n} sites")
    dp = domain_pack(domain)
    dpsi = float(max(psi.max() - psi.min(), 0.0))
    d2 = np.sum((pts - pts[i]) ** 2, axis=1)
    psii = float(psi[i])
    if ball_aware and psii > 0.0:
        r = (np.sqrt(psii) + np.sqrt(psii + dpsi)) * (1.0 + 1e-9)
    else:
        # full mode: start from the distance that holds ~64 sites, grow as needed
        r = float(np.sqrt(np.partition(d2, min(64, n - 1))[min(64, n - 1)])) * 1.5 + 1e-12
    gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
    while True:
        sub = np.nonzero(d2 <= r * r)[0]  # increasing global indices, contains i
        m, li = len(sub), int(np.searchsorted(sub, i))
        smv, smf, sml = 128, 64, 512
        while True:  # the reference's capacities, reached by doubling strides as build_diagram_packed
            status = np.zeros(m, dtype=np.int64)
            nv, nf, nl = (np.zeros(m, dtype=np.int64) for _ in range(3))
            verts, planes = np.zeros((m, smv, 3)), np.zeros((m, smf, 4))
            tags, lp, lv = (np.zeros((m, smf), dtype=np.int64), np.zeros((m, smf + 1), dtype=np.int64),
                            np.zeros((m, sml), dtype=np.int64))
            _k._batch_build(pts[sub], psi[sub], *dp.args(), *gargs, dp.tol, dpsi, ball_aware, smv, smf, sml,
                            status, nv, nf, nl, verts, planes, tags, lp, lv)
            if status[li] != 3 or (smv, smf, sml) == (_k.MAX_V, _k.MAX_F, _k.MAX_L):
                break
            smv, smf, sml = min(2 * smv, _k.MAX_V), min(2 * smf, _k.MAX_F), min(2 * sml, _k.MAX_L)
        st = int(status[li])
        if st == 3:
            raise RuntimeError("cell exceeded kernel buffer capacity")
        if st == 1:
            return None
        # ball-aware: the subset holds every site within the stop radius (psi_i > 0) or
        # the build processes none (psi_i <= 0: the domain cell, _kernels.py:1239-1248)
        done = ball_aware or m == n
        if not done:
            v = verts[li, :int(nv[li])]
            rfar = float(np.sqrt(np.max(np.sum((v - pts[i]) ** 2, axis=1))))
            need = rfar + np.sqrt(rfar * rfar + dpsi)
            done = need * (1.0 + 1e-9) <= r
            r = max(2.0 * r, need * 1.01)
        if done:
            nfi = int(nf[li])
            t = np.zeros(_k.MAX_F, dtype=np.int64)
            t[:nfi] = np.where(tags[li, :nfi] >= 0, sub[np.maximum(tags[li, :nfi], 0)], tags[li, :nfi])
            lpi = np.zeros(_k.MAX_F + 1, dtype=np.int64)
            lpi[:nfi + 1] = lp[li, :nfi + 1]
            vi = np.zeros((_k.MAX_V, 3))
            vi[:int(nv[li])] = verts[li, :int(nv[li])]
            pli = np.zeros((_k.MAX_F, 4))
            pli[:nfi] = planes[li, :nfi]
            lvi = np.zeros(_k.MAX_L, dtype=np.int64)
            lvi[:int(nl[li])] = lv[li, :int(nl[li])]
            return unpack_cell(vi, np.array([nv[li], nfi, nl[li]]), pli, t, lpi, lvi)


class PackedDiagram:
    """All unrestricted Laguerre cells in fixed-stride packed storage
    (laguerre.py:186-222 of the reference; host numpy arrays)."""

    def __init__(self, pts, psi, status, nv, nf, nl, verts, planes, tags, lp, lv, domain: ConvexCell):
        self.pts, self.psi = pts, psi
        self.status, self.nv, self.nf, self.nl = status, nv, nf, nl  # status 0 ok, 1 empty
        self.verts, self.planes, self.tags, self.lp, self.lv = verts, planes, tags, lp, lv
        self.domain = domain

    def __len__(self):
        return len(self.status)

    def is_empty(self, i: int) -> bool:
        return self.status[i] != 0

    def cell(self, i: int):
        from . import _kernels as _k
        from .geom import unpack_cell

        if self.status[i] != 0:
            return None
        nf = int(self.nf[i])
        lp = np.empty(_k.MAX_F + 1, dtype=np.int64)
        lp[:nf + 1] = self.lp[i, :nf + 1]
        return unpack_cell(self.verts[i], np.array([self.nv[i], nf, self.nl[i]]), self.planes[i],
                           self.tags[i], lp, self.lv[i])

    def neighbors(self, i: int) -> np.ndarray:
        """Site indices of the facet neighbours of cell i."""
        t = self.tags[i, :int(self.nf[i])]
        return t[t >= 0]


def build_diagram_packed(sites, domain: ConvexCell, grid=None, ball_aware: bool = False) -> PackedDiagram:
    """Every Laguerre cell on the device (pf_batch_build), with the reference's
    capacity-doubling retry (laguerre.py:226-265).  ``grid`` is accepted for
    signature compatibility; the device builds its own bucket grid."""
    from . import _kernels as _k

    if isinstance(sites, (list, tuple)) and len(sites) and isinstance(sites[0], Site):
        pts, psi, _, _ = sites_to_arrays(sites)
    else:
        pts, psi = sites
        pts = np.asarray(pts, dtype=np.float64).reshape(-1, 3)
        psi = np.asarray(psi, dtype=np.float64)
    n = len(pts)
    dp = domain_pack(domain)
    gargs = (None, None, 0.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1, 1, 1, 1.0)
    dpsi = float(max(psi.max() - psi.min(), 0.0)) if n else 0.0
    smv, smf, sml = 128, 64, 512
    while True:
        status = np.zeros(n, dtype=np.int64)
        nv, nf, nl = (np.zeros(n, dtype=np.int64) for _ in range(3))
        verts, planes = np.zeros((n, smv, 3)), np.zeros((n, smf, 4))
        tags, lp, lv = (np.zeros((n, smf), dtype=np.int64), np.zeros((n, smf + 1), dtype=np.int64),
                        np.zeros((n, sml), dtype=np.int64))
        err = _k._batch_build(pts, psi, *dp.args(), *gargs, dp.tol, dpsi, ball_aware, smv, smf, sml,
                              status, nv, nf, nl, verts, planes, tags, lp, lv)
        if err == 0:
            break
        smv, smf, sml = smv * 2, smf * 2, sml * 2
        if smv > _k.MAX_V or smf > _k.MAX_F * 2 or sml > _k.MAX_L:
            raise RuntimeError("diagram cell exceeded kernel buffer capacity")
        smv, smf, sml = min(smv, _k.MAX_V), min(smf, _k.MAX_F), min(sml, _k.MAX_L)
    return PackedDiagram(pts, psi, status, nv, nf, nl, verts, planes, tags, lp, lv, domain)


def build_diagram(sites, domain: ConvexCell, grid=None, ball_aware: bool = False) -> list:
    """One Laguerre cell per site; empty cells are None (laguerre.py:268-272)."""
    packed = build_diagram_packed(sites, domain, grid, ball_aware)
    return [packed.cell(i) for i in range(len(packed))]
