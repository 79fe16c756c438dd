"""ctypes front-end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg import this module; the product package never does.

It restates the host-side pieces of the reference that feed the kernels
(`laguerre.SpatialGrid`, laguerre.py:45-87; `_dpsi_max`, laguerre.py:142-145)
in numpy and binds the C restatement of `_kernels.py` (potflow_oracle.c) with
argument lists identical to the numba kernels, so a test can call
``oracle.batch_evaluate(*same_args)`` exactly like
``potflow._kernels._batch_evaluate(*same_args)``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libpotflow_oracle.so")

MAX_V, MAX_F, MAX_L, MAX_P = 512, 160, 2048, 256

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        d, i64, vp = C.c_double, C.c_int64, C.c_void_p
        L.pfo_batch_evaluate.restype = i64
        L.pfo_batch_evaluate.argtypes = (
            [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
             d, d, d, d, d, d, i64, i64, i64, d, d, d, C.c_int, C.c_int, i64]
            + [vp] * 12 + [i64, i64, vp, vp])
        L.pfo_batch_build.restype = i64
        L.pfo_batch_build.argtypes = (
            [i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
             d, d, d, d, d, d, i64, i64, i64, d, d, d, C.c_int, i64, i64, i64]
            + [vp] * 9)
        L.pfo_knn.restype = i64
        L.pfo_knn.argtypes = [i64, vp, vp, vp, d, d, d, d, d, d, i64, i64, i64, d,
                              d, d, d, i64, vp]
        L.pfo_clip.restype = C.c_int
        L.pfo_clip.argtypes = [vp] * 12 + [d, d, d, d, i64, d]
        L.pfo_piece_integrals.restype = None
        L.pfo_piece_integrals.argtypes = [vp, i64, vp]
        L.pfo_num_threads.restype = C.c_int
        L.pfo_set_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data if a is not None else None


def _chk(a, dtype):
    assert isinstance(a, np.ndarray) and a.dtype == dtype and a.flags.c_contiguous, \
        (a.dtype if isinstance(a, np.ndarray) else type(a))
    return a


def set_threads(n: int) -> int:
    lib().pfo_set_threads(int(n))
    return lib().pfo_num_threads()


def num_threads() -> int:
    return lib().pfo_num_threads()


# ---------------------------------------------------------------------------
# host-side restatements (laguerre.py)
# ---------------------------------------------------------------------------

class SpatialGrid:
    """Restatement of laguerre.SpatialGrid (laguerre.py:45-87)."""

    def __init__(self, points, lo, hi, domain_volume, target_cell_size=None):
        points = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        n = len(points)
        lo = np.asarray(lo, np.float64)
        hi = np.asarray(hi, np.float64)
        extent = np.maximum(hi - lo, 1e-300)
        if target_cell_size is None:
            target_cell_size = (domain_volume / max(n, 1)) ** (1.0 / 3.0)
        dims = np.clip(np.ceil(extent / max(target_cell_size, 1e-300)).astype(np.int64), 1, 128)
        h = extent / dims
        self.lo = lo.copy()
        self.dims = dims
        self.h = h
        self.inv_h = 1.0 / h
        self.h_min = float(h.min())
        self.points = points
        ij = np.clip(((points - lo) * self.inv_h).astype(np.int64), 0, dims - 1)
        lin = (ij[:, 0] * dims[1] + ij[:, 1]) * dims[2] + ij[:, 2]
        order = np.argsort(lin, kind="stable")
        ncell = int(dims[0] * dims[1] * dims[2])
        start = np.zeros(ncell + 1, dtype=np.int64)
        np.add.at(start, lin + 1, 1)
        np.cumsum(start, out=start)
        self.bucket_start = start
        self.bucket_sites = order.astype(np.int64)

    def kernel_args(self):
        return (self.bucket_start, self.bucket_sites,
                float(self.lo[0]), float(self.lo[1]), float(self.lo[2]),
                float(self.inv_h[0]), float(self.inv_h[1]), float(self.inv_h[2]),
                int(self.dims[0]), int(self.dims[1]), int(self.dims[2]),
                self.h_min)


def dpsi_max(psi) -> float:
    """laguerre._dpsi_max (laguerre.py:142-145)."""
    psi = np.asarray(psi)
    if len(psi) == 0:
        return 0.0
    return float(max(psi.max() - psi.min(), 0.0))


# ---------------------------------------------------------------------------
# kernels with the reference's argument lists (_kernels.py)
# ---------------------------------------------------------------------------

def batch_evaluate(pts, psi, dv, dc, dp, dt, dlp, dlv,
                   grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz,
                   gnx, gny, gnz, h_min, tol, dpsi_max_, ball_aware, want_m2, smf,
                   status, vol, ksur, cent, ipt, m2,
                   fcount, ftag, farea_o, fh_o, fnrm, fcent_o,
                   i0=0, i1=0, clip_count=None, cells=None):
    """_kernels._batch_evaluate (_kernels.py:1362-1478); optional [i0, i1) cell range
    (of ``cells`` when given: a bounded sample of cell indices)."""
    f8, i8 = np.float64, np.int64
    n = len(pts)
    args = [_chk(pts, f8), _chk(psi, f8), _chk(dv, f8), _chk(dc, i8), _chk(dp, f8),
            _chk(dt, i8), _chk(dlp, i8), _chk(dlv, i8), _chk(grid_start, i8),
            _chk(grid_sites, i8)]
    outs = [_chk(status, i8), _chk(vol, f8), _chk(ksur, f8), _chk(cent, f8), _chk(ipt, f8),
            _chk(m2, f8), _chk(fcount, i8), _chk(ftag, i8), _chk(farea_o, f8), _chk(fh_o, f8),
            _chk(fnrm, f8), _chk(fcent_o, f8)]
    if clip_count is not None:
        _chk(clip_count, i8)
    return int(lib().pfo_batch_evaluate(
        n, *[_p(a) for a in args], lox, loy, loz, ihx, ihy, ihz, gnx, gny, gnz, h_min, tol,
        dpsi_max_, int(bool(ball_aware)), int(bool(want_m2)), int(smf),
        *[_p(a) for a in outs], int(i0), int(i1), _p(clip_count),
        _p(None if cells is None else _chk(np.ascontiguousarray(cells, np.int64), i8))))


def batch_build(pts, psi, dv, dc, dp, dt, dlp, dlv,
                grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz,
                gnx, gny, gnz, h_min, tol, dpsi_max_, ball_aware,
                smv, smf, sml,
                out_status, out_nv, out_nf, out_nl,
                out_verts, out_planes, out_tags, out_lp, out_lv):
    """_kernels._batch_build (_kernels.py:1481-1559)."""
    f8, i8 = np.float64, np.int64
    n = len(pts)
    args = [_chk(pts, f8), _chk(psi, f8), _chk(dv, f8), _chk(dc, i8), _chk(dp, f8),
            _chk(dt, i8), _chk(dlp, i8), _chk(dlv, i8), _chk(grid_start, i8),
            _chk(grid_sites, i8)]
    outs = [_chk(out_status, i8), _chk(out_nv, i8), _chk(out_nf, i8), _chk(out_nl, i8),
            _chk(out_verts, f8), _chk(out_planes, f8), _chk(out_tags, i8), _chk(out_lp, i8),
            _chk(out_lv, i8)]
    return int(lib().pfo_batch_build(
        n, *[_p(a) for a in args], lox, loy, loz, ihx, ihy, ihz, gnx, gny, gnz, h_min, tol,
        dpsi_max_, int(bool(ball_aware)), int(smv), int(smf), int(sml),
        *[_p(a) for a in outs]))


def knn_kernel(pts, grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz,
               gnx, gny, gnz, h_min, qx, qy, qz, k, out_idx):
    """_kernels._knn (_kernels.py:1562-1620)."""
    return int(lib().pfo_knn(len(pts), _p(_chk(pts, np.float64)), _p(grid_start), _p(grid_sites),
                             lox, loy, loz, ihx, ihy, ihz, gnx, gny, gnz, h_min,
                             float(qx), float(qy), float(qz), int(k), _p(out_idx)))


def clip_into(va, ca, pa, ta, lpa, lva, vb, cb, pb, tb, lpb, lvb, nx, ny, nz, dd, tag, tol):
    """_kernels._clip_into (_kernels.py:109-319)."""
    return int(lib().pfo_clip(*[_p(a) for a in (va, ca, pa, ta, lpa, lva, vb, cb, pb, tb, lpb, lvb)],
                              float(nx), float(ny), float(nz), float(dd), int(tag), float(tol)))


def piece_integrals(pieces, npc):
    """_kernels._piece_integrals (_kernels.py:331-390)."""
    pieces = np.ascontiguousarray(pieces, dtype=np.float64)
    out = np.zeros(4)
    lib().pfo_piece_integrals(_p(pieces), int(npc), _p(out))
    return tuple(out)


def alloc_outputs(n: int, smf: int):
    """Caller-allocated outputs of _batch_evaluate (shapes per SURVEY.md §8(b))."""
    return dict(
        status=np.zeros(n, np.int64), vol=np.zeros(n), ksur=np.zeros(n),
        cent=np.zeros((n, 3)), ipt=np.zeros((n, 3)), m2=np.zeros(n),
        fcount=np.zeros(n, np.int64), ftag=np.zeros((n, smf), np.int64),
        farea=np.zeros((n, smf)), fh=np.zeros((n, smf)),
        fnrm=np.zeros((n, smf, 3)), fcent=np.zeros((n, smf, 3)))


OUT_ORDER = ("status", "vol", "ksur", "cent", "ipt", "m2",
             "fcount", "ftag", "farea", "fh", "fnrm", "fcent")


def evaluate(pts, psi, domain_pack_args, tol, grid: SpatialGrid, ball_aware=True,
             want_m2=True, smf=32, dpsi=None, i0=0, i1=0, clip_count=None, cells=None):
    """Convenience wrapper: allocate outputs and run batch_evaluate."""
    pts = np.ascontiguousarray(pts, np.float64)
    psi = np.ascontiguousarray(psi, np.float64)
    n = len(pts)
    o = alloc_outputs(n, smf)
    if dpsi is None:
        dpsi = dpsi_max(psi)
    err = batch_evaluate(pts, psi, *domain_pack_args, *grid.kernel_args(), tol, dpsi,
                         ball_aware, want_m2, smf, *[o[k] for k in OUT_ORDER],
                         i0=i0, i1=i1, clip_count=clip_count, cells=cells)
    o["err"] = err
    return o
