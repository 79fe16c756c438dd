"""Drop-in replacement of the reference's ``potflow._kernels`` batch entry points.

Same function names, same positional arguments, same output arrays and the
same returned flag word as /root/reference/pkg/src/potflow/_kernels.py, but
the work runs on the B200 through libpotflow_b200.so:

* ``_batch_evaluate``  _kernels.py:1362-1478 -> pf_batch_evaluate
* ``_batch_build``     _kernels.py:1481-1559 -> pf_batch_build
* ``_knn``             _kernels.py:1562-1620 -> pf_knn

Arrays may be numpy (copied to the device and back, as a drop-in for the numba
call) or torch CUDA tensors (used in place, no host round trip).  The host
grid arguments (grid_start ... h_min) are accepted for signature
compatibility; the device builds its own bucket grid from ``pts`` because the
processed-candidate order is the global (d^2, j) order either way
(_kernels.py:1293-1304), so results do not depend on the bucket layout.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .laguerre import upload_domain

MAX_V, MAX_F, MAX_L, MAX_P = 512, 160, 2048, 256
CLIP_CUT, CLIP_UNTOUCHED, CLIP_EMPTY, CLIP_OVERFLOW, CLIP_DEGENERATE = 0, 1, 2, 3, 4
RF_OUTSIDE, RF_UNTOUCHED, RF_FULLCIRCLE, RF_GENPOLY = 0, 1, 2, 3
CELL_EMPTY, CELL_FULLBALL, CELL_CLIPPED = 0, 1, 2
FLAG_OVERFLOW, FLAG_DEGENERATE_INTERIOR, FLAG_UNSTABLE_PROJECTION = 1, 2, 4


def _is_torch(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _to_dev(x, dtype):
    import torch

    if _is_torch(x):
        if x.device.type != "cuda" or x.dtype != dtype or not x.is_contiguous():
            raise TypeError("torch inputs must be contiguous CUDA tensors of the reference dtype")
        return x
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


def _host(x):
    if _is_torch(x):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _batch_evaluate(pts, psi, dv, dc, dp, dt, dlp, dlv,
                    grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz,
                    gnx, gny, gnz, h_min, tol, dpsi_max, ball_aware, want_m2,
                    smf,
                    status, vol, ksur, cent, ipt, m2,
                    fcount, ftag, farea_o, fh_o, fnrm, fcent_o, *, parity_mode=None):
    """Build and evaluate every restricted cell (see module docstring).
    ``parity_mode`` (keyword only; None = the context's setting, see
    ``_lib.set_parity_mode``): True restricts the facets exactly as the
    reference does, False with the robust correction."""
    with _lib.parity(parity_mode):
        return _batch_evaluate_impl(pts, psi, dv, dc, dp, dt, dlp, dlv, tol, dpsi_max, ball_aware,
                                    want_m2, smf, [status, vol, ksur, cent, ipt, m2, fcount, ftag,
                                                   farea_o, fh_o, fnrm, fcent_o])


def _batch_evaluate_impl(pts, psi, dv, dc, dp, dt, dlp, dlv, tol, dpsi_max, ball_aware, want_m2, smf,
                         outs_host):
    import torch

    f8, i8 = torch.float64, torch.int64
    dtypes = [i8, f8, f8, f8, f8, f8, i8, i8, f8, f8, f8, f8]
    on_device = _is_torch(pts)
    c = _lib.ctx()
    upload_domain(c, _host(dv), _host(dc), _host(dp), _host(dt), _host(dlp), _host(dlv), float(tol))
    if not on_device:
        return _batch_evaluate_host(c, pts, psi, tol, dpsi_max, ball_aware, want_m2, smf, outs_host,
                                    dtypes)
    p = _to_dev(pts, f8)
    w = _to_dev(psi, f8)
    outs = [_to_dev(o, t) for o, t in zip(outs_host, dtypes)]
    n = int(p.shape[0])
    err = int(_lib.lib().pf_batch_evaluate_ex(
        c, n, _lib.ptr(p), _lib.ptr(w), float(tol), float(dpsi_max), int(bool(ball_aware)),
        int(bool(want_m2)), int(smf), *[_lib.ptr(o) for o in outs], None, 0, None,
        None, 1, _lib.stream_ptr()))
    _lib.check(err, "pf_batch_evaluate_ex")
    return err


def _chunk_bounds(n: int, K: int) -> np.ndarray:
    """Index-range boundaries [0 = b_0 <= ... <= b_K = n] of the host drop-in's
    ranges (pf_batch_evaluate_host's range_bounds, pf_host.cu): equal, except
    the last three shrink (1/2, 1/4, 1/8 of one) so the work left after the
    last kernel is short, and with K >= 10 the first two (1/4, 1/2) so the
    host's scatter starts early."""
    wts = np.ones(K)
    if K >= 6:
        wts[-3:] = (0.5, 0.25, 0.125)
    if K >= 10:
        wts[:2] = (0.25, 0.5)
    bnd = np.rint(np.concatenate([[0.0], np.cumsum(wts)]) / wts.sum() * n).astype(np.int64)
    bnd[0], bnd[-1] = 0, n
    return bnd


def default_chunks(n: int) -> int:
    """Index ranges of the host drop-in: ~12k+ cells per range, 4 to 16 (fewer
    for small scenes, where each range's fixed cost shows: C2 97k 8.6 -> 6.9 ms
    with 8 instead of 16; C4 / C5 are fastest at 16)."""
    return int(min(16, max(4, n // 12000)))


# bytes copied host->device / device->host by the last host-array call
last_copy_bytes = (0, 0)


def _batch_evaluate_host(c, pts, psi, tol, dpsi_max, ball_aware, want_m2, smf, outs_host, dtypes,
                         chunks: int | None = None):
    """Host-array drop-in through pf_batch_evaluate_host (pf_host.cu): the
    caller's arrays (pageable numpy, as the numba kernel takes them) are read
    and written in place; only what the reference writes is written.  Output
    arrays that are not C-contiguous arrays of the reference dtype go through
    a temporary and are copied back."""
    import ctypes as C
    import os

    global last_copy_bytes
    npd = [np.int64, np.float64, np.float64, np.float64, np.float64, np.float64, np.int64, np.int64,
           np.float64, np.float64, np.float64, np.float64]
    p = np.ascontiguousarray(pts, np.float64).reshape(-1, 3)
    w = np.ascontiguousarray(psi, np.float64).reshape(-1)
    n = int(p.shape[0])
    direct, tmp = [], []
    for o, t in zip(outs_host, npd):
        if isinstance(o, np.ndarray) and o.dtype == t and o.flags.c_contiguous and o.flags.writeable:
            direct.append(o)
            tmp.append(None)
        else:
            a = np.array(_host(o), dtype=t, order="C", copy=True)
            direct.append(a)
            tmp.append(a)
    K = int(chunks or int(os.environ.get("PF_E2E_CHUNKS", "0")) or default_chunks(n))
    h2d, d2h = C.c_int64(0), C.c_int64(0)
    err = int(_lib.lib().pf_batch_evaluate_host(
        c, n, p.ctypes.data, w.ctypes.data, float(tol), float(dpsi_max), int(bool(ball_aware)),
        int(bool(want_m2)), int(smf), *[a.ctypes.data for a in direct], K, C.byref(h2d), C.byref(d2h)))
    _lib.check(err, "pf_batch_evaluate_host")
    last_copy_bytes = (int(h2d.value), int(d2h.value))
    for o, a in zip(outs_host, tmp):
        if a is not None:
            if _is_torch(o):
                o.copy_(__import__("torch").from_numpy(a).reshape(o.shape))
            else:
                o[...] = a.reshape(np.shape(o))
    return err


def _batch_build(pts, psi, dv, dc, dp, dt, dlp, dlv,
                 grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz,
                 gnx, gny, gnz, h_min, tol, dpsi_max, ball_aware,
                 smv, smf, sml,
                 out_status, out_nv, out_nf, out_nl,
                 out_verts, out_planes, out_tags, out_lp, out_lv):
    """Build every Laguerre cell into fixed-stride packed storage (returns the flag word)."""
    import torch

    f8, i8 = torch.float64, torch.int64
    outs_host = [out_status, out_nv, out_nf, out_nl, out_verts, out_planes, out_tags, out_lp, out_lv]
    dtypes = [i8, i8, i8, i8, f8, f8, i8, i8, i8]
    c = _lib.ctx()
    upload_domain(c, _host(dv), _host(dc), _host(dp), _host(dt), _host(dlp), _host(dlv), float(tol))
    on_device = _is_torch(pts)
    p, w = _to_dev(pts, f8), _to_dev(psi, f8)
    if on_device:
        outs = [_to_dev(o, t) for o, t in zip(outs_host, dtypes)]
    else:
        # the reference writes only the used prefix of each row: start from the caller's arrays
        outs = [torch.from_numpy(np.ascontiguousarray(o)).to("cuda") for o in outs_host]
    n = int(p.shape[0])
    err = int(_lib.lib().pf_batch_build(
        c, n, _lib.ptr(p), _lib.ptr(w), float(tol), float(dpsi_max), int(bool(ball_aware)), int(smv),
        int(smf), int(sml), *[_lib.ptr(o) for o in outs], 1, _lib.stream_ptr()))
    _lib.check(err, "pf_batch_build")
    if not on_device:
        for h, d in zip(outs_host, outs):
            h[...] = d.cpu().numpy().reshape(h.shape)
    return err


def _knn(pts, grid_start, grid_sites, lox, loy, loz, ihx, ihy, ihz,
         gnx, gny, gnz, h_min, qx, qy, qz, k, out_idx):
    """Exact k nearest sites of one query (writes out_idx, returns the count)."""
    import torch

    from .geom import box_domain

    p = _to_dev(pts, torch.float64)
    n = int(p.shape[0])
    kk = min(int(k), n)
    if kk <= 0:
        return 0
    lo = np.array([lox, loy, loz], dtype=np.float64)
    hi = lo + np.array([gnx / ihx, gny / ihy, gnz / ihz])
    from .laguerre import domain_pack

    dom = box_domain(lo, hi)
    dpk = domain_pack(dom)
    c = _lib.ctx()
    upload_domain(c, *dpk.args(), dpk.tol)
    q = torch.tensor([[qx, qy, qz]], dtype=torch.float64, device="cuda")
    res = torch.empty((1, kk), dtype=torch.int64, device="cuda")
    got = _lib.check(_lib.lib().pf_knn(c, n, _lib.ptr(p), 1, _lib.ptr(q), kk, _lib.ptr(res),
                                       1, _lib.stream_ptr()), "pf_knn")
    vals = res[0, :got]
    if _is_torch(out_idx):
        out_idx[:got] = vals
    else:
        out_idx[:got] = vals.cpu().numpy()
    return int(got)
