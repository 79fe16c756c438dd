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
                    fcount, ftag, farea_o, fh_o, fnrm, fcent_o):
    """Build and evaluate every restricted cell (see module docstring)."""
    import torch

    f8, i8 = torch.float64, torch.int64
    outs_host = [status, vol, ksur, cent, ipt, m2, fcount, ftag, farea_o, fh_o, fnrm, fcent_o]
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
    ranges: equal, except the last three shrink (1/2, 1/4, 1/8 of one) so the
    device->host copy left after the last kernel is short."""
    wts = np.ones(K)
    if K >= 6:
        wts[-3:] = (0.5, 0.25, 0.125)
    bnd = np.rint(np.concatenate([[0.0], np.cumsum(wts)]) / wts.sum() * n).astype(np.int64)
    bnd[0], bnd[-1] = 0, n
    return bnd


def _batch_evaluate_host(c, pts, psi, tol, dpsi_max, ball_aware, want_m2, smf, outs_host, dtypes,
                         chunks: int | None = None):
    """Host-array drop-in: inputs copied in, every output copied back into the
    caller's arrays.  The cells are evaluated in `chunks` index ranges (each in
    bucket order) and the device->host copy of one range runs on a side stream
    while the next range computes, so the round trip hides behind the kernels
    (the copies are asynchronous when the caller's arrays are pinned)."""
    import os

    import torch

    L = _lib.lib()
    n = int(np.asarray(pts).shape[0])
    K = chunks or int(os.environ.get("PF_E2E_CHUNKS", "16"))
    K = max(1, min(K, max(n, 1)))

    def h2d(x, dtype):
        return torch.from_numpy(np.ascontiguousarray(x, dtype)).to("cuda", non_blocking=True)

    bnd = _chunk_bounds(n, K)
    p = h2d(pts, np.float64)
    w = h2d(psi, np.float64)
    outs = [torch.empty(o.shape, dtype=t, device="cuda") for o, t in zip(outs_host, dtypes)]
    err_acc = torch.zeros(1, dtype=torch.int64, device="cuda")
    comp = torch.cuda.current_stream()
    sptr = _lib.stream_ptr()
    copy = torch.cuda.Stream()
    prep_s = torch.cuda.Stream()  # host->device prep: its own stream (the other copy direction)
    # Per index range, on the prep stream ahead of the range's kernels: cent /
    # ipt / m2 start from the caller's values (the reference leaves them
    # untouched for capacity-overflowed cells, _kernels.py:1393-1399) and the
    # fixed-stride slots past fcount start zero (the reference leaves them
    # untouched; callers allocate zeros) -- off the critical path.
    src = [torch.from_numpy(np.ascontiguousarray(outs_host[k], np.float64)) for k in (3, 4, 5)]
    prep = []
    prep_s.wait_stream(comp)
    with torch.cuda.stream(prep_s):
        for k in range(K):
            i0, i1 = int(bnd[k]), int(bnd[k + 1])
            for j, sk in zip((3, 4, 5), src):
                outs[j][i0:i1].copy_(sk[i0:i1].view(outs[j][i0:i1].shape), non_blocking=True)
            for j in range(7, len(outs)):
                outs[j][i0:i1].zero_()
            e = torch.cuda.Event()
            e.record(prep_s)
            prep.append(e)
    _lib.check(L.pf_grid_build(c, n, _lib.ptr(p), _lib.ptr(w), 0.0, sptr), "pf_grid_build")
    order = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(L.pf_grid_order(c, _lib.ptr(order), sptr), "pf_grid_order")
    hosts = [torch.from_numpy(h.reshape(h.shape)) if isinstance(h, np.ndarray) and h.flags.c_contiguous
             and h.flags.writeable else None for h in outs_host]
    if K > 1:
        # cells of each index range in bucket order: one stable sort by range id
        rid = torch.bucketize(order.long(), torch.as_tensor(bnd[1:-1], device="cuda"), right=True)
        cells_all = order[torch.sort(rid, stable=True).indices]
        offs = [0] + torch.cumsum(torch.bincount(rid, minlength=K), 0).tolist()
    for k in range(K):
        i0, i1 = int(bnd[k]), int(bnd[k + 1])
        cells = cells_all[offs[k]:offs[k + 1]] if K > 1 else None
        comp.wait_event(prep[k])
        _lib.check(L.pf_batch_evaluate_async(
            c, n, _lib.ptr(p), _lib.ptr(w), float(tol), float(dpsi_max), int(bool(ball_aware)),
            int(bool(want_m2)), int(smf), *[_lib.ptr(o) for o in outs], _lib.ptr(cells),
            0 if cells is None else int(cells.numel()), None, _lib.ptr(err_acc), 0, sptr),
            "pf_batch_evaluate_async")
        ev = torch.cuda.Event()
        ev.record(comp)
        with torch.cuda.stream(copy):
            copy.wait_event(ev)
            for h, t, d in zip(outs_host, hosts, outs):
                if t is not None:
                    t[i0:i1].copy_(d[i0:i1].view(t[i0:i1].shape), non_blocking=True)
    copy.synchronize()
    prep_s.synchronize()
    comp.synchronize()
    for h, t, d in zip(outs_host, hosts, outs):
        if t is None:
            h[...] = d.cpu().numpy().reshape(h.shape)
    return int(err_acc.item())


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
                                       _lib.stream_ptr()), "pf_knn")
    vals = res[0, :got]
    if _is_torch(out_idx):
        out_idx[:got] = vals
    else:
        out_idx[:got] = vals.cpu().numpy()
    return int(got)
