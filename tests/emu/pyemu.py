"""ctypes wrapper of the host warp-emulator build of the cell kernel (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libpfemu.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = C.CDLL(_LIB)
        d, i, vp = C.c_double, C.c_int, C.c_void_p
        L.pfemu_evaluate.restype = C.c_int64
        L.pfemu_evaluate.argtypes = ([i, vp, vp, vp, i, vp, vp, i, vp, vp, i]
                                     + [d] * 6 + [i] * 3 + [d, d, i, i, i, d] + [vp] * 14
                                     + [i, C.c_uint64, vp, vp])
        L.pfemu_ws_bytes.restype = i
        L.pfemu_ws_bytes.argtypes = [i]
        L.pfemu_set_strict.argtypes = [i]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def evaluate(pts, psi, pack, tol, grid_lo, grid_ih, grid_gn, dpsi, ball_aware=True,
             want_m2=True, smf=32, t_init=0.0, tier=0, seed=1, parity_mode=False):
    """pack = (dv, dc, dp, dt, dlp, dlv) in the reference's packed layout."""
    lib().pfemu_set_strict(int(bool(parity_mode)))
    dv, dc, dp, dt, dlp, dlv = pack
    nv, nf, nl = int(dc[0]), int(dc[1]), int(dc[2])
    dv = np.ascontiguousarray(dv[:nv], np.float64)
    dp = np.ascontiguousarray(dp[:nf], np.float64)
    dt = np.ascontiguousarray(dt[:nf], np.int32)
    dlp = np.ascontiguousarray(dlp[:nf + 1], np.int32)
    dlv = np.ascontiguousarray(dlv[:nl], np.int32)
    pts = np.ascontiguousarray(pts, np.float64)
    psi = np.ascontiguousarray(psi, np.float64)
    n = len(pts)
    o = dict(status=np.zeros(n, np.int64), vol=np.zeros(n), ksur=np.zeros(n),
             cent=np.zeros((n, 3)), ipt=np.zeros((n, 3)), m2=np.zeros(n),
             fcount=np.zeros(n, np.int64), ftag=np.zeros((n, smf), np.int64),
             farea=np.zeros((n, smf)), fh=np.zeros((n, smf)), fnrm=np.zeros((n, smf, 3)),
             fcent=np.zeros((n, smf, 3)), flags=np.zeros(n, np.int32), census=np.zeros(n, np.int32))
    nret = np.zeros(1, np.int32)
    ncoll = np.zeros(1, np.int64)
    keys = ("status", "vol", "ksur", "cent", "ipt", "m2", "fcount", "ftag", "farea", "fh",
            "fnrm", "fcent", "flags", "census")
    err = lib().pfemu_evaluate(n, _p(pts), _p(psi), _p(dv), nv, _p(dp), _p(dt), nf, _p(dlp),
                               _p(dlv), nl, *[float(x) for x in grid_lo],
                               *[float(x) for x in grid_ih], *[int(x) for x in grid_gn],
                               float(tol), float(dpsi), int(bool(ball_aware)), int(bool(want_m2)),
                               int(smf), float(t_init), *[_p(o[k]) for k in keys], int(tier),
                               int(seed), _p(nret), _p(ncoll))
    o["err"] = int(err)
    o["n_retry"] = int(nret[0])
    o["n_coll"] = int(ncoll[0])
    return o
