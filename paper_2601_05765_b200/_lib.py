"""Loader of the in-tree sm_100a library (libpotflow_b200.so) and its C ABI.

There is no CPU fallback: if the library or a B200 is missing, every entry
point raises.  Signatures follow include/potflow_b200.h.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# PF_LIB_PATH: load a variant build (development experiments only)
LIB_PATH = os.environ.get("PF_LIB_PATH") or os.path.join(_HERE, "libpotflow_b200.so")

_lib = None
_lock = threading.Lock()
_ctx: dict[int, C.c_void_p] = {}


class PotflowCudaError(RuntimeError):
    """Raised when the CUDA library is missing or a device call fails."""


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise PotflowCudaError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        d, i, i64, vp = C.c_double, C.c_int, C.c_int64, C.c_void_p
        L.pf_version.restype = C.c_char_p
        L.pf_last_error.restype = C.c_char_p
        L.pf_launch_count.restype = C.c_ulonglong
        L.pf_fp64_peak.argtypes = [vp, vp]
        L.pf_fp64_peak.restype = i
        L.pf_ctx_create.argtypes = [C.POINTER(vp), i]
        L.pf_ctx_destroy.argtypes = [vp]
        L.pf_set_domain.argtypes = [vp, vp, vp, vp, vp, vp, vp, d]
        L.pf_grid_build.argtypes = [vp, i64, vp, vp, d, vp]
        L.pf_grid_build_dims.argtypes = [vp, i64, vp, vp, vp]
        L.pf_grid_info.argtypes = [vp, vp, vp, vp]
        L.pf_grid_export.argtypes = [vp, vp, vp, vp]
        L.pf_dpsi_max.argtypes = [vp, i64, vp, vp, vp]
        L.pf_batch_evaluate.restype = i64
        L.pf_batch_evaluate.argtypes = [vp, i64, vp, vp, d, d, i, i, i64] + [vp] * 12 + [i, vp]
        L.pf_batch_evaluate_ex.restype = i64
        L.pf_batch_evaluate_ex.argtypes = ([vp, i64, vp, vp, d, d, i, i, i64] + [vp] * 12
                                           + [vp, i64, vp, vp, i, vp])
        L.pf_last_cells_ms.argtypes = [vp, vp]
        L.pf_last_cells_ms.restype = i
        L.pf_evaluate_lean.argtypes = [vp, i64, vp, vp, i, i64] + [vp] * 7 + [vp]
        L.pf_last_census.argtypes = [vp, vp, vp]
        L.pf_last_retry_count.argtypes = [vp, vp]
        L.pf_batch_evaluate_async.restype = i
        L.pf_batch_evaluate_async.argtypes = ([vp, i64, vp, vp, d, d, i, i, i64] + [vp] * 12
                                              + [vp, i64, vp, vp, i, vp])
        L.pf_batch_evaluate_host.restype = i64
        L.pf_batch_evaluate_host.argtypes = ([vp, i64, vp, vp, d, d, i, i, i64] + [vp] * 12 + [i, vp, vp])
        L.pf_batch_build.restype = i64
        L.pf_batch_build.argtypes = [vp, i64, vp, vp, d, d, i, i64, i64, i64] + [vp] * 9 + [i, vp]
        L.pf_stage_timing.argtypes = [vp, i]
        L.pf_stage_times.argtypes = [vp, vp, vp, vp]
        L.pf_stage_timing.restype = i
        L.pf_stage_times.restype = i
        L.pf_grid_order.restype = i
        L.pf_grid_order.argtypes = [vp, vp, vp]
        L.pf_facets_csr.restype = i
        L.pf_facets_csr.argtypes = [vp, i64, i64] + [vp] * 6 + [i64] + [vp] * 7 + [vp]
        L.pf_knn.restype = i64
        L.pf_knn.argtypes = [vp, i64, vp, i64, vp, i64, vp, i, vp]
        L.pf_set_parity_mode.argtypes = [vp, i]
        L.pf_get_parity_mode.argtypes = [vp]
        for name in ("pf_ctx_create", "pf_ctx_destroy", "pf_set_domain", "pf_grid_build",
                     "pf_grid_build_dims", "pf_grid_info", "pf_grid_export", "pf_dpsi_max", "pf_evaluate_lean",
                     "pf_last_census", "pf_last_retry_count", "pf_set_parity_mode", "pf_get_parity_mode"):
            getattr(L, name).restype = i
        _lib = L
    return _lib


def check(rc: int, what: str) -> int:
    if rc < 0:
        msg = lib().pf_last_error().decode(errors="replace")
        raise PotflowCudaError(f"{what} failed: {msg}")
    return rc


def ctx(device: int | None = None):
    """Per-process, per-device library context."""
    import torch

    if not torch.cuda.is_available():
        raise PotflowCudaError("no CUDA device visible: the B200 path has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    c = _ctx.get(dev)
    if c is None:
        h = C.c_void_p()
        with torch.cuda.device(dev):
            check(lib().pf_ctx_create(C.byref(h), dev), "pf_ctx_create")
        _ctx[dev] = h
        c = h
    return c


def set_parity_mode(on: bool, device: int | None = None) -> None:
    """Parity mode of this device's context: every evaluation restricts the
    facets exactly as the reference does (_kernels.py:411-675), including its
    spurious-entry / wrapped-arc outcomes.  Default off."""
    check(lib().pf_set_parity_mode(ctx(device), int(bool(on))), "pf_set_parity_mode")


def parity_mode(device: int | None = None) -> bool:
    return bool(lib().pf_get_parity_mode(ctx(device)))


class parity(object):
    """Context manager: ``with _lib.parity(True): ...`` (restores the previous mode)."""

    def __init__(self, on):
        self.on = on

    def __enter__(self):
        self.prev = None
        if self.on is not None:
            self.prev = parity_mode()
            set_parity_mode(self.on)
        return self

    def __exit__(self, *a):
        if self.prev is not None:
            set_parity_mode(self.prev)


def stream_ptr(stream=None) -> int:
    import torch

    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes through)."""
    if t is None:
        return None
    return int(t.data_ptr())
