"""Evaluation of restricted Laguerre cells (power cell ∩ ball) on the B200.

This is the torch-level face of ``pf_batch_evaluate`` / ``pf_evaluate_lean``
(the SPEC's ``restricted_cell.evaluate_cell`` over all sites, SPEC.md:231;
reference kernel _kernels.py:1362-1478).  Inputs and outputs are CUDA tensors.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .geom import ConvexCell
from .laguerre import domain_pack, upload_domain


@dataclass
class RestrictedDiagram:
    status: "torch.Tensor"   # int64 [n]  0 EMPTY / 1 FULLBALL / 2 CLIPPED
    vol: "torch.Tensor"      # f64 [n]   |V_i|
    ksur: "torch.Tensor"     # f64 [n]   |K_i| free-surface area
    cent: "torch.Tensor"     # f64 [n,3]
    ipt: "torch.Tensor"      # f64 [n,3] interior point used for the projection
    m2: "torch.Tensor"       # f64 [n]
    fcount: "torch.Tensor"   # int64 [n]
    ftag: "torch.Tensor"     # int64 [n,smf] neighbour j >= 0 or domain face -(k+1)
    farea: "torch.Tensor"    # f64 [n,smf] |B_ij|
    fh: "torch.Tensor"       # f64 [n,smf] signed height h_ij
    fnrm: "torch.Tensor"     # f64 [n,smf,3]
    fcent: "torch.Tensor"    # f64 [n,smf,3]
    flags: int


def alloc(n: int, smf: int):
    import torch

    f8, i8 = dict(dtype=torch.float64, device="cuda"), dict(dtype=torch.int64, device="cuda")
    return [torch.zeros(n, **i8), torch.zeros(n, **f8), torch.zeros(n, **f8),
            torch.zeros((n, 3), **f8), torch.zeros((n, 3), **f8), torch.zeros(n, **f8),
            torch.zeros(n, **i8), torch.zeros((n, smf), **i8), torch.zeros((n, smf), **f8),
            torch.zeros((n, smf), **f8), torch.zeros((n, smf, 3), **f8),
            torch.zeros((n, smf, 3), **f8)]


def evaluate(pts, psi, domain: ConvexCell, ball_aware: bool = True, want_m2: bool = True,
             smf: int = 32, dpsi_max: float | None = None, out=None,
             parity_mode: bool | None = None) -> RestrictedDiagram:
    """Build + evaluate every restricted cell.  ``pts`` [n,3], ``psi`` [n] CUDA f64 tensors.
    ``parity_mode`` (None = the context's setting): restrict exactly as the
    reference does (True) or with the robust correction (False), DESIGN.md §5.1."""
    with _lib.parity(parity_mode):
        return _evaluate(pts, psi, domain, ball_aware, want_m2, smf, dpsi_max, out)


def _evaluate(pts, psi, domain, ball_aware, want_m2, smf, dpsi_max, out):
    import torch

    pts = torch.as_tensor(pts, dtype=torch.float64, device="cuda").contiguous()
    psi = torch.as_tensor(psi, dtype=torch.float64, device="cuda").contiguous()
    n = pts.shape[0]
    dpk = domain_pack(domain)
    c = _lib.ctx()
    upload_domain(c, *dpk.args(), dpk.tol)
    o = alloc(n, smf) if out is None else out
    err = int(_lib.lib().pf_batch_evaluate(
        c, n, _lib.ptr(pts), _lib.ptr(psi), float(dpk.tol),
        -1.0 if dpsi_max is None else float(dpsi_max), int(ball_aware), int(want_m2), int(smf),
        *[_lib.ptr(t) for t in o], 1, _lib.stream_ptr()))
    _lib.check(err, "pf_batch_evaluate")
    return RestrictedDiagram(*o, flags=err)


@dataclass
class FacetCSR:
    row_ptr: "torch.Tensor"  # int64 [n+1]
    tag: "torch.Tensor"      # int64 [nnz] neighbour j >= 0 or domain face -(k+1)
    area: "torch.Tensor"     # f64 [nnz]
    h: "torch.Tensor"        # f64 [nnz]
    nrm: "torch.Tensor"      # f64 [nnz,3]
    cent: "torch.Tensor"     # f64 [nnz,3]


def facets_csr(d: RestrictedDiagram) -> FacetCSR:
    """Compact per-facet CSR of an evaluation's fixed-stride facet arrays
    (pf_facets_csr): row i holds the min(fcount[i], smf) facets of
    cell i in the fixed-stride order."""
    import ctypes as C

    import torch

    L = _lib.lib()
    n, smf = d.ftag.shape
    nnz = C.c_int64(0)
    args = [_lib.ctx(), n, smf] + [_lib.ptr(t) for t in (d.fcount, d.ftag, d.farea, d.fh, d.fnrm, d.fcent)]
    # size query (cap 0 fails when there are facets: read nnz from it)
    L.pf_facets_csr(*args, 0, C.byref(nnz), *([None] * 6), _lib.stream_ptr())
    m = int(nnz.value)
    f8, i8 = dict(dtype=torch.float64, device="cuda"), dict(dtype=torch.int64, device="cuda")
    out = FacetCSR(torch.empty(n + 1, **i8), torch.empty(m, **i8), torch.empty(m, **f8), torch.empty(m, **f8),
                   torch.empty((m, 3), **f8), torch.empty((m, 3), **f8))
    _lib.check(L.pf_facets_csr(*args, m, C.byref(nnz), _lib.ptr(out.row_ptr), _lib.ptr(out.tag),
                               _lib.ptr(out.area), _lib.ptr(out.h), _lib.ptr(out.nrm), _lib.ptr(out.cent),
                               _lib.stream_ptr()), "pf_facets_csr")
    return out


def census(n: int):
    """Per-cell processed-candidate counts of the last evaluation (int32 [n])."""
    import torch

    t = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().pf_last_census(_lib.ctx(), _lib.ptr(t), _lib.stream_ptr()), "pf_last_census")
    return t


def retry_count() -> int:
    import ctypes as C

    v = C.c_int64(0)
    _lib.check(_lib.lib().pf_last_retry_count(_lib.ctx(), C.byref(v)), "pf_last_retry_count")
    return int(v.value)
