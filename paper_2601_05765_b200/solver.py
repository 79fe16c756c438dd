"""Damped Newton (KMT) solve of the semi-discrete partial OT problem on the B200.

The reference ships this component as specification only (SPEC.md:267-336,
PAPER.md:116-135 Algorithm 1, Eq. 2 at PAPER.md:191-196).  The whole loop runs
in libpotflow_b200.so (pf_newton_solve): lean cell evaluations, ELL Hessian
assembly, deterministic Jacobi-PCG, KMT damping on the minimum cell volume.
Host synchronisation: one scalar read per Newton iteration / damping trial and
one per batch of 8 CG iterations.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geom import ConvexCell
from .laguerre import domain_pack, upload_domain

STATUS = {0: "converged", 1: "max_newton", 2: "DampingStall", 3: "InitFailure"}


class NewtonStats(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("evaluations", C.c_int),
                ("cg_iterations", C.c_int), ("damping_halvings", C.c_int),
                ("init_doublings", C.c_int), ("worst_initial", C.c_double),
                ("worst_final", C.c_double), ("last_alpha", C.c_double), ("flags", C.c_int64)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["status_name"] = STATUS.get(self.status, "?")
        return d


@dataclass
class PotState:
    psi: "torch.Tensor"
    stats: dict
    smf: int


def _bind():
    L = _lib.lib()
    if not getattr(L, "_newton_bound", False):
        vp, i, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
        L.pf_newton_solve.argtypes = [vp, i64, vp, vp, vp, i, d, i, i, d, i, C.POINTER(NewtonStats), vp]
        L.pf_newton_solve.restype = i
        L.pf_newton_last_state.argtypes = [vp, vp, vp, vp, vp, i64, i, vp]
        L.pf_newton_last_state_ex.argtypes = [vp, vp, vp, vp, vp, vp, i64, i, vp]
        L.pf_newton_last_state_ex.restype = i
        L.pf_newton_last_state.restype = i
        L.pf_newton_hessian.argtypes = [i64, i, vp, vp, vp, vp, vp, vp, d, vp, vp, vp, vp, vp]
        L.pf_newton_hessian.restype = i
        L.pf_pcg.argtypes = [i64, i, vp, vp, vp, vp, vp, vp, d, i, vp]
        L.pf_pcg.restype = i
        L.pf_newton_gradient.argtypes = [i64, vp, vp, vp, vp, vp]
        L.pf_newton_gradient.restype = i
        L._newton_bound = True
    return L


def newton_solve(pts, nu, domain: ConvexCell, psi_init=None, eps_vol: float = 0.01,
                 max_newton: int = 100, smf: int = 32, ball_aware: bool = True) -> PotState:
    """Solve for psi such that every restricted cell has volume nu_i within eps_vol.

    ``psi_init=None`` -> cold start kappa (3 nu / 4 pi)^(2/3) with kappa doubling
    (SPEC.md:311-315); otherwise a warm start from the given weights.
    """
    import torch

    L = _bind()
    pts = torch.as_tensor(pts, dtype=torch.float64, device="cuda").contiguous()
    nu = torch.as_tensor(nu, dtype=torch.float64, device="cuda").contiguous()
    n = pts.shape[0]
    if psi_init is None:
        psi = torch.zeros(n, dtype=torch.float64, device="cuda")
        cold = 1
    else:
        psi = torch.as_tensor(psi_init, dtype=torch.float64, device="cuda").clone().contiguous()
        cold = 0
    dpk = domain_pack(domain)
    c = _lib.ctx()
    upload_domain(c, *dpk.args(), dpk.tol)
    tau = 1e-12 * domain.diagonal() ** 2
    st = NewtonStats()
    _lib.check(L.pf_newton_solve(c, n, _lib.ptr(pts), _lib.ptr(nu), _lib.ptr(psi), cold,
                                 float(eps_vol), int(max_newton), int(smf), float(tau),
                                 int(ball_aware), C.byref(st), _lib.stream_ptr()),
               "pf_newton_solve")
    return PotState(psi=psi, stats=st.as_dict(), smf=smf)


def last_state(n: int, smf: int):
    """(vol, ksur, fcount, ftag, farea) of the last solve's final evaluation."""
    import torch

    L = _bind()
    vol = torch.empty(n, dtype=torch.float64, device="cuda")
    ksur = torch.empty_like(vol)
    fcount = torch.empty(n, dtype=torch.int32, device="cuda")
    ftag = torch.empty((n, smf), dtype=torch.int32, device="cuda")
    farea = torch.empty((n, smf), dtype=torch.float64, device="cuda")
    _lib.check(L.pf_newton_last_state(_lib.ptr(vol), _lib.ptr(ksur), _lib.ptr(fcount), _lib.ptr(ftag),
                                      _lib.ptr(farea), n, smf, _lib.stream_ptr()), "pf_newton_last_state")
    return vol, ksur, fcount, ftag, farea
