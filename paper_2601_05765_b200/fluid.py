"""Free-surface fluid step: advection + partial-OT projection + barycentric spring.

The reference ships this component as specification only (SPEC.md:338-404,
PAPER.md:332-334 and 374-381); this is its in-scope part:

    x <- x + dt v, reflected into the domain box by tau_geom
    psi <- newton_solve(x, nu, warm psi)
    F_p = (c_i - x_i) / eps^2,  F_g = m g,  v <- v + dt/m (F_p + F_g)

Viscosity and surface tension are out of scope.
All state stays in device tensors; the per-particle updates are CUDA kernels
in libpotflow_b200.so (pf_fluid_advect / pf_fluid_forces).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib, solver
from .geom import ConvexCell


class OtNonConvergence(RuntimeError):
    """The step's Newton solve did not converge (SPEC.md fluid_sim.step errors):
    the simulation halts with the flagged state attached."""

    def __init__(self, diag: dict, state: "FluidState"):
        super().__init__(f"step {diag['step']}: Newton {diag['status_name']}")
        self.diag = diag
        self.state = state


@dataclass
class FluidState:
    x: "torch.Tensor"       # [n,3] positions (sites)
    v: "torch.Tensor"       # [n,3] velocities
    nu: "torch.Tensor"      # [n] prescribed volumes
    rho: "torch.Tensor"     # [n] mass densities
    psi: "torch.Tensor | None" = None  # carried Laguerre weights (warm start)
    step_index: int = 0
    time: float = 0.0
    history: list = field(default_factory=list)


@dataclass
class SimParams:
    dt: float = 1e-3
    eps: float = 5e-3
    gravity: tuple = (0.0, 0.0, -9.81)
    tau_geom: float | None = None  # default: 1e-9 x domain diagonal
    eps_vol: float = 0.01
    max_newton: int = 100
    smf: int = 32
    best_effort: bool = False  # continue past a non-converged solve (SPEC.md --best-effort)


def _bind():
    L = solver._bind()
    if not getattr(L, "_fluid_bound", False):
        vp, i64, d = C.c_void_p, C.c_int64, C.c_double
        L.pf_fluid_advect.argtypes = [i64, vp, vp, d, vp, vp, d, vp]
        L.pf_fluid_advect.restype = C.c_int
        L.pf_fluid_forces.argtypes = [i64, vp, vp, vp, vp, vp, d, d, vp, vp]
        L.pf_fluid_forces.restype = C.c_int
        L._fluid_bound = True
    return L


def make_state(pts, vel, nu, rho) -> FluidState:
    import torch

    def t(a):
        return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")

    return FluidState(t(pts), t(vel), t(nu), t(rho))


def step(state: FluidState, params: SimParams, domain: ConvexCell) -> dict:
    """One time step; returns diagnostics (Newton stats, volume error)."""
    import torch

    L = _bind()
    n = state.x.shape[0]
    lo, hi = domain.bbox()
    tau = params.tau_geom if params.tau_geom is not None else 1e-9 * domain.diagonal()
    lo_a = (C.c_double * 3)(*[float(v) for v in lo])
    hi_a = (C.c_double * 3)(*[float(v) for v in hi])
    s = _lib.stream_ptr()
    # (1)-(2) advect and reflect
    _lib.check(L.pf_fluid_advect(n, _lib.ptr(state.x), _lib.ptr(state.v), float(params.dt), lo_a, hi_a,
                                 float(tau), s), "pf_fluid_advect")
    # (3) partial-OT projection with the carried weights
    res = solver.newton_solve(state.x, state.nu, domain, psi_init=state.psi, eps_vol=params.eps_vol,
                              max_newton=params.max_newton, smf=params.smf)
    state.psi = res.psi
    # (4) centroids of the final evaluation
    cent = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    _lib.check(L.pf_newton_last_state_ex(None, None, None, None, None, _lib.ptr(cent), n, params.smf, s),
               "pf_newton_last_state_ex")
    # (5)-(7) spring pressure + gravity, velocity update
    g = (C.c_double * 3)(*[float(v) for v in params.gravity])
    _lib.check(L.pf_fluid_forces(n, _lib.ptr(state.x), _lib.ptr(cent), _lib.ptr(state.nu),
                                 _lib.ptr(state.rho), _lib.ptr(state.v), float(params.dt),
                                 float(params.eps), g, s), "pf_fluid_forces")
    state.step_index += 1
    state.time += params.dt
    diag = {"step": state.step_index, **{k: res.stats[k] for k in
            ("status_name", "iterations", "evaluations", "cg_iterations", "damping_halvings",
                 "worst_final")}}
    state.history.append(diag)
    if res.stats["status"] != 0 and not params.best_effort:
        raise OtNonConvergence(diag, state)
    return diag
