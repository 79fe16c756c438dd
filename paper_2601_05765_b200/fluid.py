"""Free-surface fluid step: advection + partial-OT projection + barycentric spring.

The reference ships this component as specification only (SPEC.md:338-404,
PAPER.md:332-334 and 374-381); this is its in-scope part:

    x <- x + dt v, reflected into the domain box by tau_geom
    psi <- newton_solve(x, nu, warm psi)
    F_p = k (c_i - x_i) / eps^2,  F_g = m g,  v <- v + dt/m (F_p + F_g)
    k = m (spring="gallouet_merigot", default: the paper's Gallouet-Merigot
    acceleration) or k = 1 (spring="spec":
    SPEC.md pressure_force as printed)

With viscosity, wall friction or surface tension (the first
"next" row of SURVEY §8(f)) the velocity update is implicit:

    (m/dt I + mu L) v <- m/dt v + F_p + F_g + F_t      (Eq. 4)

L the fluid graph Laplacian with the P1 weights |B_ij| / (2 |p_j - p_i|) of the
step's restricted facets (wall facets: zero wall velocity), F_t = gamma times the
graph Laplacian of the positions with wall ghosts; three Jacobi-PCG solves
(pf_fluid_forces_implicit).  All state stays in device tensors; the
per-particle updates are CUDA kernels in libpotflow_b200.so.
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


SPRINGS = {"gallouet_merigot": 0, "spec": 1}  # PF_SPRING_GM / PF_SPRING_SPEC


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
    viscosity: float = 0.0            # mu (fluid-fluid)
    boundary_viscosity: float = 0.0   # mu_b (fluid-wall friction, zero wall velocity)
    surface_tension: float = 0.0      # gamma
    boundary_affinity: float = 1.0    # weight of the wall ghosts in the surface-tension Laplacian
    implicit: bool | None = None      # None: implicit iff any of the three above is non-zero
    visc_rtol: float = 1e-10
    spring: str = "gallouet_merigot"  # or "spec": F_p = (c - x)/eps^2 as SPEC.md prints it

    def spring_code(self) -> int:
        if self.spring not in SPRINGS:
            raise ValueError(f"spring must be one of {sorted(SPRINGS)}")
        return SPRINGS[self.spring]


def _bind():
    L = solver._bind()
    if not getattr(L, "_fluid_bound", False):
        vp, i64, d, i = C.c_void_p, C.c_int64, C.c_double, C.c_int
        L.pf_fluid_forces_implicit.argtypes = ([i64, i] + [vp] * 9 + [d, d, vp, d, d, d, d, vp, i, i]
                                               + [vp] * 6 + [d, vp])
        L.pf_fluid_forces_implicit.restype = C.c_int
        L.pf_fluid_advect.argtypes = [i64, vp, vp, d, vp, vp, d, vp]
        L.pf_fluid_advect.restype = C.c_int
        L.pf_fluid_forces.argtypes = [i64, vp, vp, vp, vp, vp, d, d, vp, i, vp]
        L.pf_fluid_forces.restype = C.c_int
        L.pf_pressure_force.argtypes = [i64, vp, vp, vp, vp, d, i, vp, vp]
        L.pf_pressure_force.restype = C.c_int
        L._fluid_bound = True
    return L


def pressure_force(x, cent, nu, rho, eps: float, spring: str = "gallouet_merigot"):
    """F_p = k (c - x) / eps^2 per particle (SPEC.md pressure_force), [n,3] CUDA f64."""
    import torch

    L = _bind()
    t = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()  # noqa: E731
    x, cent, nu, rho = t(x), t(cent), t(nu), t(rho)
    F = torch.empty_like(x)
    _lib.check(L.pf_pressure_force(x.shape[0], _lib.ptr(x), _lib.ptr(cent), _lib.ptr(nu), _lib.ptr(rho),
                                   float(eps), SPRINGS[spring], _lib.ptr(F), _lib.stream_ptr()),
               "pf_pressure_force")
    return F


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
    # (5)-(7) spring pressure + gravity (+ surface tension, viscosity), velocity update
    g = (C.c_double * 3)(*[float(v) for v in params.gravity])
    implicit = params.implicit
    if implicit is None:
        implicit = bool(params.viscosity or params.boundary_viscosity or params.surface_tension)
    visc_cg = 0
    if implicit:
        visc_cg = implicit_forces(state, params, domain, cent, g)
    else:
        _lib.check(L.pf_fluid_forces(n, _lib.ptr(state.x), _lib.ptr(cent), _lib.ptr(state.nu),
                                     _lib.ptr(state.rho), _lib.ptr(state.v), float(params.dt),
                                     float(params.eps), g, params.spring_code(), s), "pf_fluid_forces")
    state.step_index += 1
    state.time += params.dt
    diag = {"step": state.step_index, **{k: res.stats[k] for k in
            ("status_name", "iterations", "evaluations", "cg_iterations", "damping_halvings",
                 "worst_final")}}
    diag["viscosity_cg_iterations"] = visc_cg
    state.history.append(diag)
    if res.stats["status"] != 0 and not params.best_effort:
        raise OtNonConvergence(diag, state)
    return diag


def implicit_forces(state: FluidState, params: SimParams, domain: ConvexCell, cent, g) -> int:
    """Implicit velocity update on the step's final evaluation (see module doc)."""
    import torch

    from .laguerre import domain_pack

    L = _bind()
    n, smf = state.x.shape[0], params.smf
    vol, _, fcount, ftag, farea = solver.last_state(n, smf)
    dpk = domain_pack(domain)
    ndom = int(dpk.args()[1][1])
    planes = torch.as_tensor(np.ascontiguousarray(dpk.args()[2][:ndom]), dtype=torch.float64, device="cuda")
    f8, i4 = dict(dtype=torch.float64, device="cuda"), dict(dtype=torch.int32, device="cuda")
    hcnt, hcol = torch.empty(n, **i4), torch.empty((n, smf), **i4)
    hval, diag = torch.empty((n, smf), **f8), torch.empty(n, **f8)
    rhs, sol = torch.empty(3 * n, **f8), torch.empty(n, **f8)
    P = _lib.ptr
    it = L.pf_fluid_forces_implicit(
        n, smf, P(state.x), P(cent), P(vol), P(fcount), P(ftag), P(farea), P(state.nu), P(state.rho),
        P(state.v), float(params.dt), float(params.eps), g, float(params.viscosity),
        float(params.boundary_viscosity), float(params.surface_tension), float(params.boundary_affinity),
        P(planes), ndom, params.spring_code(), P(hcnt), P(hcol), P(hval), P(diag), P(rhs), P(sol), float(params.visc_rtol),
        _lib.stream_ptr())
    return _lib.check(it, "pf_fluid_forces_implicit")
