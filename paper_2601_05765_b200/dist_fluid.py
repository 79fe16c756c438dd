"""Fluid step on the exchange data plane: one process per
GPU, each owning the particles of its x-slab -- nothing is replicated.

Per step (the single-GPU ``fluid.step`` restated over owned particles):

1. advect the owned particles (``pf_fluid_advect``: x += dt v, reflected);
2. migrate: particles that left the slab move to their new owner with their
   velocity, volume, density and carried weight (``halo.SlabComm.migrate``);
3. Newton with the carried weights (``dist_solver.DistNewtonLocal``): the
   ghost layer is exchanged from the owned particles, the CG halo per
   iteration, convergence tested on the device;
4. spring + gravity on the owned particles from their cell centroids
   (``pf_fluid_forces``).

Viscosity / surface tension (the implicit solve of ``fluid.implicit_forces``)
stay single-GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .dist_solver import Comm, DistNewtonLocal
from .fluid import OtNonConvergence, SimParams, _bind
from .halo import SlabComm


class CudaParticleOps:
    """The per-particle kernels of the single-GPU step on owned tensors."""

    def advect(self, x, v, dt, lo, hi, tau):
        L = _bind()
        lo_a = (C.c_double * 3)(*[float(t) for t in lo])
        hi_a = (C.c_double * 3)(*[float(t) for t in hi])
        _lib.check(L.pf_fluid_advect(x.shape[0], _lib.ptr(x), _lib.ptr(v), float(dt), lo_a, hi_a, float(tau),
                                     _lib.stream_ptr()), "pf_fluid_advect")

    def forces(self, x, cent, nu, rho, v, dt, eps, g, spring):
        L = _bind()
        ga = (C.c_double * 3)(*[float(t) for t in g])
        _lib.check(L.pf_fluid_forces(x.shape[0], _lib.ptr(x), _lib.ptr(cent), _lib.ptr(nu), _lib.ptr(rho),
                                     _lib.ptr(v), float(dt), float(eps), ga, int(spring), _lib.stream_ptr()),
                   "pf_fluid_forces")


class DistFluid:
    """Owned particles of this rank (tensors on its device, global-id order)."""

    def __init__(self, gid, x, v, nu, rho, domain, cuts, params: SimParams | None = None, group=None,
                 ops_factory=None, particle_ops=None, slack: float = 1.5):
        import torch

        self.torch = torch
        self.params = params or SimParams()
        self.domain = domain
        self.cuts = np.asarray(cuts, dtype=np.float64)
        self.group = group
        self.comm = Comm(group)
        self.sc = SlabComm(self.cuts, self.comm)
        self.ops_factory = ops_factory
        self.pops = particle_ops or CudaParticleOps()
        self.slack = slack
        f8 = dict(dtype=torch.float64)
        dev = torch.as_tensor(gid).device
        self.gid = torch.as_tensor(gid, dtype=torch.int64, device=dev)
        self.x = torch.as_tensor(x, **f8, device=dev).contiguous().clone()
        self.v = torch.as_tensor(v, **f8, device=dev).contiguous().clone()
        self.nu = torch.as_tensor(nu, **f8, device=dev).contiguous().clone()
        self.rho = torch.as_tensor(rho, **f8, device=dev).contiguous().clone()
        self.psi = None
        self.step_index = 0
        self.history = []

    def step(self) -> dict:
        t = self.torch
        p = self.params
        lo, hi = self.domain.bbox()
        tau = p.tau_geom if p.tau_geom is not None else 1e-9 * self.domain.diagonal()
        # (1) advect
        self.pops.advect(self.x, self.v, p.dt, lo, hi, tau)
        # (2) migrate to the new owners
        fields = {"pts": self.x, "v": self.v, "nu": self.nu, "rho": self.rho}
        if self.psi is not None:
            fields["psi"] = self.psi
        self.gid, f = self.sc.migrate(self.gid, fields)
        self.x, self.v, self.nu, self.rho = f["pts"], f["v"], f["nu"], f["rho"]
        psi_init = f.get("psi")
        # (3) partial-OT projection with the carried weights
        dn = DistNewtonLocal(self.gid, self.x, self.nu, self.domain, self.cuts, group=self.group, smf=p.smf,
                             slack=self.slack, ops_factory=self.ops_factory)
        res = dn.solve(psi_init=psi_init, eps_vol=p.eps_vol, max_newton=p.max_newton)
        self.psi = t.as_tensor(res.psi_owned, dtype=t.float64, device=self.gid.device)
        cent = dn.ops.result()["cent"].to(self.gid.device).contiguous()
        # (4) spring pressure + gravity, velocity update
        self.pops.forces(self.x, cent, self.nu, self.rho, self.v, p.dt, p.eps, p.gravity, p.spring_code())
        self.step_index += 1
        diag = {"step": self.step_index, "n_owned": int(self.gid.numel()),
                **{k: res.stats[k] for k in ("status_name", "iterations", "evaluations", "cg_iterations",
                                             "damping_halvings", "worst_final", "repartitions",
                                             "halo_entries")}}
        self.history.append(diag)
        if res.stats["status"] != 0 and not p.best_effort:
            raise OtNonConvergence(diag, None)
        return diag
