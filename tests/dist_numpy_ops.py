"""TEST INFRASTRUCTURE ONLY: a numpy stand-in for dist_solver.CudaOps, so the
partitioned Newton orchestration (halo exchange, all-reduces, re-partition,
PCG recurrences) can run over gloo on CPU.  Cells are evaluated by the CPU
oracle; never imported by the product package."""
from __future__ import annotations

import numpy as np
import torch

from oracle import pyoracle as O


class NumpyOps:
    def __init__(self, pts_local, nu_local, rows, dom_args, tol, smf, tau):
        self.torch = torch
        self.pts = np.ascontiguousarray(pts_local, np.float64)
        self.nu = np.ascontiguousarray(nu_local, np.float64)
        self.rows = np.asarray(rows, np.int64)
        self.n = len(self.pts)
        self.dom_args, self.tol, self.smf, self.tau = dom_args, tol, smf, tau
        self.grid = O.SpatialGrid(self.pts, [0, 0, 0], [1, 1, 1], 1.0)
        n = self.n
        self.psi = np.zeros(n)
        self.psi_t = np.zeros(n)
        self.slots = [None, None]
        # vectors are torch CPU tensors sharing numpy storage (halo exchange works in place)
        self.v = {k: torch.zeros(n, dtype=torch.float64) for k in ("g", "x", "r", "z", "p", "Ap", "diag", "s")}
        self.sc = [0.0, 0.0, 0.0]
        self.cols = self.vals = None

    def _n(self, k):
        return self.v[k].numpy()

    # weights
    def set_psi(self, psi_local):
        self.psi[:] = psi_local

    def cold_psi(self, kappa):
        self.psi[:] = kappa * (3.0 * self.nu / (4.0 * np.pi)) ** (2.0 / 3.0)

    def vec_psi(self):
        return torch.from_numpy(self.psi)

    def rescue_nearest(self):
        from scipy.spatial import cKDTree

        o = self.slots[0]
        r = self.rows
        e = r[~(o["vol"][r] > 0.0)]
        if len(e) == 0:
            return
        _, nn = cKDTree(self.pts).query(self.pts[e], k=2)
        j = np.where(nn[:, 0] == e, nn[:, 1], nn[:, 0])
        self.psi[e] = np.maximum(self.psi[e], self.psi[j])

    def rescue(self, kappa):
        o = self.slots[0]
        r = self.rows
        e = ~(o["vol"][r] > 0.0)
        rr = r[e]
        self.psi[rr] = np.maximum(self.psi[rr], kappa * (3.0 * self.nu[rr] / (4.0 * np.pi)) ** (2.0 / 3.0))

    def psi_host(self, trial=False):
        return (self.psi_t if trial else self.psi).copy()

    def search_radius_max(self, dpsi, trial=False):
        ps = np.maximum((self.psi_t if trial else self.psi)[self.rows], 0.0)
        return float((np.sqrt(ps) + np.sqrt(ps + dpsi)).max()) if len(ps) else 0.0

    def psi_minmax(self, trial=False):
        ps = (self.psi_t if trial else self.psi)[self.rows]
        return torch.tensor([-ps.min(), ps.max()], dtype=torch.float64)

    def trial(self, alpha):
        self.psi_t[:] = self.psi + alpha * self._n("x")

    def accept(self):
        self.psi[:] = self.psi_t
        self.slots.reverse()

    # evaluation / Newton pieces
    def evaluate(self, dpsi, trial=False):
        ps = self.psi_t if trial else self.psi
        o = O.evaluate(self.pts, ps, self.dom_args, self.tol, self.grid, want_m2=False, smf=self.smf,
                       dpsi=dpsi, i0=0, i1=len(self.rows), cells=self.rows)
        self.slots[1 if trial else 0] = o

    def grad_stats(self, trial=False):
        o = self.slots[1 if trial else 0]
        r = self.rows
        v, nu = o["vol"][r], self.nu[r]
        self._n("g")[r] = nu - v
        return torch.tensor([np.max(np.abs(v - nu) / nu), -v.min(), -nu.min()], dtype=torch.float64)

    def hessian(self):
        from oracle.newton_ref import hessian_ell

        o = self.slots[0]
        cols, vals, diag = hessian_ell(self.pts, self.psi, o, self.tau, self.smf)
        self.cols, self.vals = cols, vals
        self._n("diag")[:] = diag

    def cg_init(self):
        r = self.rows
        b, d = self._n("g")[r], self._n("diag")[r]
        z = b / d
        self._n("x")[:] = 0.0
        self._n("r")[r] = b
        self._n("z")[r] = z
        self._n("p")[r] = z
        return torch.tensor([float(b @ z), float(b @ b)], dtype=torch.float64)

    def cg_spmv(self):
        r = self.rows
        p = self._n("p")
        c, v = self.cols[r], self.vals[r]
        ps = np.where(c >= 0, p[np.maximum(c, 0)], 0.0)
        Ap = self._n("diag")[r] * p[r] + (v * ps).sum(1)
        self._n("Ap")[r] = Ap
        return torch.tensor([float(p[r] @ Ap)], dtype=torch.float64)

    def cg_update(self, rz, pAp):
        r = self.rows
        alpha = float(rz[0]) / float(pAp[0]) if float(pAp[0]) != 0.0 else 0.0
        x, rr_, z = self._n("x"), self._n("r"), self._n("z")
        x[r] += alpha * self._n("p")[r]
        rr_[r] -= alpha * self._n("Ap")[r]
        z[r] = rr_[r] / self._n("diag")[r]
        return torch.tensor([float(rr_[r] @ z[r]), float(rr_[r] @ rr_[r])], dtype=torch.float64)

    def cg_pdir(self, rz_new, rz_old):
        r = self.rows
        beta = float(rz_new[0]) / float(rz_old[0]) if float(rz_old[0]) != 0.0 else 0.0
        p = self._n("p")
        p[r] = self._n("z")[r] + beta * p[r]

    def cg1_init(self):
        r = self.rows
        b, d = self._n("g")[r], self._n("diag")[r]
        self._n("x")[:] = 0.0
        self._n("r")[r] = b
        self._n("z")[r] = b / d
        self._n("p")[r] = 0.0
        self._n("s")[r] = 0.0

    def cg1_spmv_dots(self):
        r = self.rows
        u = self._n("z")
        c, v = self.cols[r], self.vals[r]
        us = np.where(c >= 0, u[np.maximum(c, 0)], 0.0)
        w = self._n("diag")[r] * u[r] + (v * us).sum(1)
        self._n("Ap")[r] = w
        rr = self._n("r")[r]
        return torch.tensor([float(rr @ u[r]), float(w @ u[r]), float(rr @ rr)], dtype=torch.float64)

    def cg1_step(self, red, first):
        g, dl = float(red[0]), float(red[1])
        if first:
            beta, alpha = 0.0, (g / dl if dl != 0.0 else 0.0)
        else:
            beta = g / self.sc[0] if self.sc[0] != 0.0 else 0.0
            den = dl - (beta * g / self.sc[1] if self.sc[1] != 0.0 else 0.0)
            alpha = g / den if den != 0.0 else 0.0
        self.sc = [g, alpha, beta]
        r = self.rows
        p, s = self._n("p"), self._n("s")
        p[r] = self._n("z")[r] + beta * p[r]
        s[r] = self._n("Ap")[r] + beta * s[r]
        self._n("x")[r] += alpha * p[r]
        self._n("r")[r] -= alpha * s[r]
        self._n("z")[r] = self._n("r")[r] / self._n("diag")[r]

    # device-side convergence variant (dist_solver.CudaOps.cg1_step_conv)
    def cg1_conv_reset(self):
        self.conv = [0.0, 0]  # done, iterations
        self.bb = 0.0

    def cg1_spmv_dots_c(self):
        if self.conv[0]:
            return torch.zeros(3, dtype=torch.float64)
        return self.cg1_spmv_dots()

    def cg1_step_conv(self, red, rtol, max_iter):
        if self.conv[0]:
            return
        it, rr = self.conv[1], float(red[2])
        if it == 0:
            self.bb = rr
            if not rr > 0.0:
                self.conv[0] = 1.0
                return
        elif np.sqrt(rr) <= rtol * np.sqrt(self.bb) or it >= max_iter or not np.isfinite(rr):
            self.conv[0] = 1.0
            return
        self.cg1_step(red, it == 0)
        self.conv[1] = it + 1

    def cg1_status(self):
        return bool(self.conv[0]), int(self.conv[1])

    def vec(self, name):
        return self.v[name]

    def index(self, ix):
        return torch.as_tensor(np.asarray(ix, np.int64))

    def tensor(self, vals):
        return torch.tensor(vals, dtype=torch.float64)

    def owned(self, name):
        src = self.psi if name == "psi" else self._n(name)
        return src[self.rows].copy()


def _result(self):
    o = self.slots[0]
    r = self.rows
    return {"vol": torch.as_tensor(o["vol"][r]), "cent": torch.as_tensor(np.ascontiguousarray(o["cent"][r]))}


NumpyOps.result = _result


class NumpyParticleOps:
    """numpy restatement of pf_fluid_advect / pf_fluid_forces (csrc/pf_newton.cu
    k_advect, k_forces) on CPU tensors, for the distributed fluid step tests."""

    def advect(self, x, v, dt, lo, hi, tau):
        X, V = x.numpy(), v.numpy()
        lo_ = np.asarray(lo, np.float64) + tau
        hi_ = np.asarray(hi, np.float64) - tau
        p = X + dt * V
        below, above = p < lo_, p > hi_
        p = np.where(below, lo_ + (lo_ - p), p)
        V[below] = -V[below]
        above = p > hi_
        p = np.where(above, hi_ - (p - hi_), p)
        V[above] = -V[above]
        X[:] = np.minimum(np.maximum(p, lo_), hi_)

    def forces(self, x, cent, nu, rho, v, dt, eps, g, spring):
        m = (rho * nu).numpy()[:, None]
        ks = (m if spring == 0 else np.ones_like(m)) * (1.0 / (eps * eps))
        f = ks * (cent.numpy() - x.numpy()) + m * np.asarray(g, np.float64)[None, :]
        v.numpy()[:] += dt * f / m
