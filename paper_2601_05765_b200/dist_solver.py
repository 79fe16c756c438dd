"""Spatially partitioned damped Newton solve across ranks.

One process per GPU.  Rank r owns the cells of an x-slab and holds as ghosts
every site within the (slack-widened) ball-aware search radius of its cells
(`partition.halo_plan`); its local arrays keep the global index order, so its
cells are bit-identical to the single-GPU ones.  Per Newton iteration
(the algorithm of `pf_newton_solve`):

* evaluation of the owned cells with the all-reduced weight slack dpsi
  (`pf_evaluate_lean_cells`), gradient statistics all-reduced (one MAX of
  three scalars: worst error, -min volume, -min nu);
* Hessian rows of the owned cells (`pf_rows_hessian`), columns may be ghosts;
* Jacobi-PCG in the single-reduction form (Chronopoulos & Gear): per
  iteration one halo exchange of the preconditioned residual (P2P send/recv
  to the slab neighbours) and ONE all-reduce of three scalars (the classic
  two-reduction form is kept as cg="classic");
* one halo exchange of the Newton step x, after which every damping trial
  psi + alpha x is formed locally for owned and ghost sites alike.

The ghost margin is checked before every evaluation (weights grow during a
solve); when a rank's search radius outgrows it, all ranks re-partition from
the all-gathered weights.  The device work goes through `CudaOps` (the C ABI
in pf_dist.cu / pf_runtime.cu); the orchestration is backend-agnostic so the
CPU tests drive it with a numpy stand-in over gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import partition

STATUS = {0: "converged", 1: "max_newton", 2: "DampingStall", 3: "InitFailure"}


# ---------------------------------------------------------------------------
# communication (torch.distributed; NCCL on GPUs, gloo for CPU tests)
# ---------------------------------------------------------------------------
class Comm:
    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if self.on else 0
        self.world = dist.get_world_size(group) if self.on else 1
        self.gloo = self.on and dist.get_backend(group) == "gloo"
        # PF_DIST_FORCE_COLLECTIVES=1: issue the collectives even with one rank
        # (tests: drives the NCCL path on a one-GPU box)
        import os

        self.force = self.on and os.environ.get("PF_DIST_FORCE_COLLECTIVES") == "1"

    def active(self) -> bool:
        """Whether the exchanges and reductions go through torch.distributed."""
        return self.on and (self.world > 1 or self.force)

    def _staged(self, t):
        return t.cpu() if (self.gloo and t.is_cuda) else t

    def all_reduce(self, t, op="sum"):
        """In-place all-reduce of a small tensor (sum or max)."""
        if not self.active():
            return t
        d = self.dist
        s = self._staged(t)
        d.all_reduce(s, op=d.ReduceOp.SUM if op == "sum" else d.ReduceOp.MAX, group=self.group)
        if s is not t:
            t.copy_(s)
        return t

    def exchange(self, vec, plan: partition.HaloPlan, idx_send: dict, idx_recv: dict):
        """Fill the ghost entries of `vec` (local-length) from their owners."""
        if not self.active() or (not plan.send and not plan.recv):
            return vec
        import torch

        d = self.dist
        bufs_s = {q: self._staged(vec.index_select(0, ix)) for q, ix in idx_send.items()}
        bufs_r = {q: torch.empty(len(ix), dtype=vec.dtype,
                                 device="cpu" if self.gloo else vec.device) for q, ix in idx_recv.items()}
        ops = [d.P2POp(d.isend, b, self._peer(q)) for q, b in bufs_s.items()]
        ops += [d.P2POp(d.irecv, b, self._peer(q)) for q, b in bufs_r.items()]
        if ops:
            for r in d.batch_isend_irecv(ops):
                r.wait()
        for q, ix in idx_recv.items():
            vec.index_copy_(0, ix, bufs_r[q].to(vec.device))
        return vec

    def _peer(self, q):
        return self.dist.get_global_rank(self.group, q) if self.group is not None else q

    def all_gather_objects(self, obj):
        if not self.active():
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


# ---------------------------------------------------------------------------
# device backend (the product path)
# ---------------------------------------------------------------------------
def _bind():
    from . import _lib

    L = _lib.lib()
    if not getattr(L, "_dist_bound", False):
        vp, i, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
        L.pf_evaluate_lean_cells.argtypes = [vp, i64, vp, vp, d, i, i64, vp, i64] + [vp] * 7 + [i, vp]
        L.pf_rows_gradient.argtypes = [i, vp, vp, vp, vp, vp, vp]
        L.pf_rows_hessian.argtypes = [i, vp, i, vp, vp, vp, vp, vp, vp, d, vp, vp, vp, vp, vp]
        L.pf_dcg_init.argtypes = [i, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pf_dcg_spmv.argtypes = [i, vp, i, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pf_dcg_update.argtypes = [i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pf_dcg_pdir.argtypes = [i, vp, vp, vp, vp, vp, vp]
        L.pf_daxpy.argtypes = [i64, vp, d, vp, vp, vp]
        L.pf_cg1_init.argtypes = [i, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pf_cg1_spmv_dots.argtypes = [i, vp, i, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pf_cg1_step.argtypes = [i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i, vp]
        L.pf_cg1_spmv_dots_c.argtypes = [i, vp, i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.pf_cg1_step_conv.argtypes = [i, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, d, i, vp]
        for name in ("pf_cg1_init", "pf_cg1_spmv_dots", "pf_cg1_step", "pf_cg1_spmv_dots_c", "pf_cg1_step_conv"):
            getattr(L, name).restype = i
        for name in ("pf_evaluate_lean_cells", "pf_rows_gradient", "pf_rows_hessian", "pf_dcg_init",
                     "pf_dcg_spmv", "pf_dcg_update", "pf_dcg_pdir", "pf_daxpy"):
            getattr(L, name).restype = i
        L._dist_bound = True
    return L


class CudaOps:
    """Per-rank device state of one partition: local sites, owned rows, the
    evaluation buffers (current + trial), Hessian and CG vectors."""

    def __init__(self, pts_local: np.ndarray, nu_local: np.ndarray, rows: np.ndarray, domain,
                 smf: int, ball_aware: bool, tau_psi: float):
        import torch

        from . import _lib
        from .laguerre import domain_pack, upload_domain

        self.torch = torch
        self.L = _bind()
        self._lib = _lib
        dev = dict(device="cuda")
        f8, i4 = dict(dtype=torch.float64, **dev), dict(dtype=torch.int32, **dev)
        self.n = n = len(pts_local)
        self.smf, self.ball_aware, self.tau = smf, int(ball_aware), float(tau_psi)
        # numpy arrays or tensors (the exchange data plane hands over device tensors)
        self.pts = torch.as_tensor(pts_local, **f8).contiguous()
        self.nu = torch.as_tensor(nu_local, **f8).contiguous()
        self.rows = torch.as_tensor(rows, **i4).contiguous()
        self.nrows = len(rows)
        self.psi = torch.zeros(n, **f8)
        self.psi_t = torch.zeros(n, **f8)
        self.slots = [dict(vol=torch.zeros(n, **f8), ksur=torch.zeros(n, **f8),
                           fcount=torch.zeros(n, **i4), ftag=torch.zeros((n, smf), **i4),
                           farea=torch.zeros((n, smf), **f8), cent=torch.zeros((n, 3), **f8))
                      for _ in range(2)]
        self.v = {k: torch.zeros(n, **f8) for k in ("g", "x", "r", "z", "p", "Ap", "diag", "s")}
        self.cg1_sc = torch.zeros(8, **f8)
        self.hcnt = torch.zeros(n, **i4)
        self.hcol = torch.zeros((n, smf), **i4)
        self.hval = torch.zeros((n, smf), **f8)
        self.flags = torch.zeros(1, dtype=torch.int64, **dev)
        self.scal = torch.zeros(16, **f8)
        dpk = domain_pack(domain)
        self.ctx = _lib.ctx()
        upload_domain(self.ctx, *dpk.args(), dpk.tol)
        _lib.check(_lib.lib().pf_grid_build(self.ctx, n, _lib.ptr(self.pts), None, 0.0, self._s()),
                   "pf_grid_build")

    def _s(self):
        return self._lib.stream_ptr()

    def p(self, t):
        return self._lib.ptr(t)

    def chk(self, rc, what):
        self._lib.check(rc, what)

    # --- weights ---------------------------------------------------------
    def set_psi(self, psi_local: np.ndarray):
        self.psi.copy_(self.torch.as_tensor(psi_local))

    def cold_psi(self, kappa: float):
        self.psi.copy_(kappa * (3.0 * self.nu / (4.0 * np.pi)) ** (2.0 / 3.0))

    def vec_psi(self):
        return self.psi

    def rescue_nearest(self):
        """An owned empty cell takes the weight of its nearest other site."""
        torch = self.torch
        s = self.slots[0]
        r = self.rows.long()
        e = r[~(s["vol"].index_select(0, r) > 0.0)]
        m = int(e.numel())
        if m == 0:
            return
        q = self.pts.index_select(0, e).contiguous()
        nn = torch.empty((m, 2), dtype=torch.int64, device="cuda")
        # the grid of self.pts (built in __init__; self.pts is never written) is reused
        self.chk(self._lib.lib().pf_knn(self.ctx, self.n, self.p(self.pts), m, self.p(q), 2, self.p(nn),
                                        0, self._s()), "pf_knn")
        j = torch.where(nn[:, 0] == e, nn[:, 1], nn[:, 0])
        self.psi.index_copy_(0, e, torch.maximum(self.psi.index_select(0, e), self.psi.index_select(0, j)))

    def rescue(self, kappa: float):
        """psi_i <- max(psi_i, kappa (3 nu_i/4 pi)^(2/3)) on the owned cells left empty."""
        s = self.slots[0]
        r = self.rows.long()
        emp = ~(s["vol"].index_select(0, r) > 0.0)
        cand = kappa * (3.0 * self.nu.index_select(0, r) / (4.0 * np.pi)) ** (2.0 / 3.0)
        cur = self.psi.index_select(0, r)
        self.psi.index_copy_(0, r, self.torch.where(emp, self.torch.maximum(cur, cand), cur))

    def psi_host(self, trial=False) -> np.ndarray:
        return (self.psi_t if trial else self.psi).cpu().numpy()

    def search_radius_max(self, dpsi: float, trial=False) -> float:
        ps = (self.psi_t if trial else self.psi).index_select(0, self.rows.long()).clamp_min(0.0)
        if self.nrows == 0:
            return 0.0
        return float((ps.sqrt() + (ps + dpsi).sqrt()).max())

    def psi_minmax(self, trial=False):
        """local (-min, max) of the owned weights as a tensor for a MAX all-reduce"""
        ps = (self.psi_t if trial else self.psi).index_select(0, self.rows.long())
        if self.nrows == 0:
            return self.torch.tensor([-np.inf, -np.inf], dtype=self.torch.float64, device="cuda")
        return self.torch.stack([-ps.min(), ps.max()])

    def trial(self, alpha: float):
        self.chk(self.L.pf_daxpy(self.n, self.p(self.psi), float(alpha), self.p(self.v["x"]),
                                 self.p(self.psi_t), self._s()), "pf_daxpy")

    def accept(self):
        self.psi.copy_(self.psi_t)
        self.slots.reverse()

    # --- evaluation and Newton pieces --------------------------------------
    def evaluate(self, dpsi: float, trial=False):
        s = self.slots[1 if trial else 0]
        ps = self.psi_t if trial else self.psi
        self.chk(self.L.pf_evaluate_lean_cells(
            self.ctx, self.n, self.p(self.pts), self.p(ps), float(dpsi), self.ball_aware, self.smf,
            self.p(self.rows), self.nrows, self.p(s["vol"]), self.p(s["ksur"]), self.p(s["fcount"]),
            self.p(s["ftag"]), self.p(s["farea"]), self.p(s["cent"]), self.p(self.flags), 0, self._s()),
            "pf_evaluate_lean_cells")

    def grad_stats(self, trial=False):
        s = self.slots[1 if trial else 0]
        out = self.scal[8:11]
        self.chk(self.L.pf_rows_gradient(self.nrows, self.p(self.rows), self.p(self.nu), self.p(s["vol"]),
                                         self.p(self.v["g"]), self.p(out), self._s()), "pf_rows_gradient")
        return out.clone()

    def hessian(self):
        s = self.slots[0]
        self.chk(self.L.pf_rows_hessian(
            self.nrows, self.p(self.rows), self.smf, self.p(self.pts), self.p(self.psi), self.p(s["fcount"]),
            self.p(s["ftag"]), self.p(s["farea"]), self.p(s["ksur"]), self.tau, self.p(self.hcnt),
            self.p(self.hcol), self.p(self.hval), self.p(self.v["diag"]), self._s()), "pf_rows_hessian")

    def cg_init(self):
        v = self.v
        out = self.torch.zeros(2, dtype=self.torch.float64, device="cuda")
        self.chk(self.L.pf_dcg_init(self.nrows, self.p(self.rows), self.p(v["g"]), self.p(v["diag"]),
                                    self.p(v["x"]), self.p(v["r"]), self.p(v["z"]), self.p(v["p"]),
                                    self.p(out), self._s()), "pf_dcg_init")
        return out

    def cg_spmv(self):
        v = self.v
        out = self.torch.zeros(1, dtype=self.torch.float64, device="cuda")
        self.chk(self.L.pf_dcg_spmv(self.nrows, self.p(self.rows), self.smf, self.p(self.hcnt),
                                    self.p(self.hcol), self.p(self.hval), self.p(v["diag"]), self.p(v["p"]),
                                    self.p(v["Ap"]), self.p(out), self._s()), "pf_dcg_spmv")
        return out

    def cg_update(self, rz, pAp):
        v = self.v
        out = self.torch.zeros(2, dtype=self.torch.float64, device="cuda")
        self.chk(self.L.pf_dcg_update(self.nrows, self.p(self.rows), self.p(v["diag"]), self.p(v["x"]),
                                      self.p(v["r"]), self.p(v["z"]), self.p(v["p"]), self.p(v["Ap"]),
                                      self.p(rz), self.p(pAp), self.p(out), self._s()), "pf_dcg_update")
        return out

    def cg_pdir(self, rz_new, rz_old):
        v = self.v
        self.chk(self.L.pf_dcg_pdir(self.nrows, self.p(self.rows), self.p(v["z"]), self.p(v["p"]),
                                    self.p(rz_new), self.p(rz_old), self._s()), "pf_dcg_pdir")

    # single-reduction PCG (u = z, w = Ap)
    def cg1_init(self):
        v = self.v
        self.chk(self.L.pf_cg1_init(self.nrows, self.p(self.rows), self.p(v["g"]), self.p(v["diag"]),
                                    self.p(v["x"]), self.p(v["r"]), self.p(v["z"]), self.p(v["p"]),
                                    self.p(v["s"]), self._s()), "pf_cg1_init")

    def cg1_spmv_dots(self):
        v = self.v
        out = self.torch.zeros(3, dtype=self.torch.float64, device="cuda")
        self.chk(self.L.pf_cg1_spmv_dots(self.nrows, self.p(self.rows), self.smf, self.p(self.hcnt),
                                         self.p(self.hcol), self.p(self.hval), self.p(v["diag"]), self.p(v["z"]),
                                         self.p(v["r"]), self.p(v["Ap"]), self.p(out), self._s()),
                 "pf_cg1_spmv_dots")
        return out

    def cg1_step(self, red, first: bool):
        v = self.v
        self.chk(self.L.pf_cg1_step(self.nrows, self.p(self.rows), self.p(v["diag"]), self.p(v["x"]),
                                    self.p(v["r"]), self.p(v["z"]), self.p(v["Ap"]), self.p(v["p"]),
                                    self.p(v["s"]), self.p(red), self.p(self.cg1_sc), int(first), self._s()),
                 "pf_cg1_step")

    # device-side convergence (one host read per batch of iterations)
    def cg1_conv_reset(self):
        self.cg1_sc.zero_()

    def cg1_spmv_dots_c(self):
        v = self.v
        out = self.torch.zeros(3, dtype=self.torch.float64, device="cuda")
        self.chk(self.L.pf_cg1_spmv_dots_c(self.nrows, self.p(self.rows), self.smf, self.p(self.hcnt),
                                           self.p(self.hcol), self.p(self.hval), self.p(v["diag"]),
                                           self.p(v["z"]), self.p(v["r"]), self.p(v["Ap"]), self.p(out),
                                           self.p(self.cg1_sc), self._s()), "pf_cg1_spmv_dots_c")
        return out

    def cg1_step_conv(self, red, rtol: float, max_iter: int):
        v = self.v
        self.chk(self.L.pf_cg1_step_conv(self.nrows, self.p(self.rows), self.p(v["diag"]), self.p(v["x"]),
                                         self.p(v["r"]), self.p(v["z"]), self.p(v["Ap"]), self.p(v["p"]),
                                         self.p(v["s"]), self.p(red), self.p(self.cg1_sc), float(rtol),
                                         int(max_iter), self._s()), "pf_cg1_step_conv")

    def cg1_status(self):
        sc = self.cg1_sc[4:6].cpu()
        return bool(sc[0] != 0.0), int(sc[1])

    def vec(self, name):
        return self.v[name]

    def index(self, ix: np.ndarray):
        return self.torch.as_tensor(ix, dtype=self.torch.int64, device="cuda")

    def tensor(self, vals):
        return self.torch.tensor(vals, dtype=self.torch.float64, device="cuda")

    def scalar(self, t) -> float:
        return float(t)

    def owned(self, name: str) -> np.ndarray:
        src = self.psi if name == "psi" else self.v[name]
        return src.index_select(0, self.rows.long()).cpu().numpy()

    def result(self):
        s = self.slots[0]
        r = self.rows.long()
        return {k: s[k].index_select(0, r) for k in ("vol", "ksur", "fcount", "cent")}


# ---------------------------------------------------------------------------
# the solver
# ---------------------------------------------------------------------------
@dataclass
class DistResult:
    psi_owned: np.ndarray        # weights of the owned sites (global order)
    owned_global: np.ndarray     # their global indices
    stats: dict = field(default_factory=dict)


class DistNewton:
    """Partitioned Newton solve.  `pts` / `nu` are the global arrays (replicated
    on every rank); ops_factory(pts_local, nu_local, rows) builds the backend."""

    def __init__(self, pts: np.ndarray, nu: np.ndarray, domain, group=None, smf: int = 32,
                 ball_aware: bool = True, slack: float = 1.5, ops_factory=None, axis_lo=None,
                 axis_hi=None, cg: str = "single"):
        self.pts = None if pts is None else np.ascontiguousarray(pts, dtype=np.float64)
        self.nu = None if nu is None else np.ascontiguousarray(nu, dtype=np.float64)
        self.domain = domain
        self.comm = Comm(group)
        self.smf, self.ball_aware, self.slack = smf, ball_aware, slack
        self.cg = cg  # "single": one all-reduce per CG iteration; "classic": two
        self.cg_batch = 8  # CG iterations per host convergence read (device-side test)
        # slab boundaries: x-quantiles of the sites (balanced) unless given
        self.lo, self.hi = axis_lo, axis_hi
        self.tau = 1e-12 * domain.diagonal() ** 2
        self.ops_factory = ops_factory or (lambda p, n, r: CudaOps(p, n, r, domain, smf, ball_aware,
                                                                   self.tau))
        self.repartitions = 0
        self.halo_entries = 0

    # --- partition --------------------------------------------------------
    def _partition(self, psi_global: np.ndarray, dpsi: float, psi_plan: np.ndarray | None = None):
        """Slabs, ghosts and halo plan.  The ghost margin is sized from
        ``psi_plan`` (default the weights themselves): a trial re-partition
        passes the trial weights psi + alpha x, whose search radii the trial
        evaluation needs."""
        c = self.comm
        self.slab, self.plan = partition.halo_plan(self.pts, psi_global if psi_plan is None else psi_plan,
                                                   dpsi, c.world, c.rank, self.lo, self.hi, self.slack)
        l2g = self.slab.local_to_global
        self.ops = self.ops_factory(self.pts[l2g], self.nu[l2g], self.slab.owned_local)
        self.ops.set_psi(psi_global[l2g])
        self.idx_send = {q: self.ops.index(ix) for q, ix in self.plan.send.items()}
        self.idx_recv = {q: self.ops.index(ix) for q, ix in self.plan.recv.items()}
        self.halo_entries = self.plan.volume()

    def _gather_global(self, local_vals: np.ndarray) -> np.ndarray:
        """Global array from every rank's owned entries of a local-length array."""
        own = self.slab.owned_local
        parts = self.comm.all_gather_objects((self.slab.local_to_global[own], local_vals[own]))
        out = np.zeros(len(self.pts))
        for g, v in parts:
            out[g] = v
        return out

    def _dpsi(self, trial=False) -> float:
        t = self.comm.all_reduce(self.ops.psi_minmax(trial), "max")
        lo, hi = -float(t[0]), float(t[1])
        return max(hi - lo, 0.0) if np.isfinite(hi) else 0.0

    def _margin_ok(self, dpsi: float, trial=False) -> bool:
        need = self.ops.search_radius_max(dpsi, trial)
        bad = self.ops.tensor([1.0 if need > self.slab.ghost_margin else 0.0])
        return float(self.comm.all_reduce(bad, "max")[0]) == 0.0

    def _evaluate(self, trial=False):
        """Evaluate the owned cells (current or trial weights); returns the
        all-reduced (worst, min vol, min nu)."""
        dpsi = self._dpsi(trial)
        for _ in range(8):
            if self._margin_ok(dpsi, trial):
                break
            # weights outgrew the ghost layer: re-partition, with the margin
            # sized for the weights being evaluated (the trial weights
            # psi + alpha x on a damping trial)
            self._repartition(dpsi, trial)
            self.repartitions += 1
            if trial:
                self.ops.trial(self._alpha)
            dpsi = self._dpsi(trial)
        else:
            raise RuntimeError("ghost layer still too thin after 8 re-partitions")
        self.ops.evaluate(dpsi, trial)
        st = self.comm.all_reduce(self.ops.grad_stats(trial), "max")
        st = [float(v) for v in st.cpu()]
        return st[0], -st[1], -st[2]

    def _repartition(self, dpsi: float, trial: bool):
        """Re-partition from the all-gathered global weights (replicated mode)."""
        psi_g = self._gather_global(self.ops.psi_host(False))
        x_g = self._gather_global(self.ops.vec("x").cpu().numpy()) if trial else None
        self._partition(psi_g, dpsi, psi_g + self._alpha * x_g if trial else None)
        if trial:
            self.ops.vec("x").copy_(self.ops.torch.as_tensor(x_g[self.slab.local_to_global]))

    def _start(self, psi_init):
        """Initial weights (cold: the free balls' (3 nu / 4 pi)^(2/3)) and the
        first partition; returns whether the start is cold."""
        cold = psi_init is None
        psi0 = (3.0 * self.nu / (4.0 * np.pi)) ** (2.0 / 3.0) if cold else np.asarray(psi_init, np.float64)
        lo_, hi_ = float(psi0.min()), float(psi0.max())
        self._partition(psi0, max(hi_ - lo_, 0.0))
        return cold

    # --- Jacobi-PCG ---------------------------------------------------------
    def _pcg1(self, rtol: float, max_iter: int = 10000) -> int:
        """Single-reduction Jacobi-PCG (Chronopoulos & Gear): per iteration one halo
        exchange of u = D^-1 r and ONE all-reduce of (r.u, w.u, r.r), w = A u.
        With a backend that tests convergence on the device (cg1_step_conv) the
        iterations are stream-ordered and the host reads one flag per
        ``cg_batch`` iterations (iterations past convergence are no-ops)."""
        o, c = self.ops, self.comm
        o.cg1_init()
        if self.cg_batch > 1 and hasattr(o, "cg1_step_conv"):
            o.cg1_conv_reset()
            while True:
                for _ in range(self.cg_batch):
                    c.exchange(o.vec("z"), self.plan, self.idx_send, self.idx_recv)
                    red = c.all_reduce(o.cg1_spmv_dots_c(), "sum")
                    o.cg1_step_conv(red, rtol, max_iter)
                done, it = o.cg1_status()
                if done:
                    return it
        bb, it = 0.0, 0
        while True:
            c.exchange(o.vec("z"), self.plan, self.idx_send, self.idx_recv)
            red = c.all_reduce(o.cg1_spmv_dots(), "sum")
            rr = float(red[2])
            if it == 0:
                bb = rr
                if not bb > 0.0:
                    return 0
            elif np.sqrt(rr) <= rtol * np.sqrt(bb) or it >= max_iter or not np.isfinite(rr):
                return it
            o.cg1_step(red, it == 0)
            it += 1

    def _pcg(self, rtol: float, max_iter: int = 10000) -> int:
        o, c = self.ops, self.comm
        t = c.all_reduce(o.cg_init(), "sum")
        rz, bb = t[0:1].clone(), float(t[1])
        if not bb > 0.0:
            return 0
        it = 0
        while True:
            c.exchange(o.vec("p"), self.plan, self.idx_send, self.idx_recv)
            pAp = c.all_reduce(o.cg_spmv(), "sum")
            t = c.all_reduce(o.cg_update(rz, pAp), "sum")
            rz_new, rr = t[0:1].clone(), float(t[1])
            it += 1
            if np.sqrt(rr) <= rtol * np.sqrt(bb) or it >= max_iter or not np.isfinite(float(rz_new)):
                break
            o.cg_pdir(rz_new, rz)
            rz = rz_new
        return it

    # --- Newton (same control flow as pf_newton_solve) -------
    def solve(self, psi_init: np.ndarray | None = None, eps_vol: float = 0.01,
              max_newton: int = 100) -> DistResult:
        S = dict(status=0, iterations=0, evaluations=0, cg_iterations=0, damping_halvings=0,
                 init_doublings=0, worst_initial=0.0, worst_final=0.0, last_alpha=0.0)
        self._alpha = 1.0
        cold = self._start(psi_init)
        if cold:
            kappa = 1.0
            while True:
                self.ops.cold_psi(kappa)
                S["evaluations"] += 1
                worst, vmin, nmin = self._evaluate()
                if vmin > 0.0:
                    break
                kappa *= 2.0
                S["init_doublings"] += 1
                if kappa > 1024.0:
                    S["status"] = 3
                    return self._result(S)
        else:
            S["evaluations"] += 1
            worst, vmin, nmin = self._evaluate()
            if not vmin > 0.0:  # warm start with per-cell rescue (SPEC.md init_weights)
                self.ops.rescue_nearest()
                self.comm.exchange(self.ops.vec_psi(), self.plan, self.idx_send, self.idx_recv)
                S["init_doublings"] += 1
                S["evaluations"] += 1
                worst, vmin, nmin = self._evaluate()
            kappa = 1.0
            while not vmin > 0.0:
                if kappa > 1024.0:
                    S["status"] = 3
                    return self._result(S)
                self.ops.rescue(kappa)
                self.comm.exchange(self.ops.vec_psi(), self.plan, self.idx_send, self.idx_recv)
                S["init_doublings"] += 1
                S["evaluations"] += 1
                worst, vmin, nmin = self._evaluate()
                kappa *= 2.0
        floor_v = 0.5 * min(nmin, vmin)
        S["worst_initial"] = worst
        for _ in range(max_newton):
            if worst <= eps_vol:
                break
            self.ops.hessian()
            rtol = 1e-4 if worst < 10.0 * eps_vol else 1e-3
            S["cg_iterations"] += self._pcg1(rtol) if self.cg == "single" else self._pcg(rtol)
            # the step's ghost entries, then every trial is local
            self.comm.exchange(self.ops.vec("x"), self.plan, self.idx_send, self.idx_recv)
            alpha, accepted = 1.0, False
            while alpha >= 2.0 ** -20:
                self._alpha = alpha
                self.ops.trial(alpha)
                S["evaluations"] += 1
                w_t, vmin_t, _ = self._evaluate(trial=True)
                if vmin_t >= floor_v:
                    accepted = True
                    break
                alpha *= 0.5
                S["damping_halvings"] += 1
            if not accepted:
                S["status"] = 2
                break
            self.ops.accept()
            S["iterations"] += 1
            S["last_alpha"] = alpha
            worst = w_t
        S["worst_final"] = worst
        if S["status"] == 0 and worst > eps_vol:
            S["status"] = 1
        return self._result(S)

    def _result(self, S) -> DistResult:
        S["status_name"] = STATUS.get(S["status"], "?")
        S["repartitions"] = self.repartitions
        S["halo_entries"] = self.halo_entries
        S["world"] = self.comm.world
        own = self.slab.owned_local
        return DistResult(psi_owned=self.ops.owned("psi"), owned_global=self.slab.local_to_global[own],
                          stats=S)


class DistNewtonLocal(DistNewton):
    """The same partitioned solve with no replicated arrays: every rank passes
    only the sites it owns (global ids, positions, volumes as tensors on its
    device, gid order) and the x-slab cuts.  The local set (owned + ghosts)
    and the CG halo plan come from ``halo.SlabComm.ghosts`` (all-to-alls of
    the owned rows within each peer's margin); a re-partition re-exchanges the
    ghosts with a wider margin from the owned weights -- nothing is gathered.
    Per-cell results and the Newton iterations equal ``DistNewton``'s
    (tests/test_halo_gloo.py)."""

    def __init__(self, gid, pts, nu, domain, cuts, group=None, smf: int = 32, ball_aware: bool = True,
                 slack: float = 1.5, ops_factory=None, cg: str = "single"):
        import torch

        from . import halo

        super().__init__(None, None, domain, group=group, smf=smf, ball_aware=ball_aware, slack=slack,
                         ops_factory=ops_factory, cg=cg)
        self.torch = torch
        self.halo = halo
        self.gid = torch.as_tensor(gid, dtype=torch.int64)
        dev = self.gid.device
        self.own_pts = torch.as_tensor(pts, dtype=torch.float64, device=dev).contiguous()
        self.own_nu = torch.as_tensor(nu, dtype=torch.float64, device=dev).contiguous()
        self.sc = halo.SlabComm(cuts, self.comm)

    def _exchange(self, psi_own, dpsi: float, psi_plan_own=None, x_own=None):
        t = self.torch
        dev = self.gid.device
        psi_own = t.as_tensor(psi_own, dtype=t.float64, device=dev)
        plan = psi_own if psi_plan_own is None else t.as_tensor(psi_plan_own, dtype=t.float64, device=dev)
        margin = self.halo.ghost_margin(plan.cpu().numpy(), dpsi, self.slack)
        fields = {"pts": self.own_pts, "nu": self.own_nu, "psi": psi_own}
        if x_own is not None:
            fields["x"] = t.as_tensor(x_own, dtype=t.float64, device=dev)
        loc = self.sc.ghosts(self.gid, fields, margin)
        owned = loc.owned.cpu().numpy().astype(np.int32)
        self.slab = partition.Slab(self.comm.rank, self.comm.world, loc.lo, loc.hi, loc.gid.cpu().numpy(),
                                   owned, margin)
        self.plan = loc.plan
        lp = loc.fields["pts"] if dev.type == "cuda" else loc.fields["pts"].numpy()
        ln = loc.fields["nu"] if dev.type == "cuda" else loc.fields["nu"].numpy()
        self.ops = self.ops_factory(lp, ln, owned)
        self.ops.set_psi(loc.fields["psi"] if dev.type == "cuda" else loc.fields["psi"].numpy())
        if x_own is not None:
            self.ops.vec("x").copy_(loc.fields["x"])
        self.idx_send = {q: self.ops.index(ix) for q, ix in self.plan.send.items()}
        self.idx_recv = {q: self.ops.index(ix) for q, ix in self.plan.recv.items()}
        self.halo_entries = self.plan.volume()

    def _partition(self, psi, dpsi, psi_plan=None):
        self._exchange(psi, dpsi, psi_plan)

    def _repartition(self, dpsi: float, trial: bool):
        psi_own = self.ops.owned("psi")
        x_own = self.ops.owned("x") if trial else None
        self._exchange(psi_own, dpsi, psi_own + self._alpha * x_own if trial else None, x_own)

    def _start(self, psi_init):
        t = self.torch
        cold = psi_init is None
        if cold:
            psi0 = (3.0 * self.own_nu / (4.0 * np.pi)) ** (2.0 / 3.0)
        else:
            psi0 = t.as_tensor(psi_init, dtype=t.float64, device=self.gid.device)
        if psi0.numel():
            mm = t.stack([-psi0.min(), psi0.max()])
        else:
            mm = t.tensor([-np.inf, -np.inf], dtype=t.float64, device=psi0.device)
        if self.comm.gloo and mm.is_cuda:
            mm = mm.cpu()
        mm = self.comm.all_reduce(mm, "max")
        lo_, hi_ = -float(mm[0]), float(mm[1])
        self._partition(psi0, max(hi_ - lo_, 0.0) if np.isfinite(hi_) else 0.0)
        return cold
