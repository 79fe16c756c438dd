"""Viscosity, wall friction and surface tension
on the device: the implicit update (m/dt I + mu L) v = m/dt v + F against a
scipy restatement assembled from the same step's restricted facets, and the
SPEC examples (mu = 0 is the explicit update; a uniform velocity field is a
Laplacian kernel; two particles under strong viscosity move together)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _state(sc):
    from paper_2601_05765_b200 import fluid

    return fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)


def _run(sc, **kw):
    from paper_2601_05765_b200 import fluid, geom

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    st = _state(sc)
    prm = fluid.SimParams(dt=1e-3, eps=kw.pop("eps", 5e-3), gravity=kw.pop("gravity", (0.0, 0.0, -9.81)), **kw)
    d = fluid.step(st, prm, dom)
    return st, d, prm, dom


def test_zero_viscosity_is_the_explicit_update():
    from paper_2601_05765_b200 import scenes

    sc = scenes.c2_dam_break(m=10)
    a, _, _, _ = _run(sc, implicit=False)
    b, d, _, _ = _run(sc, implicit=True)
    assert d["viscosity_cg_iterations"] > 0
    va, vb = a.v.cpu().numpy(), b.v.cpu().numpy()
    assert np.max(np.abs(va - vb)) <= 1e-9 * max(1.0, np.max(np.abs(va)))


def test_implicit_update_matches_restatement():
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    import torch

    from paper_2601_05765_b200 import _lib, fluid, geom, laguerre, scenes, solver

    sc = scenes.c2_dam_break(m=10)
    mu, mu_b, gam, aff = 0.05, 0.02, 2e-4, 0.7
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    st = _state(sc)
    prm = fluid.SimParams(dt=1e-3, eps=5e-3, viscosity=mu, boundary_viscosity=mu_b, surface_tension=gam,
                          boundary_affinity=aff)
    v0 = st.v.cpu().numpy().copy()
    fluid.step(st, prm, dom)
    x = st.x.cpu().numpy()
    n, smf = sc.n, prm.smf
    vol, _, fc, ft, fa = [t.cpu().numpy() for t in solver.last_state(n, smf)]
    cent = torch.empty((n, 3), dtype=torch.float64, device="cuda")
    fluid._bind().pf_newton_last_state_ex(None, None, None, None, None, _lib.ptr(cent), n, smf,
                                           _lib.stream_ptr())
    cent = cent.cpu().numpy()
    planes = laguerre.domain_pack(dom).args()[2][:6]
    m = sc.rho * sc.nu
    rows, cols, vals = [], [], []
    diag = m / prm.dt
    ftt = np.zeros((n, 3))
    for i in range(n):
        for s in range(min(fc[i], smf)):
            j, A = int(ft[i, s]), fa[i, s]
            if j >= 0:
                w = 0.5 * A / np.linalg.norm(x[j] - x[i])
                rows.append(i); cols.append(j); vals.append(-mu * w)
                diag[i] += mu * w
                ftt[i] += w * (x[j] - x[i])
            else:
                nrm, dd = planes[-j - 1, :3], planes[-j - 1, 3]
                dist = dd - nrm @ x[i]
                vi = vol[i] if vol[i] > 0 else sc.nu[i]
                diag[i] += mu_b * 0.5 * A / (max(dist, 1e-300) * vi)
                gvec = (dist - np.cbrt(vi)) * nrm
                if np.linalg.norm(gvec) > 0:
                    ftt[i] += aff * 0.5 * A / np.linalg.norm(gvec) * gvec
    M = sp.csr_matrix((vals, (rows, cols)), shape=(n, n)) + sp.diags(diag)
    g = np.array([0.0, 0.0, -9.81])
    rhs = (m / prm.dt)[:, None] * v0 + m[:, None] * (cent - x) / prm.eps ** 2 + m[:, None] * g + gam * ftt
    v_ref = np.stack([spl.spsolve(M.tocsc(), rhs[:, a]) for a in range(3)], 1)
    v = st.v.cpu().numpy()
    assert np.max(np.abs(v - v_ref)) <= 1e-7 * np.max(np.abs(v_ref))


def test_uniform_velocity_is_a_laplacian_kernel():
    from paper_2601_05765_b200 import scenes

    sc = scenes.c2_dam_break(m=10)
    sc.vel[:] = np.array([0.3, -0.2, 0.1])
    st, _, _, _ = _run(sc, viscosity=10.0, eps=1e10, gravity=(0.0, 0.0, 0.0))
    v = st.v.cpu().numpy()
    assert np.max(np.abs(v - sc.vel)) <= 1e-8


def test_two_particles_strong_viscosity_move_together():
    from paper_2601_05765_b200 import scenes

    pts = np.array([[0.45, 0.5, 0.5], [0.55, 0.5, 0.5]])
    nu = np.full(2, 4.0 / 3.0 * np.pi * 0.07 ** 3)
    vel = np.array([[1.0, 0.0, 0.0], [-1.0, 0.0, 0.0]])
    sc = scenes.Scene("two", pts, nu, vel, np.full(2, 1000.0))
    st, _, _, _ = _run(sc, viscosity=1e12, eps=1e10, gravity=(0.0, 0.0, 0.0))
    v = st.v.cpu().numpy()
    assert np.max(np.abs(v - v.mean(0))) <= 1e-6
