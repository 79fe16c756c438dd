"""Fluid step (A17) on the device: advection + reflection, warm-started Newton
every step, spring-to-centroid + gravity velocity update.
Checked against a torch restatement of the same update formulas."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_dam_break_steps():
    import torch

    from paper_2601_05765_b200 import fluid, geom, scenes, solver

    sc = scenes.c2_dam_break(m=12)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
    prm = fluid.SimParams(dt=1e-3, eps=5e-3)
    for k in range(3):
        x0, v0 = st.x.clone(), st.v.clone()
        d = fluid.step(st, prm, dom)
        assert d["status_name"] == "converged", d
        assert d["worst_final"] <= prm.eps_vol
        # restate the update with the device centroids
        xa = x0 + prm.dt * v0
        lo, hi = 1e-9 * dom.diagonal(), 1.0 - 1e-9 * dom.diagonal()
        assert torch.all(st.x >= lo) and torch.all(st.x <= hi)
        inside = (xa > lo) & (xa < hi)
        assert torch.allclose(st.x[inside], xa[inside], rtol=0, atol=1e-15)
        _, _, _, _, _ = solver.last_state(sc.n, prm.smf)
        cent = torch.empty((sc.n, 3), dtype=torch.float64, device="cuda")
        import ctypes as C

        from paper_2601_05765_b200 import _lib

        L = fluid._bind()
        L.pf_newton_last_state_ex(None, None, None, None, None, _lib.ptr(cent), sc.n, prm.smf,
                                  _lib.stream_ptr())
        m = (st.rho * st.nu)[:, None]
        g = torch.tensor(prm.gravity, dtype=torch.float64, device="cuda")
        v_ref = torch.where(inside, v0, -v0) + prm.dt * (m * (cent - st.x) / prm.eps ** 2 + m * g) / m
        assert torch.allclose(st.v, v_ref, rtol=1e-12, atol=1e-12)
    # total volume conserved within n * eps_vol * mean(nu) (SPEC.md fluid invariants)
    vol = solver.last_state(sc.n, prm.smf)[0]
    assert abs(float(vol.sum()) - float(sc.nu.sum())) <= sc.n * prm.eps_vol * float(sc.nu.mean())


def test_chocs_wall_impact_converges():
    """C3 (BASELINE configs[2]): 500k particles flying radially at 5 m/s hit the
    walls around step 50; every step's warm-started Newton solve converges,
    the KMT line search is exercised, and the nearest-site rescue keeps the
    warm start valid through the impact."""
    from paper_2601_05765_b200 import fluid, geom, scenes

    sc = scenes.c3_chocs()
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
    prm = fluid.SimParams(dt=1e-3, eps=5e-3)
    halvings = 0
    for _ in range(60):
        d = fluid.step(st, prm, dom)  # raises OtNonConvergence on failure
        assert d["worst_final"] <= prm.eps_vol
        halvings += d["damping_halvings"]
    assert halvings > 0
    assert float(st.x.min()) > 0.0 and float(st.x.max()) < 1.0
