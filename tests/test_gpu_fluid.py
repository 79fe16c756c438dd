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


@pytest.mark.parametrize("spring", ["spec", "gallouet_merigot"])
def test_pressure_force_spec_examples(spring):
    """SPEC.md pressure_force examples: x at the centroid -> 0; c - x =
    (eps^2, 0, 0) -> (1, 0, 0) as printed (spring="spec"); the
    Gallouet-Merigot form scales it by the particle mass m = rho nu."""
    import torch

    from paper_2601_05765_b200 import fluid

    eps = 5e-3
    x = torch.tensor([[0.3, 0.4, 0.5], [0.2, 0.2, 0.2]], dtype=torch.float64)
    c = x.clone()
    c[1, 0] += eps ** 2
    nu = torch.tensor([1e-6, 2e-6], dtype=torch.float64)
    rho = torch.tensor([1000.0, 100.0], dtype=torch.float64)
    F = fluid.pressure_force(x, c, nu, rho, eps, spring).cpu()
    assert torch.all(F[0] == 0.0)
    k = 1.0 if spring == "spec" else float(rho[1] * nu[1])
    assert torch.allclose(F[1], torch.tensor([k, 0.0, 0.0], dtype=torch.float64), rtol=1e-12, atol=0.0)


def test_step_spec_spring():
    """One step with the SPEC's literal spring (F_p = (c - x)/eps^2, v += dt/m F):
    the velocity update equals the restatement with the device centroids; a
    lone particle at its cell centroid with no gravity stays at rest (SPEC step
    example)."""
    import torch

    from paper_2601_05765_b200 import _lib, fluid, geom, scenes

    sc = scenes.c2_dam_break(m=8)
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    st = fluid.make_state(sc.pts, sc.vel, sc.nu, sc.rho)
    prm = fluid.SimParams(dt=1e-4, eps=5e-3, spring="spec")
    x0, v0 = st.x.clone(), st.v.clone()
    d = fluid.step(st, prm, dom)
    assert d["status_name"] == "converged", d
    cent = torch.empty((sc.n, 3), dtype=torch.float64, device="cuda")
    L = fluid._bind()
    L.pf_newton_last_state_ex(None, None, None, None, None, _lib.ptr(cent), sc.n, prm.smf, _lib.stream_ptr())
    m = (st.rho * st.nu)[:, None]
    g = torch.tensor(prm.gravity, dtype=torch.float64, device="cuda")
    v_ref = v0 + prm.dt * ((cent - st.x) / prm.eps ** 2 + m * g) / m
    assert torch.allclose(st.v, v_ref, rtol=1e-12, atol=1e-12)
    # lone particle at the centre of a ball that fits the domain: centroid = x, no gravity
    one = fluid.make_state(np.array([[0.5, 0.5, 0.5]]), np.zeros((1, 3)), np.array([1e-3]), np.array([1000.0]))
    d = fluid.step(one, fluid.SimParams(dt=1e-3, eps=5e-3, gravity=(0.0, 0.0, 0.0), spring="spec"), dom)
    assert d["status_name"] == "converged"
    assert float(one.v.abs().max()) <= 1e-9 and torch.allclose(one.x.cpu(), torch.tensor([[0.5, 0.5, 0.5]],
                                                                                           dtype=torch.float64))
