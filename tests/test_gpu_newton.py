"""Device Newton solve (pf_newton_solve) vs the CPU restatement: same Newton
iteration and evaluation counts, final weights within the solver tolerance,
every cell within eps_vol of its prescribed volume."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(scene):
    import torch

    from oracle import newton_ref as NR
    from paper_2601_05765_b200 import geom, laguerre, solver

    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    dpk = laguerre.domain_pack(dom)
    res = solver.newton_solve(torch.as_tensor(scene.pts, device="cuda"),
                              torch.as_tensor(scene.nu, device="cuda"), dom)
    psi_ref, st_ref = NR.newton_solve(scene.pts, scene.nu, dpk.args(), dpk.tol, dom.diagonal())
    return res, psi_ref, st_ref


@pytest.mark.parametrize("which", ["C1", "C2-small", "two-fluid-small"])
def test_newton_matches_cpu_restatement(which):
    from paper_2601_05765_b200 import scenes, solver

    sc = {"C1": lambda: scenes.c1_random(),
          "C2-small": lambda: scenes.c2_dam_break(m=20),
          "two-fluid-small": lambda: scenes.c5_two_fluid(n_target=12_000)}[which]()
    res, psi_ref, st_ref = _run(sc)
    st = res.stats
    assert st["status"] == 0 == st_ref["status"]
    assert st["iterations"] == st_ref["iterations"]
    assert st["evaluations"] == st_ref["evaluations"]
    assert abs(st["cg_iterations"] - st_ref["cg_iterations"]) <= st["iterations"]
    psi = res.psi.cpu().numpy()
    assert np.max(np.abs(psi - psi_ref) / psi_ref) < 1e-6
    vol = solver.last_state(sc.n, res.smf)[0].cpu().numpy()
    assert np.max(np.abs(vol - sc.nu) / sc.nu) <= 0.01


def test_newton_c1_survey_counts():
    from paper_2601_05765_b200 import scenes

    res, _, _ = _run(scenes.c1_random())
    st = res.stats
    assert (st["iterations"], st["evaluations"]) == (4, 5)
    assert abs(st["cg_iterations"] - 65) <= 4
