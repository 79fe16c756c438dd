"""CLI driver and frames on the device: `simulate` writes
frames and stats.csv, a frame re-evaluated from (x, psi) reproduces its stored
volumes (SPEC cli_io property, 1e-12), a warm start from a frame continues the
run, and `bench` prints the Table 1 stage columns."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_simulate_frames_and_warm_start(tmp_path):
    import torch

    from paper_2601_05765_b200 import cli, frames, geom, restricted, scenes

    out = tmp_path / "run"
    assert cli.main(["simulate", "--config", "C2", "--steps", "4", "--out", str(out), "--frame-stride", "2"]) == 0
    rows = open(out / "stats.csv").read().strip().splitlines()
    assert len(rows) == 5 and rows[0].startswith("step,")
    f = frames.read_frame(str(out / "frame_000004.potf"))
    assert f.step == 4 and f.worst_rel_error <= 0.01
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    d = restricted.evaluate(torch.as_tensor(f.x, device="cuda"), torch.as_tensor(f.psi, device="cuda"), dom)
    vol = d.vol.cpu().numpy()
    assert np.max(np.abs(vol - f.vol) / f.vol) <= 1e-12
    out2 = tmp_path / "resume"
    assert cli.main(["simulate", "--config", "C2", "--steps", "2", "--out", str(out2), "--frame-stride", "1",
                     "--warm-start", str(out / "frame_000004.potf")]) == 0
    g = frames.read_frame(str(out2 / "frame_000006.potf"))
    assert g.step == 6 and g.worst_rel_error <= 0.01
    del scenes


def test_bench_table(capsys):
    from paper_2601_05765_b200 import cli

    assert cli.main(["bench", "--sizes", "8000", "--steps", "3"]) == 0
    txt = capsys.readouterr().out
    assert "Laguerre" in txt and "Evaluation" in txt and "Complete Step" in txt


@pytest.mark.parametrize("mode", ["raw", "smooth", "depth"])
def test_render_frame(tmp_path, mode):
    from paper_2601_05765_b200 import cli

    out = tmp_path / "run"
    assert cli.main(["simulate", "--config", "C2", "--steps", "1", "--out", str(out), "--frame-stride", "1"]) == 0
    img = tmp_path / f"{mode}.ppm"
    args = ["render", str(out / "frame_000001.potf"), "--out", str(img), "--mode", mode, "--width", "160",
            "--height", "120"]
    if mode == "raw":
        args += ["--samples", "500", "--cloud", str(tmp_path / "s.xyz")]
    assert cli.main(args) == 0
    raw = open(img, "rb").read()
    assert raw.startswith(b"P6\n160 120\n255\n") and len(raw) == len(b"P6\n160 120\n255\n") + 160 * 120 * 3
    if mode == "raw":
        pts = np.loadtxt(tmp_path / "s.xyz")
        assert pts.shape == (500, 6) and np.allclose(np.linalg.norm(pts[:, 3:], axis=1), 1.0)
