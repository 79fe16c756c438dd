"""First-hit renderer (SPEC.md:406-463 examples): a lone ball's silhouette
radius within 1 px of the pinhole projection, an empty scene is all
background, and on a random scene every pixel's hit equals the brute-force
nearest ray-ball entry; each hit point lies in its ball's Laguerre cell."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_lone_ball_silhouette_and_empty_scene(tmp_path):
    from paper_2601_05765_b200 import render

    cam = render.Camera(eye=(0.5, -1.5, 0.5), look_at=(0.5, 0.5, 0.5), up=(0, 0, 1), fov=0.6, width=256, height=256)
    ids, _ = render.first_hit(np.array([[0.5, 0.5, 0.5]]), np.array([0.1 ** 2]), cam)
    mask = ids.cpu().numpy() >= 0
    r_px = np.sqrt(mask.sum() / np.pi)
    dist = 2.0
    ang = np.arcsin(0.1 / dist)
    r_ref = np.tan(ang) / np.tan(0.3) * 128  # half height = 128 px
    assert abs(r_px - r_ref) < 1.0
    ids, _ = render.first_hit(np.array([[0.5, 0.5, 0.5]]), np.array([0.0]), cam)
    assert (ids.cpu().numpy() < 0).all()
    img = render.render_raw(np.array([[0.5, 0.5, 0.5]]), np.array([0.1 ** 2]), cam)
    render.write_ppm(str(tmp_path / "ball.ppm"), img)
    assert open(tmp_path / "ball.ppm", "rb").read(2) == b"P6"


def test_random_scene_matches_brute_force():
    from paper_2601_05765_b200 import render

    rng = np.random.default_rng(2)
    n = 300
    pts = 0.2 + 0.6 * rng.random((n, 3))
    psi = (0.02 + 0.04 * rng.random(n)) ** 2
    cam = render.Camera(eye=(0.5, -1.2, 0.7), look_at=(0.5, 0.5, 0.45), fov=0.7, width=96, height=72)
    ids, ts = render.first_hit(pts, psi, cam)
    ids, ts = ids.cpu().numpy(), ts.cpu().numpy()
    cp = cam.packed()
    eye = cp[:3]
    hits = 0
    for py in range(cam.height):
        for px in range(cam.width):
            sx = (2.0 * (px + 0.5) / cam.width - 1.0) * cp[12] * cp[13]
            sy = (1.0 - 2.0 * (py + 0.5) / cam.height) * cp[12]
            d = cp[3:6] + sx * cp[6:9] + sy * cp[9:12]
            d /= np.linalg.norm(d)
            w = eye[None, :] - pts
            b = w @ d
            c = (w * w).sum(1) - psi
            disc = b * b - c
            t = np.where(disc >= 0, -b - np.sqrt(np.maximum(disc, 0)), np.inf)
            t = np.where(t >= 0, t, np.inf)
            j = int(np.argmin(t))
            if np.isfinite(t[j]):
                hits += 1
                assert ids[py, px] == j and abs(ts[py, px] - t[j]) <= 1e-12
                x = eye + t[j] * d
                pw = ((x[None, :] - pts) ** 2).sum(1) - psi
                assert pw[j] <= pw.min() + 1e-12  # the hit point lies in cell j (power membership)
            else:
                assert ids[py, px] == -1
    assert hits > 100
