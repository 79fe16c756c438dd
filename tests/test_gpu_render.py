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


def _dirs(cam):
    cp = cam.packed()
    out = np.empty((cam.height, cam.width, 3))
    for py in range(cam.height):
        for px in range(cam.width):
            sx = (2.0 * (px + 0.5) / cam.width - 1.0) * cp[12] * cp[13]
            sy = (1.0 - 2.0 * (py + 0.5) / cam.height) * cp[12]
            d = cp[3:6] + sx * cp[6:9] + sy * cp[9:12]
            out[py, px] = d / np.linalg.norm(d)
    return cp[:3], out


def test_depth_is_the_chord_length_of_the_union_of_balls():
    """Depth mode (SPEC render): a lone ball gives the analytic chord; on an
    overlapping random scene every pixel equals the brute-force union of the
    ray's ball chords."""
    from paper_2601_05765_b200 import render

    cam = render.Camera(eye=(0.5, -1.5, 0.5), look_at=(0.5, 0.5, 0.5), fov=0.5, width=65, height=65)
    r = 0.15
    dp = render.depth(np.array([[0.5, 0.5, 0.5]]), np.array([r * r]), cam).cpu().numpy()
    eye, D = _dirs(cam)
    w = eye - np.array([0.5, 0.5, 0.5])
    b = D @ w
    disc = b * b - (w @ w - r * r)
    ref = np.where(disc > 0, 2 * np.sqrt(np.maximum(disc, 0)), 0.0)
    assert abs(dp[32, 32] - 2 * r) <= 1e-12
    assert np.max(np.abs(dp - ref)) <= 1e-12

    rng = np.random.default_rng(5)
    n = 250
    pts = 0.2 + 0.6 * rng.random((n, 3))
    psi = (0.03 + 0.05 * rng.random(n)) ** 2
    cam = render.Camera(eye=(0.4, -1.3, 0.8), look_at=(0.5, 0.5, 0.45), fov=0.7, width=48, height=36)
    dp = render.depth(pts, psi, cam).cpu().numpy()
    eye, D = _dirs(cam)
    nz = 0
    for py in range(cam.height):
        for px in range(cam.width):
            d = D[py, px]
            w = eye[None, :] - pts
            b = w @ d
            disc = b * b - ((w * w).sum(1) - psi)
            m = disc > 0
            sq = np.sqrt(disc[m])
            iv = sorted(zip(-b[m] - sq, -b[m] + sq))
            tot, cov = 0.0, -np.inf
            for a, e in iv:
                lo = max(a, cov)
                if e > lo:
                    tot += e - lo
                cov = max(cov, e)
            nz += tot > 0
            assert abs(dp[py, px] - tot) <= 1e-11, (py, px, dp[py, px], tot)
    assert nz > 200
    img = render.render(pts, psi, cam, "depth")
    assert img.shape == (36, 48, 3) and img.max() == 255


def test_smooth_sdf_properties():
    """smooth_sdf (SPEC examples): a single sphere is the exact sphere SDF;
    k -> 0 is the plain min; the smooth union is <= the plain min, and at the
    midpoint of two overlapping spheres <= both distances."""
    import torch

    from paper_2601_05765_b200 import render

    rng = np.random.default_rng(3)
    p0, r0 = np.array([0.5, 0.5, 0.5]), 0.1
    x = p0 + (rng.random((800, 3)) - 0.5) * 0.35
    x = x[np.linalg.norm(x - p0, axis=1) < 0.18]  # within the sphere's neighbourhood (grid reach)
    f = render.smooth_sdf(x, p0[None, :], np.array([r0 * r0]), k=0.05).cpu().numpy()
    assert np.max(np.abs(f - (np.linalg.norm(x - p0, axis=1) - r0))) <= 1e-13

    n = 60
    pts = 0.3 + 0.4 * rng.random((n, 3))
    psi = (0.04 + 0.03 * rng.random(n)) ** 2
    x = 0.3 + 0.4 * rng.random((2000, 3))
    dist = np.linalg.norm(x[:, None, :] - pts[None, :, :], axis=2) - np.sqrt(psi)[None, :]
    plain = dist.min(1)
    f0 = render.smooth_sdf(x, pts, psi, k=1e-9).cpu().numpy()
    near = plain < 0.02  # the field is exact within the grid neighbourhood, a lower bound beyond
    assert near.sum() > 500
    assert np.max(np.abs(f0 - plain)[near]) <= 1e-9
    fk = render.smooth_sdf(x, pts, psi, k=0.03).cpu().numpy()
    assert np.all(fk <= plain + 1e-15)
    assert np.any(fk < plain - 1e-4)

    two = np.array([[0.45, 0.5, 0.5], [0.55, 0.5, 0.5]])
    w2 = np.array([0.07 ** 2, 0.07 ** 2])
    mid = torch.tensor([[0.5, 0.5, 0.5]], dtype=torch.float64)
    fm = float(render.smooth_sdf(mid, two, w2, k=0.05)[0])
    dm = 0.05 - 0.07
    assert fm <= dm and fm < dm - 1e-6


def test_smooth_mode_tends_to_raw_as_k_vanishes(tmp_path):
    """Raw vs Smooth at k -> 0 differ on < 0.5% of pixels (SPEC render example),
    and the traced hits sit on the Raw hits within the surface eps."""
    from paper_2601_05765_b200 import render

    rng = np.random.default_rng(4)
    n = 200
    pts = 0.25 + 0.5 * rng.random((n, 3))
    psi = (0.03 + 0.04 * rng.random(n)) ** 2
    cam = render.Camera(eye=(0.5, -1.2, 0.7), look_at=(0.5, 0.5, 0.45), fov=0.7, width=96, height=72)
    ids, raw_t = render.first_hit(pts, psi, cam)
    st, nrm = render.smooth_hit(pts, psi, cam, k=1e-9)
    raw_t, st = raw_t.cpu().numpy(), st.cpu().numpy()
    diff = (raw_t >= 0) != (st >= 0)
    assert diff.mean() < 0.005
    both = (raw_t >= 0) & (st >= 0)
    eps = 1e-4 * np.sqrt(3.0)
    assert np.max(np.abs(raw_t[both] - st[both])) <= 4.5 * eps  # start 4 eps before the Raw hit
    nn = np.linalg.norm(nrm.cpu().numpy()[both], axis=-1)
    assert np.all(np.abs(nn - 1) < 1e-9)
    img = render.render(pts, psi, cam, "smooth", k=0.02)
    render.write_ppm(str(tmp_path / "smooth.ppm"), img)
    assert img.shape == (72, 96, 3)


def test_sample_surface_lone_and_half_ball(tmp_path):
    """sample_surface (SPEC examples): a lone ball's samples lie on its sphere
    with normals (x - p)/r and their mean is the centre within 3 sigma; a ball
    cut by a wall gets no sample outside the domain."""
    from paper_2601_05765_b200 import render

    p0, r0 = np.array([0.5, 0.5, 0.5]), 0.1
    N = 10_000
    x, nrm, cell = render.sample_surface(p0[None, :], np.array([r0 * r0]), N, seed=7)
    x, nrm = x.cpu().numpy(), nrm.cpu().numpy()
    assert x.shape == (N, 3) and np.all(cell.cpu().numpy() == 0)
    assert np.max(np.abs(np.linalg.norm(x - p0, axis=1) - r0)) <= 1e-14
    assert np.max(np.abs(nrm - (x - p0) / r0)) <= 1e-12
    sig = r0 / np.sqrt(3.0 * N)
    assert np.all(np.abs(x.mean(0) - p0) <= 3 * sig)
    render.write_point_cloud(str(tmp_path / "s.xyz"), x[:10], nrm[:10])
    assert len(open(tmp_path / "s.xyz").read().splitlines()) == 10

    ph = np.array([[0.04, 0.5, 0.5]])
    x, _, _ = render.sample_surface(ph, np.array([r0 * r0]), 4000, seed=8)
    x = x.cpu().numpy()
    assert np.all(x[:, 0] >= 0.0)
    # the cap outside x < 0 is removed: the share of samples near the wall plane
    # matches the remaining cap area, not the full sphere
    assert x[:, 0].min() < 0.005


def test_sample_surface_membership_and_cell_counts():
    """Random overlapping scene: every sample lies on its sphere, strictly inside
    no other ball and inside the domain; per-cell counts follow |K_i| (z-scores
    of the multinomial within 5)."""
    import torch

    from paper_2601_05765_b200 import geom, render, restricted

    rng = np.random.default_rng(6)
    n = 150
    pts = 0.15 + 0.7 * rng.random((n, 3))
    psi = (0.04 + 0.04 * rng.random(n)) ** 2
    dom = geom.box_domain([0, 0, 0], [1, 1, 1])
    K = restricted.evaluate(torch.as_tensor(pts, device="cuda"), torch.as_tensor(psi, device="cuda"), dom).ksur
    K = K.cpu().numpy()
    N = 60_000
    x, nrm, cell = render.sample_surface(pts, psi, N, ksur=K, seed=9)
    x, cell = x.cpu().numpy(), cell.cpu().numpy()
    d2 = ((x[:, None, :] - pts[None, :, :]) ** 2).sum(-1)
    own = d2[np.arange(N), cell]
    assert np.max(np.abs(own - psi[cell])) <= 1e-14
    d2[np.arange(N), cell] = np.inf
    assert np.all(d2 >= psi[None, :] * (1 - 1e-12))
    assert np.all((x >= 0) & (x <= 1))
    cnt = np.bincount(cell, minlength=n)
    pr = K / K.sum()
    z = (cnt - N * pr) / np.sqrt(np.maximum(N * pr * (1 - pr), 1e-300))
    assert np.max(np.abs(z[pr > 0])) < 5.0
    assert np.all(cnt[pr == 0] == 0)
