"""Rendering of the fluid straight from the restricted diagram (SPEC.md:406-463
module `renderer`), all on the device
(csrc/pf_render.cu).  The fluid is the union of the restricted cells = the
union of the balls B(p_i, sqrt(psi_i)), so
  first_hit      smallest ball entry along the ray (the point lies in the
                 entered ball's Laguerre cell),
  depth          length of the ray inside the union of the balls (Depth mode),
  smooth_sdf     cubic smooth union of the sphere distances; Smooth mode
                 sphere-traces it (<= 64 steps, eps = 1e-4 x domain diagonal),
  sample_surface area-uniform points + normals on the free-surface patches K_i.
Raw shading: analytic normal (x - p_i)/|x - p_i|, one directional light,
Lambert; binary PPM (P6) output; point clouds as `x y z nx ny nz` text (SPEC
design decisions).  The cell-to-cell `traverse` of the SPEC is not needed by
these outputs (the union-of-balls identities above replace it) and is not built."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib


@dataclass
class Camera:
    eye: tuple
    look_at: tuple
    up: tuple = (0.0, 0.0, 1.0)
    fov: float = 0.8          # vertical field of view (rad)
    width: int = 640
    height: int = 480

    def packed(self) -> np.ndarray:
        e, t, u = (np.asarray(v, dtype=np.float64) for v in (self.eye, self.look_at, self.up))
        f = t - e
        f /= np.linalg.norm(f)
        r = np.cross(f, u)
        r /= np.linalg.norm(r)
        up = np.cross(r, f)
        return np.concatenate([e, f, r, up, [np.tan(0.5 * self.fov), self.width / self.height]])


def _bind():
    L = _lib.lib()
    if not getattr(L, "_render_bound", False):
        vp, i64, dbl, ci = C.c_void_p, C.c_int64, C.c_double, C.c_int
        L.pf_render_first_hit.argtypes = [vp, i64, vp, vp, dbl, vp, ci, ci, vp, vp, vp]
        L.pf_render_depth.argtypes = [vp, i64, vp, vp, dbl, vp, ci, ci, vp, vp]
        L.pf_render_smooth.argtypes = [vp, i64, vp, vp, dbl, dbl, dbl, vp, ci, ci, vp, vp, vp, vp]
        L.pf_smooth_sdf.argtypes = [vp, i64, vp, vp, dbl, dbl, i64, vp, vp, vp]
        L.pf_sample_surface.argtypes = [vp, i64, vp, vp, dbl, i64, vp, vp, C.c_uint64, vp, vp, vp, vp]
        L.pf_traverse.argtypes = [vp, i64, vp, vp, dbl, ci, vp, vp, vp, i64, vp, ci, ci, vp, vp, vp, vp, vp, vp, vp]
        for f in ("pf_render_first_hit", "pf_render_depth", "pf_render_smooth", "pf_smooth_sdf",
                  "pf_sample_surface", "pf_traverse"):
            getattr(L, f).restype = C.c_int
        L._render_bound = True
    return L


def _prep(pts, psi, domain):
    """device (pts, psi, rmax) with `domain` (default the unit box) uploaded: it
    bounds the bucket grid the rays walk and clips the surface samples"""
    import torch

    from .geom import box_domain
    from .laguerre import domain_pack, upload_domain

    dpk = domain_pack(domain if domain is not None else box_domain([0, 0, 0], [1, 1, 1]))
    upload_domain(_lib.ctx(), *dpk.args(), dpk.tol)
    p = torch.as_tensor(pts, dtype=torch.float64, device="cuda").contiguous()
    w = torch.as_tensor(psi, dtype=torch.float64, device="cuda").contiguous()
    rmax = float(w.clamp_min(0).max().sqrt()) if p.shape[0] else 0.0
    return p, w, rmax


def first_hit(pts, psi, cam: Camera, domain=None):
    """(hit_id int32[h, w] (-1: miss), hit_t f64[h, w]) for CUDA or numpy inputs."""
    import torch

    L = _bind()
    p, w, rmax = _prep(pts, psi, domain)
    ids = torch.empty((cam.height, cam.width), dtype=torch.int32, device="cuda")
    ts = torch.empty((cam.height, cam.width), dtype=torch.float64, device="cuda")
    cp = cam.packed()
    _lib.check(L.pf_render_first_hit(_lib.ctx(), p.shape[0], _lib.ptr(p), _lib.ptr(w), rmax,
                                     cp.ctypes.data_as(C.c_void_p), cam.width, cam.height, _lib.ptr(ids),
                                     _lib.ptr(ts), _lib.stream_ptr()), "pf_render_first_hit")
    return ids, ts


def depth(pts, psi, cam: Camera, domain=None):
    """In-fluid path length f64[h, w] of each pixel ray (SPEC Depth mode before
    normalisation): the length of the ray inside the union of the balls."""
    import torch

    L = _bind()
    p, w, rmax = _prep(pts, psi, domain)
    out = torch.empty((cam.height, cam.width), dtype=torch.float64, device="cuda")
    cp = cam.packed()
    _lib.check(L.pf_render_depth(_lib.ctx(), p.shape[0], _lib.ptr(p), _lib.ptr(w), rmax,
                                 cp.ctypes.data_as(C.c_void_p), cam.width, cam.height, _lib.ptr(out),
                                 _lib.stream_ptr()), "pf_render_depth")
    return out


class Traversal:
    """Per-ray pieces of a cell-to-cell traversal (SPEC renderer `traverse`):
    piece k < count[r] of ray r covers [t0[r, k], t1[r, k]] in power cell
    cell[r, k], inside the fluid when fluid[r, k]; consecutive pieces share
    end points.  status[r]: 0 ok, 1 the ray misses the domain, 2 the
    TraversalLoop guard (8 n facet crossings) or the piece capacity."""

    def __init__(self, cell, t0, t1, fluid, count, status):
        self.cell, self.t0, self.t1, self.fluid, self.count, self.status = cell, t0, t1, fluid, count, status

    def path(self, r: int):
        """[(cell id, t_enter, t_exit, in_fluid)] of ray r."""
        k = int(self.count[r])
        return [(int(self.cell[r, q]), float(self.t0[r, q]), float(self.t1[r, q]), bool(self.fluid[r, q]))
                for q in range(k)]

    def fluid_length(self):
        """In-fluid path length of every ray (SPEC Depth before normalisation)."""
        ln = (self.t1 - self.t0) * self.fluid
        k = np.arange(self.cell.shape[1])[None, :] < self.count[:, None]
        return (ln * k).sum(axis=1)


def traverse(pts, psi, origins, dirs, mode: str = "volume", max_segments: int = 256, domain=None,
             diagram=None) -> Traversal:
    """Cell-to-cell traversal of rays through the unrestricted power diagram
    (SPEC.md renderer `traverse`; §6: "load the current cell's
    neighbors and iteratively intersect facets facing the ray" until the
    domain boundary; "we explore the empty part of the domain through the
    unrestricted Laguerre diagram").  Within power cell i the fluid part of a
    ray is its chord of the ball B_i.  mode "volume" runs to the domain exit,
    "surface" stops after the first exit through a sphere patch.  ``diagram``:
    a laguerre.PackedDiagram in full mode (built here when None)."""
    import torch

    from .geom import box_domain
    from .laguerre import build_diagram_packed

    dom = domain if domain is not None else box_domain([0, 0, 0], [1, 1, 1])
    pts_h = np.ascontiguousarray(_host_np(pts), np.float64).reshape(-1, 3)
    psi_h = np.ascontiguousarray(_host_np(psi), np.float64).reshape(-1)
    if diagram is None:
        diagram = build_diagram_packed((pts_h, psi_h), dom, ball_aware=False)
    L = _bind()
    p, w, _ = _prep(pts_h, psi_h, dom)
    smf = int(diagram.planes.shape[1])
    nf = torch.as_tensor(np.where(diagram.status == 0, diagram.nf, 0).astype(np.int32), device="cuda")
    planes = torch.as_tensor(np.ascontiguousarray(diagram.planes), dtype=torch.float64, device="cuda")
    tags = torch.as_tensor(np.ascontiguousarray(diagram.tags).astype(np.int32), device="cuda")
    o = np.asarray(_host_np(origins), np.float64).reshape(-1, 3)
    d = np.asarray(_host_np(dirs), np.float64).reshape(-1, 3)
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    rays = torch.as_tensor(np.ascontiguousarray(np.concatenate([o, d], axis=1)), device="cuda")
    m = rays.shape[0]
    cell = torch.empty((m, max_segments), dtype=torch.int32, device="cuda")
    t0 = torch.empty((m, max_segments), dtype=torch.float64, device="cuda")
    t1 = torch.empty((m, max_segments), dtype=torch.float64, device="cuda")
    fl = torch.empty((m, max_segments), dtype=torch.uint8, device="cuda")
    cnt = torch.empty(m, dtype=torch.int32, device="cuda")
    st = torch.empty(m, dtype=torch.int32, device="cuda")
    psimax = float(psi_h.max()) if len(psi_h) else 0.0
    _lib.check(L.pf_traverse(_lib.ctx(), p.shape[0], _lib.ptr(p), _lib.ptr(w), psimax, smf, _lib.ptr(nf),
                             _lib.ptr(planes), _lib.ptr(tags), m, _lib.ptr(rays), 1 if mode == "surface" else 0,
                             int(max_segments), _lib.ptr(cell), _lib.ptr(t0), _lib.ptr(t1), _lib.ptr(fl),
                             _lib.ptr(cnt), _lib.ptr(st), _lib.stream_ptr()), "pf_traverse")
    return Traversal(cell.cpu().numpy(), t0.cpu().numpy(), t1.cpu().numpy(), fl.cpu().numpy().astype(bool),
                     cnt.cpu().numpy(), st.cpu().numpy())


def _host_np(x):
    try:
        import torch

        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
    except ImportError:
        pass
    return np.asarray(x)


def default_blend(psi) -> float:
    """SPEC open question: blend radius default 0.5 x the mean sphere radius."""
    import torch

    w = torch.as_tensor(psi, dtype=torch.float64)
    r = w[w > 0].sqrt()
    return 0.5 * float(r.mean()) if r.numel() else 1e-3


def _diag(domain) -> float:
    from .geom import box_domain
    from .laguerre import domain_pack

    v = domain_pack(domain if domain is not None else box_domain([0, 0, 0], [1, 1, 1])).args()[0]
    v = np.asarray(v).reshape(-1, 3)
    return float(np.linalg.norm(v.max(0) - v.min(0)))


def smooth_hit(pts, psi, cam: Camera, k: float | None = None, domain=None):
    """(hit_t f64[h, w] (-1 miss), normal f64[h, w, 3]) of the Smooth mode:
    sphere tracing of smooth_sdf, surface eps = 1e-4 x the domain diagonal."""
    import torch

    L = _bind()
    k = default_blend(psi) if k is None else float(k)
    _, raw_t = first_hit(pts, psi, cam, domain)
    p, w, rmax = _prep(pts, psi, domain)
    ts = torch.empty((cam.height, cam.width), dtype=torch.float64, device="cuda")
    nrm = torch.empty((cam.height, cam.width, 3), dtype=torch.float64, device="cuda")
    cp = cam.packed()
    _lib.check(L.pf_render_smooth(_lib.ctx(), p.shape[0], _lib.ptr(p), _lib.ptr(w), rmax, k, 1e-4 * _diag(domain),
                                  cp.ctypes.data_as(C.c_void_p), cam.width, cam.height, _lib.ptr(raw_t),
                                  _lib.ptr(ts), _lib.ptr(nrm), _lib.stream_ptr()), "pf_render_smooth")
    return ts, nrm


def smooth_sdf(x, pts, psi, k: float, domain=None):
    """SPEC smooth_sdf at points x[m, 3]: cubic smooth union of the sphere
    distances |x - p_j| - sqrt(psi_j) (plain min as k -> 0; <= the plain min)."""
    import torch

    L = _bind()
    p, w, rmax = _prep(pts, psi, domain)
    q = torch.as_tensor(x, dtype=torch.float64, device="cuda").reshape(-1, 3).contiguous()
    out = torch.empty(q.shape[0], dtype=torch.float64, device="cuda")
    _lib.check(L.pf_smooth_sdf(_lib.ctx(), p.shape[0], _lib.ptr(p), _lib.ptr(w), rmax, float(k), q.shape[0],
                               _lib.ptr(q), _lib.ptr(out), _lib.stream_ptr()), "pf_smooth_sdf")
    return out


class RejectionStall(RuntimeError):
    """A surface sample exhausted its draws (SPEC renderer errors)."""


def sample_surface(pts, psi, count: int, ksur=None, seed: int = 0, domain=None):
    """SPEC sample_surface: `count` points uniformly distributed by area over the
    free-surface patches K_i, with outward normals (x - p_i)/sqrt(psi_i).
    Per-cell counts are multinomial with probabilities |K_i| / sum |K|; cells
    with |K_i| / (4 pi psi_i) < 1e-6 are skipped (their area re-attributed).
    Each sample rejection-samples its sphere against the other balls and the
    domain on the device.  `ksur` (|K_i|) defaults to one restricted
    evaluation.  Returns (x f64[count, 3], normal f64[count, 3], cell int64[count])."""
    import torch

    L = _bind()
    p, w, rmax = _prep(pts, psi, domain)
    n = p.shape[0]
    if ksur is None:
        from . import restricted
        from .geom import box_domain

        ksur = restricted.evaluate(p, w, domain if domain is not None else box_domain([0, 0, 0], [1, 1, 1])).ksur
        p, w, rmax = _prep(pts, psi, domain)
    K = torch.as_tensor(ksur, dtype=torch.float64, device="cuda").clamp_min(0.0)
    frac = torch.where(w > 0, K / (4.0 * np.pi * w.clamp_min(1e-300)), torch.zeros_like(K))
    wt = torch.where(frac >= 1e-6, K, torch.zeros_like(K))
    x = torch.empty((count, 3), dtype=torch.float64, device="cuda")
    nrm = torch.empty((count, 3), dtype=torch.float64, device="cuda")
    if count == 0 or n == 0 or float(wt.sum()) <= 0.0:
        return x[:0], nrm[:0], torch.empty(0, dtype=torch.int64, device="cuda")
    gen = torch.Generator(device="cuda")
    gen.manual_seed(int(seed))
    cell = torch.multinomial(wt / wt.sum(), count, replacement=True, generator=gen)
    cell, _ = torch.sort(cell)
    tries = (64.0 / frac[cell]).ceil().clamp(64, 2 ** 40).to(torch.int64)
    st = torch.empty(count, dtype=torch.int32, device="cuda")
    _lib.check(L.pf_sample_surface(_lib.ctx(), n, _lib.ptr(p), _lib.ptr(w), rmax, count, _lib.ptr(cell),
                                   _lib.ptr(tries), int(seed) & (2 ** 64 - 1), _lib.ptr(x), _lib.ptr(nrm),
                                   _lib.ptr(st), _lib.stream_ptr()), "pf_sample_surface")
    if int(st.sum()):
        raise RejectionStall(f"{int(st.sum())} surface samples exhausted their draws")
    return x, nrm, cell


def write_point_cloud(path: str, x, normal) -> None:
    """plain-text point cloud, one `x y z nx ny nz` per line (SPEC External Interfaces)"""
    a = np.concatenate([np.asarray(x.cpu() if hasattr(x, "cpu") else x),
                        np.asarray(normal.cpu() if hasattr(normal, "cpu") else normal)], axis=1)
    np.savetxt(path, a, fmt="%.17g")


def _pixel_dirs(cam: Camera, dev):
    import torch

    cp = cam.packed()
    h, w = cam.height, cam.width
    xs = (2.0 * (torch.arange(w, device=dev, dtype=torch.float64) + 0.5) / w - 1.0) * cp[12] * cp[13]
    ys = (1.0 - 2.0 * (torch.arange(h, device=dev, dtype=torch.float64) + 0.5) / h) * cp[12]
    f, r, u = (torch.as_tensor(cp[a:a + 3], device=dev) for a in (3, 6, 9))
    d = f[None, None, :] + xs[None, :, None] * r[None, None, :] + ys[:, None, None] * u[None, None, :]
    return torch.as_tensor(cp[:3], device=dev), d / d.norm(dim=-1, keepdim=True)


def _shade(hit, nrm, d, light, color, background, fresnel=False):
    import torch

    lv = torch.as_tensor(light, dtype=torch.float64, device=nrm.device)
    lam = (nrm @ (lv / lv.norm())).clamp_min(0.0)
    shade = 0.25 + 0.75 * lam
    if fresnel:  # Schlick, F0 = 0.02 (water), as a white rim (cosmetic)
        cos = (-(nrm * d).sum(-1)).clamp(0.0, 1.0)
        fr = 0.02 + 0.98 * (1.0 - cos) ** 5
    img = torch.empty(hit.shape + (3,), dtype=torch.float64, device=nrm.device)
    for a in range(3):
        c = color[a] * shade
        if fresnel:
            c = c * (1.0 - fr) + 255.0 * fr
        img[..., a] = torch.where(hit, c, torch.full_like(shade, float(background[a])))
    return img.clamp(0, 255).round().to(torch.uint8).cpu().numpy()


def render_raw(pts, psi, cam: Camera, light=(0.3, -0.5, 0.8), color=(70, 130, 220),
               background=(245, 245, 245), domain=None) -> np.ndarray:
    """uint8 [h, w, 3] image: Lambert-shaded first hits (analytic normals
    (x - p_i)/|x - p_i|), background elsewhere."""
    import torch

    ids, ts = first_hit(pts, psi, cam, domain)
    eye, d = _pixel_dirs(cam, ids.device)
    P = torch.as_tensor(pts, dtype=torch.float64, device=ids.device)
    x = eye + ts[..., None] * d
    nrm = x - P[ids.clamp_min(0).long()]
    nrm = nrm / nrm.norm(dim=-1, keepdim=True).clamp_min(1e-300)
    return _shade(ids >= 0, nrm, d, light, color, background)


def render_depth(pts, psi, cam: Camera, domain=None, scale: float | None = None) -> np.ndarray:
    """uint8 [h, w, 3] Depth image: in-fluid path length normalised by `scale`
    (default the image maximum), white = longest; diagnostic pixels magenta."""
    import torch

    dp = depth(pts, psi, cam, domain)
    bad = dp < 0
    s = float(dp.max()) if scale is None else float(scale)
    v = (dp.clamp_min(0.0) / s if s > 0 else torch.zeros_like(dp)).clamp(0, 1) * 255.0
    img = torch.stack([v, v, v], -1)
    img[bad] = torch.tensor([255.0, 0.0, 255.0], dtype=torch.float64, device=img.device)
    return img.round().to(torch.uint8).cpu().numpy()


def render_smooth(pts, psi, cam: Camera, k: float | None = None, light=(0.3, -0.5, 0.8), color=(70, 130, 220),
                  background=(245, 245, 245), domain=None) -> np.ndarray:
    """uint8 [h, w, 3] Smooth image: sphere-traced smooth union, Lambert +
    Schlick Fresnel (non-normative shading)."""
    ts, nrm = smooth_hit(pts, psi, cam, k, domain)
    _, d = _pixel_dirs(cam, ts.device)
    return _shade(ts >= 0, nrm, d, light, color, background, fresnel=True)


def render(pts, psi, cam: Camera, mode: str = "raw", **kw) -> np.ndarray:
    """SPEC render(state, camera, mode: Raw | Smooth | Depth) -> Image"""
    m = mode.lower()
    if m == "raw":
        return render_raw(pts, psi, cam, **kw)
    if m == "depth":
        return render_depth(pts, psi, cam, **kw)
    if m == "smooth":
        return render_smooth(pts, psi, cam, **kw)
    raise ValueError(f"unknown render mode {mode!r} (raw | smooth | depth)")


def write_ppm(path: str, img: np.ndarray) -> None:
    h, w, _ = img.shape
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode())
        fh.write(np.ascontiguousarray(img, dtype=np.uint8).tobytes())
