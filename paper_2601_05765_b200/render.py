"""First-hit rendering of the fluid (SPEC.md:406-463 `first_hit` / `render`
Raw mode).  One ray per pixel on the
device (pf_render_first_hit): the fluid is the union of the restricted cells
= the union of the balls B(p_i, sqrt(psi_i)), and the first point of that
union along a ray lies on the entered ball's sphere inside its Laguerre cell.
Raw shading: analytic normal (x - p_i)/|x - p_i|, one directional light,
Lambert; binary PPM (P6) output (SPEC design decision)."""
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


def first_hit(pts, psi, cam: Camera, domain=None):
    """(hit_id int32[h, w] (-1: miss), hit_t f64[h, w]) for CUDA or numpy inputs;
    `domain` (default the unit box) bounds the bucket grid the rays walk."""
    import torch

    from .geom import box_domain
    from .laguerre import domain_pack, upload_domain

    L = _lib.lib()
    dpk = domain_pack(domain if domain is not None else box_domain([0, 0, 0], [1, 1, 1]))
    upload_domain(_lib.ctx(), *dpk.args(), dpk.tol)
    if not getattr(L, "_render_bound", False):
        vp = C.c_void_p
        L.pf_render_first_hit.argtypes = [vp, C.c_int64, vp, vp, C.c_double, vp, C.c_int, C.c_int, vp, vp, vp]
        L.pf_render_first_hit.restype = C.c_int
        L._render_bound = True
    p = torch.as_tensor(pts, dtype=torch.float64, device="cuda").contiguous()
    w = torch.as_tensor(psi, dtype=torch.float64, device="cuda").contiguous()
    n = p.shape[0]
    ids = torch.empty((cam.height, cam.width), dtype=torch.int32, device="cuda")
    ts = torch.empty((cam.height, cam.width), dtype=torch.float64, device="cuda")
    rmax = float(w.clamp_min(0).max().sqrt()) if n else 0.0
    cp = cam.packed()
    _lib.check(L.pf_render_first_hit(_lib.ctx(), n, _lib.ptr(p), _lib.ptr(w), rmax,
                                     cp.ctypes.data_as(C.c_void_p), cam.width, cam.height, _lib.ptr(ids),
                                     _lib.ptr(ts), _lib.stream_ptr()), "pf_render_first_hit")
    return ids, ts


def render_raw(pts, psi, cam: Camera, light=(0.3, -0.5, 0.8), color=(70, 130, 220),
               background=(245, 245, 245), domain=None) -> np.ndarray:
    """uint8 [h, w, 3] image: Lambert-shaded first hits, background elsewhere."""
    import torch

    ids, ts = first_hit(pts, psi, cam, domain)
    cp = cam.packed()
    h, w = cam.height, cam.width
    dev = ids.device
    xs = (2.0 * (torch.arange(w, device=dev, dtype=torch.float64) + 0.5) / w - 1.0) * cp[12] * cp[13]
    ys = (1.0 - 2.0 * (torch.arange(h, device=dev, dtype=torch.float64) + 0.5) / h) * cp[12]
    f, r, u = (torch.as_tensor(cp[a:a + 3], device=dev) for a in (3, 6, 9))
    d = f[None, None, :] + xs[None, :, None] * r[None, None, :] + ys[:, None, None] * u[None, None, :]
    d = d / d.norm(dim=-1, keepdim=True)
    hit = ids >= 0
    P = torch.as_tensor(pts, dtype=torch.float64, device=dev)
    x = torch.as_tensor(cp[:3], device=dev) + ts[..., None] * d
    nrm = x - P[ids.clamp_min(0).long()]
    nrm = nrm / nrm.norm(dim=-1, keepdim=True).clamp_min(1e-300)
    lv = torch.as_tensor(light, dtype=torch.float64, device=dev)
    lam = (nrm @ (lv / lv.norm())).clamp_min(0.0)
    shade = 0.25 + 0.75 * lam
    img = torch.empty((h, w, 3), dtype=torch.float64, device=dev)
    for a in range(3):
        img[..., a] = torch.where(hit, color[a] * shade, torch.full_like(shade, float(background[a])))
    return img.clamp(0, 255).round().to(torch.uint8).cpu().numpy()


def write_ppm(path: str, img: np.ndarray) -> None:
    h, w, _ = img.shape
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode())
        fh.write(np.ascontiguousarray(img, dtype=np.uint8).tobytes())
