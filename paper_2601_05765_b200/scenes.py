"""Synthetic seed clouds of the benchmark configurations.

All scenes live in the unit box [0,1]^3 and use numpy.random.default_rng with
the seeds the survey fixes, so the CPU oracle, the reference and the device
path see identical inputs.

C1  10k random seeds, 30% fill                       (BASELINE.json configs[0])
C2  100k dam break: 46^3 jittered lattice in [0,1/2]^3 (configs[1])
C3  500k "chocs": uniform ball of radius 1/4, radial velocity (configs[2])
C4  2M droplet: pool z in [0,0.08] + drop r=0.12 at (.5,.5,.35) (configs[3])
C5  1M two-fluid: spacing h (z<0.25) and 2h (0.25<z<0.5)   (configs[4])
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Scene:
    name: str
    pts: np.ndarray          # [n,3]
    nu: np.ndarray           # [n] prescribed volumes
    vel: np.ndarray          # [n,3]
    rho: np.ndarray          # [n] mass density
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return len(self.pts)

    def psi_cold(self, kappa: float = 1.0) -> np.ndarray:
        """Cold-start weights kappa (3 nu / 4 pi)^(2/3)."""
        return kappa * (3.0 * self.nu / (4.0 * np.pi)) ** (2.0 / 3.0)


def _lattice(m_xyz, lo, h, rng, jitter=0.05):
    axes = [lo[a] + (np.arange(m_xyz[a]) + 0.5) * h for a in range(3)]
    P = np.stack(np.meshgrid(*axes, indexing="ij"), -1).reshape(-1, 3)
    return P + rng.uniform(-jitter * h, jitter * h, P.shape)


def c1_random(n: int = 10_000, fill: float = 0.3, seed: int = 12345) -> Scene:
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 3))
    nu = np.full(n, fill / n)
    return Scene("C1-random", pts, nu, np.zeros((n, 3)), np.full(n, 1000.0), {"fill": fill})


def c2_dam_break(m: int = 46, seed: int = 7) -> Scene:
    rng = np.random.default_rng(seed)
    h = 0.5 / m
    pts = _lattice((m, m, m), (0.0, 0.0, 0.0), h, rng)
    n = len(pts)
    return Scene("C2-dam-break", pts, np.full(n, h ** 3), np.zeros((n, 3)), np.full(n, 1000.0),
                 {"h": h, "m": m, "dt": 1e-3, "eps": 5e-3, "g": (0.0, 0.0, -9.81)})


def c3_chocs(n: int = 500_000, radius: float = 0.25, seed: int = 3) -> Scene:
    rng = np.random.default_rng(seed)
    c = np.array([0.5, 0.5, 0.5])
    out = []
    need = n
    while need > 0:
        x = rng.uniform(-radius, radius, (int(need * 2.1) + 16, 3))
        x = x[np.einsum("ij,ij->i", x, x) <= radius * radius]
        out.append(x[:need])
        need -= len(out[-1])
    pts = c + np.concatenate(out)[:n]
    nu = np.full(n, (4.0 / 3.0) * np.pi * radius ** 3 / n)
    vel = 5.0 * (pts - c) / radius
    return Scene("C3-chocs", pts, nu, vel, np.full(n, 1000.0), {"dt": 1e-3})


def c4_droplet(n_target: int = 2_000_000, seed: int = 11) -> Scene:
    rng = np.random.default_rng(seed)
    h = (0.0872 / n_target) ** (1.0 / 3.0)
    m = int(np.floor(1.0 / h))
    mz = int(np.floor(0.08 / h))
    pool = _lattice((m, m, mz), (0.0, 0.0, 0.0), h, rng)
    r, c = 0.12, np.array([0.5, 0.5, 0.35])
    k = int(np.ceil(2 * r / h))
    cube = _lattice((k, k, k), tuple(c - r), h, rng)
    drop = cube[np.linalg.norm(cube - c, axis=1) <= r]
    pts = np.concatenate([pool, drop])
    n = len(pts)
    vel = np.zeros((n, 3))
    vel[len(pool):, 2] = -3.0
    return Scene("C4-droplet", pts, np.full(n, h ** 3), vel, np.full(n, 1000.0), {"h": h})


def c5_two_fluid(n_target: int = 1_000_000, seed: int = 5) -> Scene:
    rng = np.random.default_rng(seed)
    # n_A + n_B = (1/h)^2 (0.25/h) + (1/2h)^2 (0.25/2h) = (0.25 + 0.25/8) / h^3
    h = ((0.25 + 0.25 / 8.0) / n_target) ** (1.0 / 3.0)
    mA, mzA = int(np.floor(1.0 / h)), int(np.floor(0.25 / h))
    A = _lattice((mA, mA, mzA), (0.0, 0.0, 0.0), h, rng)
    hB = 2.0 * h
    mB, mzB = int(np.floor(1.0 / hB)), int(np.floor(0.25 / hB))
    B = _lattice((mB, mB, mzB), (0.0, 0.0, 0.25), hB, rng)
    pts = np.concatenate([A, B])
    nu = np.concatenate([np.full(len(A), h ** 3), np.full(len(B), hB ** 3)])
    rho = np.concatenate([np.full(len(A), 1000.0), np.full(len(B), 100.0)])
    return Scene("C5-two-fluid", pts, nu, np.zeros((len(pts), 3)), rho, {"h": h, "nA": len(A)})


CONFIGS = {
    "C1": c1_random,
    "C2": c2_dam_break,
    "C3": c3_chocs,
    "C4": c4_droplet,
    "C5": c5_two_fluid,
}


def make(name: str, **kw) -> Scene:
    return CONFIGS[name](**kw)
