"""The five BASELINE.json workloads as seeded synthetic inputs (host numpy arrays).

Inputs follow SURVEY.md §8(d): cubed-sphere cell centres and exact areas from
``grids.cubed_sphere`` (the reference's build_grid, geometry.cpp:97-123), weights
w_j = f(x_j) A_j.  BASELINE.json leaves several choices open (which harmonics, the
bump centre, the ocean mask); they are fixed here with seed 25081355 and recorded in
DESIGN.md.  Targets == sources in every config.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .grids import cubed_sphere, real_sph_harm

SEED = 25081355
# Rossby-Haurwitz wave 4 with omega = K = 7.848e-6 1/s, in the reference's day units
K_RH_PER_DAY = 7.848e-6 * 86400.0
OMEGA_EARTH_PER_DAY = 2.0 * np.pi  # BveState::omega default (applications.hpp:60)


@dataclass
class Workload:
    name: str
    level: int
    kernel: str  # laplace | biharmonic | biot_savart | sal
    degree: int
    mac: float
    n0: int
    xyz: np.ndarray
    areas: np.ndarray
    f: np.ndarray
    weights: np.ndarray
    exact: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return self.xyz.shape[0]


def rh4_zeta(p: np.ndarray, K: float = K_RH_PER_DAY, omega: float = K_RH_PER_DAY) -> np.ndarray:
    """Standard RH4 vorticity 2 w sin(lat) - K sin(lat) cos^4(lat) (R^2+3R+2) cos(4 lon),
    R = 4, with cos^4(lat) cos(4 lon) = x^4 - 6 x^2 y^2 + y^4 on the unit sphere."""
    x2, y2 = p[:, 0] ** 2, p[:, 1] ** 2
    return 2.0 * omega * p[:, 2] - K * 30.0 * p[:, 2] * (x2 * x2 - 6.0 * x2 * y2 + y2 * y2)


def make(name: str, level: int | None = None) -> Workload:
    """name in c1..c5; `level` overrides the grid level (for reduced-size parity cases)."""
    rng = np.random.Generator(np.random.MT19937(SEED))
    if name == "c1":
        L = 5 if level is None else level
        xyz, a = cubed_sphere(L)
        f = xyz[:, 0] * xyz[:, 1] * xyz[:, 2]
        # G_L = -(1/4pi) ln(1 - x.y) gives +f/12 for this degree-3 harmonic
        return Workload("c1", L, "laplace", 8, 0.7, 64, xyz, a, f, f * a, exact=f / 12.0)
    if name == "c2":
        L = 8 if level is None else level
        xyz, a = cubed_sphere(L)
        ls = rng.integers(1, 33, size=16)
        ms = np.array([rng.integers(-l, l + 1) for l in ls])
        cs = rng.standard_normal(16)
        f = np.zeros(xyz.shape[0])
        exact = np.zeros(xyz.shape[0])
        for l, m, c in zip(ls, ms, cs):
            y = real_sph_harm(int(l), int(m), xyz)
            f += c * y
            exact += c * y / (l * (l + 1.0))
        return Workload("c2", L, "laplace", 8, 0.7, 128, xyz, a, f, f * a, exact=exact,
                        meta={"harmonics": [(int(l), int(m), float(c)) for l, m, c in zip(ls, ms, cs)]})
    if name == "c3":
        L = 9 if level is None else level
        xyz, a = cubed_sphere(L)
        x0 = rng.standard_normal(3)
        x0 /= np.linalg.norm(x0)
        d = xyz - x0
        f = np.exp(-20.0 * np.einsum("ij,ij->i", d, d))
        f -= (f * a).sum() / a.sum()
        return Workload("c3", L, "biharmonic", 10, 0.6, 128, xyz, a, f, f * a, meta={"x0": x0.tolist()})
    if name == "c4":
        L = 9 if level is None else level
        xyz, a = cubed_sphere(L)
        z = rh4_zeta(xyz)
        z = z + 1e-3 * np.abs(z).max() * rng.standard_normal(z.shape[0])
        return Workload("c4", L, "biot_savart", 6, 0.7, 144, xyz, a, z, z * a,
                        meta={"dt_days": 0.01, "omega_per_day": OMEGA_EARTH_PER_DAY})
    if name == "c5":
        L = 10 if level is None else level
        xyz, a = cubed_sphere(L)
        mask = rng.random(xyz.shape[0]) < 0.7
        eta = rng.standard_normal(xyz.shape[0])
        f = np.where(mask, eta, 0.0)
        return Workload("c5", L, "sal", 10, 0.6, 256, xyz, a, f, f * a, meta={"ocean_fraction": float(mask.mean())})
    raise ValueError(f"unknown workload {name}")
