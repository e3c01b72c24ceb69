"""Input generation for the benchmark configs (host side, numpy).

Restates the reference's cubed-sphere grid generator ``build_grid(CubedSphere, L)``
(/root/reference/proj/src/geometry.cpp:97-123) and the field helpers the configs use
(``real_sph_harm``, ``rossby_haurwitz_zeta``; applications.cpp:14-49, 148-153).  This is
input generation, not the hot path: the same arrays are handed to the B200 engine and to
the reference, so bitwise agreement with the reference's own generator is not needed
(tests/test_grids.py checks it anyway: centres and areas agree bit for bit).
"""
from __future__ import annotations

import math

import numpy as np

PI = 3.14159265358979323846


def face_point_from_plane(face: int, X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """geometry.cpp:37-48 (vectorised)."""
    s = 1.0 / np.sqrt((1.0 + X * X) + Y * Y)
    sX, sY = s * X, s * Y
    out = np.empty(X.shape + (3,))
    comps = {
        0: (s, sX, sY),
        1: (-sX, s, sY),
        2: (-s, -sX, sY),
        3: (sX, -s, sY),
        4: (-sY, sX, s),
        5: (sY, sX, -s),
    }[face]
    for k in range(3):
        out[..., k] = comps[k]
    return out


def _dot(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return (a[..., 0] * b[..., 0] + a[..., 1] * b[..., 1]) + a[..., 2] * b[..., 2]


def _cross(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    return np.stack(
        [
            a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
            a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
            a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0],
        ],
        axis=-1,
    )


def _tri_area(a, b, c):
    """spherical_triangle_area (geometry.cpp:70-74)."""
    num = _dot(a, _cross(b, c))
    den = ((1.0 + _dot(a, b)) + _dot(b, c)) + _dot(c, a)
    return 2.0 * np.arctan2(num, den)


def cubed_sphere(level: int) -> tuple[np.ndarray, np.ndarray]:
    """Cell centres (n x 3) and exact spherical areas (n) of the level-`level` equiangular
    cubed sphere, 6 * 4**level cells ordered face -> i (xi) -> j (eta) (geometry.cpp:97-123)."""
    m = 1 << level
    d = (PI / 2.0) / m
    # libm tan on the 1-D node sets (m + 1 values), as the reference does
    edge = np.array([math.tan(-PI / 4.0 + i * d) for i in range(m + 1)])
    tc = np.array([math.tan(-PI / 4.0 + (i + 0.5) * d) for i in range(m)])
    I, J = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
    centers, areas = [], []
    for f in range(6):
        centers.append(face_point_from_plane(f, tc[I], tc[J]).reshape(-1, 3))
        p00 = face_point_from_plane(f, edge[I], edge[J])
        p10 = face_point_from_plane(f, edge[I + 1], edge[J])
        p11 = face_point_from_plane(f, edge[I + 1], edge[J + 1])
        p01 = face_point_from_plane(f, edge[I], edge[J + 1])
        areas.append((_tri_area(p00, p10, p11) + _tri_area(p00, p11, p01)).reshape(-1))
    return np.ascontiguousarray(np.concatenate(centers)), np.concatenate(areas)


def _assoc_legendre(l: int, m: int, z: np.ndarray) -> np.ndarray:
    """P_l^m(z) without the Condon-Shortley phase (applications.cpp:14-34)."""
    pmm = np.ones_like(z)
    if m > 0:
        s = np.sqrt(np.maximum(0.0, 1.0 - z * z))
        fact = 1.0
        for _ in range(m):
            pmm = pmm * (fact * s)
            fact += 2.0
    if l == m:
        return pmm
    pmm1 = z * (2.0 * m + 1.0) * pmm
    if l == m + 1:
        return pmm1
    pll = pmm1
    for ll in range(m + 2, l + 1):
        pll = (z * (2.0 * ll - 1.0) * pmm1 - (ll + m - 1.0) * pmm) / (ll - m)
        pmm, pmm1 = pmm1, pll
    return pll


def real_sph_harm(l: int, m: int, p: np.ndarray) -> np.ndarray:
    """Orthonormal real spherical harmonic (applications.cpp:38-49)."""
    am = abs(m)
    ratio = 1.0
    for i in range(l - am + 1, l + am + 1):
        ratio /= float(i)
    norm = math.sqrt((2.0 * l + 1.0) / (4.0 * PI) * ratio)
    plm = _assoc_legendre(l, am, p[:, 2])
    if m == 0:
        return norm * plm
    lon = np.arctan2(p[:, 1], p[:, 0])
    trig = np.cos(am * lon) if m > 0 else np.sin(am * lon)
    return math.sqrt(2.0) * norm * plm * trig


def rossby_haurwitz_zeta(p: np.ndarray) -> np.ndarray:
    """applications.cpp:148-153: (2 pi/7) z + 30 z (x^4 - 6 x^2 y^2 + y^4)."""
    x2, y2 = p[:, 0] ** 2, p[:, 1] ** 2
    return (2.0 * PI / 7.0) * p[:, 2] + 30.0 * p[:, 2] * (x2 * x2 - 6.0 * x2 * y2 + y2 * y2)
