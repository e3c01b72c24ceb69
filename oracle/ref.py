"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/_ref/libcsfs_ref.so, the
UNMODIFIED reference library (compiled by oracle/Makefile from /root/reference/proj/src)
plus oracle/ref_shim.cpp.  Only tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libcsfs_ref.so")
KINDS = {"laplace": 0, "biharmonic": 1, "biot_savart": 2, "sal": 3}
DEFAULT_SAL = (-2.7, -6.21196, 6.1, 1025.0 / 5517.0)

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{REF_SO} missing: run `make -C oracle ref` (needs /root/reference)")
        L = C.CDLL(REF_SO)
        P, S, I, D = C.c_void_p, C.c_size_t, C.c_int, C.c_double
        L.csref_last_error.restype = C.c_char_p
        L.csref_grid.restype = C.c_longlong
        L.csref_grid.argtypes = [I, I, P, P]
        L.csref_sum.argtypes = [I, P, S, P, P, S, I, P, D, I, I, I, I, P, P]
        L.csref_tree_new.restype = P
        L.csref_tree_new.argtypes = [P, S, I, I, I]
        L.csref_tree_free.argtypes = [P]
        L.csref_tree_ncl.argtypes = [P]
        L.csref_tree_depth.argtypes = [P]
        L.csref_tree_export.argtypes = [P, P, P, P, P, P, P]
        L.csref_upward.argtypes = [P, P, P]
        L.csref_lists.argtypes = [P, P, D, I, P, P, P, P, P]
        L.csref_dilog.restype = D
        L.csref_dilog.argtypes = [D]
        L.csref_kernel_try_eval.argtypes = [I, P, P, P, P]
        L.csref_bary_basis_1d.argtypes = [I, D, P]
        L.csref_face_project.argtypes = [P, P, P, P]
        L.csref_sph_harm_many.argtypes = [I, I, P, S, P]
        L.csref_rh_zeta_many.argtypes = [P, S, P]
        L.csref_bve_step.argtypes = [P, P, P, S, D, D, D, I, I, I]
        L.csref_bve_remesh.argtypes = [P, P, P, P, S, I]
        L.csref_read_particles.restype = C.c_longlong
        L.csref_read_particles.argtypes = [C.c_char_p, P, P]
        L.csref_bve_step_remesh.argtypes = [P, P, P, P, P, S, D, D, D, I, I, I, I]
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def grid(kind: str, level: int) -> tuple[np.ndarray, np.ndarray]:
    k = {"icosahedral": 0, "cubed_sphere": 1, "latlon": 2}[kind]
    n = lib().csref_grid(k, level, None, None)
    if n < 0:
        raise ValueError(lib().csref_last_error().decode())
    xyz, a = np.empty((n, 3)), np.empty(n)
    lib().csref_grid(k, level, _p(xyz), _p(a))
    return xyz, a


def read_particles_csv(path):
    """The reference's read_particles_csv: (xyz, weights), or raises ValueError("CODE: msg")."""
    n = lib().csref_read_particles(str(path).encode(), None, None)
    if n < 0:
        raise ValueError(lib().csref_last_error().decode())
    xyz, w = np.empty((n, 3)), np.empty(n)
    lib().csref_read_particles(str(path).encode(), _p(xyz), _p(w))
    return xyz, w


def _sal(sal):
    return np.array(sal if sal is not None else DEFAULT_SAL, dtype=np.float64)


def summed(method: int, txyz, sxyz, sw, kernel: str, mac=0.7, degree=6, n0=-1, shrink=True,
           threads=0, sal=None) -> tuple[np.ndarray, np.ndarray]:
    """method 0 direct, 1 cstc, 2 csfmm -> (values, stats[15])."""
    txyz = np.ascontiguousarray(txyz, dtype=np.float64)
    sxyz = np.ascontiguousarray(sxyz, dtype=np.float64)
    sw = np.ascontiguousarray(sw, dtype=np.float64)
    dim = 3 if kernel == "biot_savart" else 1
    out = np.empty(txyz.shape[0] * dim)
    st = np.zeros(16)
    s4 = _sal(sal)
    rc = lib().csref_sum(method, _p(txyz), txyz.shape[0], _p(sxyz), _p(sw), sxyz.shape[0], KINDS[kernel],
                         _p(s4), mac, degree, n0, 1 if shrink else 0, threads, _p(out), _p(st))
    if rc == 1:
        raise ValueError(lib().csref_last_error().decode())
    if rc:
        raise RuntimeError(lib().csref_last_error().decode())
    return out, st


def csfmm(txyz, sxyz, sw, kernel, **kw):
    return summed(2, txyz, sxyz, sw, kernel, **kw)


def direct(txyz, sxyz, sw, kernel, threads=0, sal=None):
    return summed(0, txyz, sxyz, sw, kernel, threads=threads, sal=sal)[0]


class Tree:
    """csfs::ClusterTree built by the reference (cluster_tree.cpp:29-147)."""

    def __init__(self, xyz, degree, n0, shrink=True):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.n = xyz.shape[0]
        self.degree = degree
        self.h = lib().csref_tree_new(_p(xyz), self.n, degree, n0, 1 if shrink else 0)
        if not self.h:
            raise ValueError(lib().csref_last_error().decode())
        self.ncl = lib().csref_tree_ncl(self.h)
        self.depth = lib().csref_tree_depth(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().csref_tree_free(self.h)

    def export(self) -> dict:
        np_ = self.degree + 1
        perm = np.empty(self.n, np.int32)
        ints = np.empty((self.ncl, 10), np.int32)
        dbls = np.empty((self.ncl, 8))
        proxy = np.empty((self.ncl, np_ * np_, 3))
        xi, eta = np.empty(self.n), np.empty(self.n)
        lib().csref_tree_export(self.h, _p(perm), _p(ints), _p(dbls), _p(proxy), _p(xi), _p(eta))
        return {"perm": perm, "ints": ints, "dbls": dbls, "proxy": proxy, "xi": xi, "eta": eta,
                "depth": self.depth}

    def upward(self, w) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64)
        np_ = self.degree + 1
        pw = np.empty((self.ncl, np_ * np_))
        lib().csref_upward(self.h, _p(w), _p(pw))
        return pw


def lists(tt: Tree, ts: Tree, mac: float, n0: int) -> dict:
    counts = np.zeros(4, np.int64)
    lib().csref_lists(tt.h, ts.h, mac, n0, _p(counts), None, None, None, None)
    bufs = [np.empty((int(counts[k]), 2), np.int32) for k in range(4)]
    lib().csref_lists(tt.h, ts.h, mac, n0, _p(counts), *[_p(b) for b in bufs])
    return dict(zip(["pp", "pc", "cp", "cc"], bufs))


def dilog(x: float) -> float:
    return lib().csref_dilog(float(x))


def kernel_try_eval(kernel: str, x, y, sal=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(3)
    ok = lib().csref_kernel_try_eval(KINDS[kernel], _p(_sal(sal)), _p(x), _p(y), _p(out))
    return bool(ok), out


def bary_basis_1d(degree: int, x: float) -> np.ndarray:
    out = np.empty(degree + 1)
    lib().csref_bary_basis_1d(degree, float(x), _p(out))
    return out


def sph_harm(l, m, xyz):
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    out = np.empty(xyz.shape[0])
    lib().csref_sph_harm_many(l, m, _p(xyz), xyz.shape[0], _p(out))
    return out


def bve_step(xyz, zeta, areas, omega, dt, mac=0.7, degree=6, n0=-1, threads=0):
    xyz = np.array(xyz, dtype=np.float64, order="C")
    zeta = np.array(zeta, dtype=np.float64)
    areas = np.ascontiguousarray(areas, dtype=np.float64)
    rc = lib().csref_bve_step(_p(xyz), _p(zeta), _p(areas), xyz.shape[0], omega, dt, mac, degree, n0, threads)
    if rc:
        raise RuntimeError(lib().csref_last_error().decode())
    return xyz, zeta


def bve_remesh(xyz, zeta, grid, tracer=None, neighbors=12):
    """The reference's bve_remesh (applications.cpp:329-371): returns (grid, zeta', tracer')."""
    xyz = np.array(xyz, dtype=np.float64, order="C")
    zeta = np.array(zeta, dtype=np.float64)
    tr = None if tracer is None else np.array(tracer, dtype=np.float64)
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    rc = lib().csref_bve_remesh(_p(xyz), _p(zeta), _p(tr), _p(grid), xyz.shape[0], neighbors)
    if rc:
        raise RuntimeError(lib().csref_last_error().decode())
    return xyz, zeta, tr


def bve_step_remesh(xyz, zeta, areas, grid, omega, dt, tracer=None, mac=0.7, degree=6, n0=-1, neighbors=12,
                    threads=0):
    """The reference's bve_step with remesh on (its default BveStepOptions)."""
    xyz = np.array(xyz, dtype=np.float64, order="C")
    zeta = np.array(zeta, dtype=np.float64)
    tr = None if tracer is None else np.array(tracer, dtype=np.float64)
    areas = np.ascontiguousarray(areas, dtype=np.float64)
    grid = np.ascontiguousarray(grid, dtype=np.float64)
    rc = lib().csref_bve_step_remesh(_p(xyz), _p(zeta), _p(tr), _p(areas), _p(grid), xyz.shape[0], omega, dt, mac,
                                     degree, n0, neighbors, threads)
    if rc:
        raise RuntimeError(lib().csref_last_error().decode())
    return xyz, zeta, tr
