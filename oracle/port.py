"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of oracle/_build/libcsfmm_oracle.so, our C
restatement of the reference CSFMM (oracle/csfmm_oracle.c).  Pinned bitwise against the
reference library (oracle/_ref) and the committed golden fixtures by tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "_build", "libcsfmm_oracle.so")
KINDS = {"laplace": 0, "biharmonic": 1, "biot_savart": 2, "sal": 3}

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            import subprocess

            subprocess.run(["make", "-C", HERE, "port"], check=True, capture_output=True)
        L = C.CDLL(SO)
        P, L_, I, D = C.c_void_p, C.c_long, C.c_int, C.c_double
        L.port_csfmm.argtypes = [P, L_, P, P, L_, I, P, D, I, I, I, P, P]
        L.port_direct.argtypes = [P, L_, P, P, L_, I, P, P]
        L.port_tree_new.restype = P
        L.port_tree_new.argtypes = [P, L_, I, I, I]
        L.port_tree_free.argtypes = [P]
        L.port_tree_ncl.argtypes = [P]
        L.port_tree_depth.argtypes = [P]
        L.port_tree_export.argtypes = [P, P, P, P, P]
        L.port_upward.argtypes = [P, P, P]
        L.port_lists.argtypes = [P, P, D, I, P, P, P, P, P]
        L.port_dilog.restype = D
        L.port_dilog.argtypes = [D]
        L.port_kernel_eval.argtypes = [I, P, P, P, P]
        L.port_bary_basis_1d.argtypes = [I, D, P]
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _sal(sal):
    return None if sal is None else np.ascontiguousarray(sal, dtype=np.float64)


def csfmm(txyz, sxyz, sw, kernel, mac=0.7, degree=6, n0=-1, shrink=True, sal=None, counts=False):
    txyz = np.ascontiguousarray(txyz, dtype=np.float64)
    sxyz = np.ascontiguousarray(sxyz, dtype=np.float64)
    sw = np.ascontiguousarray(sw, dtype=np.float64)
    dim = 3 if kernel == "biot_savart" else 1
    out = np.empty(txyz.shape[0] * dim)
    cnt = np.zeros(4, np.int64)
    s4 = _sal(sal)
    rc = lib().port_csfmm(_p(txyz), txyz.shape[0], _p(sxyz), _p(sw), sxyz.shape[0], KINDS[kernel], _p(s4),
                          mac, degree, n0, 1 if shrink else 0, _p(out), _p(cnt))
    if rc:
        raise ValueError("invalid argument (reference: std::invalid_argument)")
    return (out, cnt) if counts else out


def direct(txyz, sxyz, sw, kernel, sal=None):
    txyz = np.ascontiguousarray(txyz, dtype=np.float64)
    sxyz = np.ascontiguousarray(sxyz, dtype=np.float64)
    sw = np.ascontiguousarray(sw, dtype=np.float64)
    dim = 3 if kernel == "biot_savart" else 1
    out = np.empty(txyz.shape[0] * dim)
    s4 = _sal(sal)
    lib().port_direct(_p(txyz), txyz.shape[0], _p(sxyz), _p(sw), sxyz.shape[0], KINDS[kernel], _p(s4), _p(out))
    return out


class Tree:
    def __init__(self, xyz, degree, n0, shrink=True):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        self.n, self.degree = xyz.shape[0], degree
        self.h = lib().port_tree_new(_p(xyz), self.n, degree, n0, 1 if shrink else 0)
        if not self.h:
            raise ValueError("invalid tree arguments")
        self.ncl = lib().port_tree_ncl(self.h)
        self.depth = lib().port_tree_depth(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().port_tree_free(self.h)

    def export(self) -> dict:
        npp = (self.degree + 1) ** 2
        perm = np.empty(self.n, np.int32)
        ints = np.empty((self.ncl, 10), np.int32)
        dbls = np.empty((self.ncl, 8))
        proxy = np.empty((self.ncl, npp, 3))
        lib().port_tree_export(self.h, _p(perm), _p(ints), _p(dbls), _p(proxy))
        return {"perm": perm, "ints": ints, "dbls": dbls, "proxy": proxy, "depth": self.depth}

    def upward(self, w) -> np.ndarray:
        w = np.ascontiguousarray(w, dtype=np.float64)
        pw = np.empty((self.ncl, (self.degree + 1) ** 2))
        lib().port_upward(self.h, _p(w), _p(pw))
        return pw


def lists(tt: Tree, ts: Tree, mac: float, n0: int) -> dict:
    counts = np.zeros(4, np.int64)
    lib().port_lists(tt.h, ts.h, mac, n0, _p(counts), None, None, None, None)
    bufs = [np.empty((int(counts[k]), 2), np.int32) for k in range(4)]
    lib().port_lists(tt.h, ts.h, mac, n0, _p(counts), *[_p(b) for b in bufs])
    return dict(zip(["pp", "pc", "cp", "cc"], bufs))


def dilog(x: float) -> float:
    return lib().port_dilog(float(x))


def kernel_eval(kernel, x, y, sal=None):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(3)
    ok = lib().port_kernel_eval(KINDS[kernel], _p(_sal(sal)), _p(x), _p(y), _p(out))
    return bool(ok), out


def bary_basis_1d(degree: int, x: float) -> np.ndarray:
    out = np.empty(degree + 1)
    lib().port_bary_basis_1d(degree, float(x), _p(out))
    return out
