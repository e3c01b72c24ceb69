"""Python binding of the C-ABI (include/csfs_b200.h) — used by the tests and bench.py.

It mirrors the reference's C++ summation API (/root/reference/proj/include/csfs/
summation.hpp, kernels.hpp): ``Kernel`` / ``SalParams`` / ``TraversalConfig`` /
``SumStats`` / ``PotentialField`` and ``csfmm_sum`` / ``direct_sum`` /
``summed_potential``, with the same argument meaning and the same
``ValueError``-for-``std::invalid_argument`` behaviour and messages.  Every call goes
through libcsfs_b200.so; there is no CPU path — if the library or an sm_100 device is
missing, the call raises.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSFS_B200_LIB") or os.path.join(_HERE, "libcsfs_b200.so")

OK, INVALID_ARGUMENT, CUDA_ERROR, NCCL_ERROR, OUT_OF_MEMORY = 0, 1, 2, 3, 4


class KernelKind(enum.IntEnum):
    Laplace = 0
    Biharmonic = 1
    BiotSavart = 2
    Sal = 3


class Method(enum.IntEnum):
    Direct = 0
    Cstc = 1
    Csfmm = 2


_KIND_NAMES = {"laplace": KernelKind.Laplace, "biharmonic": KernelKind.Biharmonic,
               "biot_savart": KernelKind.BiotSavart, "sal": KernelKind.Sal}


@dataclass
class SalParams:  # kernels.hpp:18-23
    a1: float = -2.7
    b0: float = -6.21196
    b1: float = 6.1
    rho_ratio: float = 1025.0 / 5517.0


@dataclass
class Kernel:  # kernels.hpp:32-49
    kind: KernelKind = KernelKind.Laplace
    sal: SalParams = field(default_factory=SalParams)

    def out_dim(self) -> int:
        return 3 if self.kind == KernelKind.BiotSavart else 1

    def singular_at_coincidence(self) -> bool:
        return self.kind != KernelKind.Biharmonic

    def name(self) -> str:
        return {v: k for k, v in _KIND_NAMES.items()}[KernelKind(self.kind)]

    @staticmethod
    def parse(name: str, sal: SalParams | None = None) -> "Kernel":
        if name not in _KIND_NAMES:
            raise ValueError("unknown kernel: " + name)
        return Kernel(_KIND_NAMES[name], sal or SalParams())


@dataclass
class TraversalConfig:  # summation.hpp:22-31
    method: Method = Method.Csfmm
    mac: float = 0.7
    degree: int = 6
    n0: int = -1
    shrink: bool = True
    threads: int = 0  # accepted for API parity; the device decides its own parallelism

    def resolved_n0(self) -> int:
        return self.n0 if self.n0 >= 0 else 4 * self.degree * self.degree


class _CKernel(C.Structure):
    _fields_ = [("kind", C.c_int), ("a1", C.c_double), ("b0", C.c_double), ("b1", C.c_double),
                ("rho_ratio", C.c_double)]


class _CConfig(C.Structure):
    _fields_ = [("mac", C.c_double), ("degree", C.c_int), ("n0", C.c_int), ("shrink", C.c_int)]


class SumStats(C.Structure):  # summation.hpp:44-53 + B200 extras
    _fields_ = [("t_tree_build", C.c_double), ("t_upward", C.c_double), ("t_traversal", C.c_double),
                ("t_downward", C.c_double), ("t_total", C.c_double),
                ("pp", C.c_uint64), ("pc", C.c_uint64), ("cp", C.c_uint64), ("cc", C.c_uint64),
                ("src_depth", C.c_int), ("src_clusters", C.c_int), ("src_leaves", C.c_int),
                ("tgt_depth", C.c_int), ("tgt_clusters", C.c_int), ("tgt_leaves", C.c_int),
                ("t_lists", C.c_double), ("t_interact", C.c_double),
                ("evals_pp", C.c_uint64), ("evals_pc", C.c_uint64), ("evals_cp", C.c_uint64),
                ("evals_cc", C.c_uint64), ("shared_tree", C.c_int),
                ("evals_executed", C.c_uint64), ("symmetric_pairs", C.c_int),
                ("n_ranks", C.c_int), ("t_exchange", C.c_double), ("traversal_fallback", C.c_int),
                ("symmetric_partials", C.c_uint64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


@dataclass
class PotentialField:  # summation.hpp:34-41
    out_dim: int
    values: np.ndarray  # (n * out_dim,) target-major, input order

    def size(self) -> int:
        return self.values.size // self.out_dim


@dataclass
class ParticleSet:  # cluster_tree.hpp:13-18
    positions: np.ndarray  # (n, 3)
    weights: np.ndarray  # (n,)

    def size(self) -> int:
        return self.positions.shape[0]


_lib = None


def lib() -> C.CDLL:
    """Load libcsfs_b200.so (fails loudly when it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P, S, I, D = C.c_void_p, C.c_size_t, C.c_int, C.POINTER(C.c_double)
        L.csfs_b200_create.argtypes = [C.POINTER(P), I]
        L.csfs_b200_destroy.argtypes = [P]
        L.csfs_b200_last_error.argtypes = [P]
        L.csfs_b200_last_error.restype = C.c_char_p
        L.csfs_b200_csfmm.argtypes = [P, P, S, P, P, S, C.POINTER(_CKernel), C.POINTER(_CConfig), P,
                                      C.POINTER(SumStats)]
        L.csfs_b200_csfmm_device.argtypes = [P, P, S, P, P, S, C.POINTER(_CKernel), C.POINTER(_CConfig),
                                             P, C.POINTER(SumStats), P]
        L.csfs_b200_direct.argtypes = [P, P, S, P, P, S, C.POINTER(_CKernel), P]
        L.csfs_b200_cstc.argtypes = [P, P, S, P, P, S, C.POINTER(_CKernel), C.POINTER(_CConfig), P,
                                     C.POINTER(SumStats)]
        L.csfs_b200_cstc_device.argtypes = [P, P, S, P, P, S, C.POINTER(_CKernel), C.POINTER(_CConfig), P,
                                            C.POINTER(SumStats), P]
        L.csfs_b200_direct_device.argtypes = [P, P, S, P, P, S, C.POINTER(_CKernel), P, P]
        L.csfs_b200_tree_info.argtypes = [P, I, C.POINTER(I), C.POINTER(I), C.POINTER(S), C.POINTER(I)]
        L.csfs_b200_tree_export.argtypes = [P, I, P, P, P, P]
        L.csfs_b200_lists_export.argtypes = [P, C.POINTER(C.c_longlong), P, P, P, P]
        L.csfs_b200_proxy_weights_export.argtypes = [P, P]
        L.csfs_b200_kernel_launches.restype = C.c_uint64
        L.csfs_b200_kernel_launches.argtypes = []
        L.csfs_b200_probe_fp64.argtypes = [P, C.POINTER(C.c_double)]
        L.csfs_b200_part_plan.argtypes = [P, P, S, P, P, S, C.POINTER(_CKernel), C.POINTER(_CConfig), P]
        L.csfs_b200_part_units.argtypes = [P, I, C.POINTER(I), P, P, P]
        L.csfs_b200_bve_step.argtypes = [P, P, P, P, S, C.c_double, C.c_double, C.POINTER(_CConfig),
                                         C.POINTER(SumStats)]
        L.csfs_b200_bve_step_device.argtypes = [P, P, P, P, S, C.c_double, C.c_double, C.POINTER(_CConfig),
                                                C.POINTER(SumStats), P]
        L.csfs_b200_bve_remesh.argtypes = [P, P, P, P, P, S, I]
        L.csfs_b200_bve_remesh_device.argtypes = [P, P, P, P, P, S, I, P]
        L.csfs_b200_eval_pairs.argtypes = [P, C.POINTER(_CKernel), P, P, S, P]
        L.csfs_b200_eval_math.argtypes = [P, I, P, S, P]
        L.csfs_b200_part_sizes.argtypes = [P, C.POINTER(S), C.POINTER(S)]
        L.csfs_b200_part_upward.argtypes = [P, C.c_longlong, C.c_longlong, P]
        L.csfs_b200_part_eval.argtypes = [P, C.c_longlong, C.c_longlong, P, P]
        L.csfs_b200_part_finish.argtypes = [P, P, P]
        L.csfs_b200_create_multi.argtypes = [C.POINTER(P), I, P]
        L.csfs_b200_create_rank.argtypes = [C.POINTER(P), I, I, I, C.c_char_p]
        L.csfs_b200_create_emulated.argtypes = [C.POINTER(P), I, I]
        L.csfs_b200_nccl_unique_id.argtypes = [C.c_char_p]
        L.csfs_b200_group_info.argtypes = [P, C.POINTER(I), C.POINTER(I), P, P, P]
        L.csfs_b200_leaf_histogram.argtypes = [P, I, P, I, C.POINTER(I)]
        L.csfs_b200_group_phases.argtypes = [P, P, I, C.POINTER(I)]
        _lib = L
    return _lib


def _ptr(a: np.ndarray) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def _dptr(x) -> C.c_void_p:
    """Device pointer from a torch tensor (data_ptr) or a raw integer address."""
    return C.c_void_p(x.data_ptr() if hasattr(x, "data_ptr") else int(x))


def _ckernel(k: Kernel) -> _CKernel:
    return _CKernel(int(k.kind), k.sal.a1, k.sal.b0, k.sal.b1, k.sal.rho_ratio)


def _cconfig(c: TraversalConfig) -> _CConfig:
    return _CConfig(float(c.mac), int(c.degree), int(c.n0), 1 if c.shrink else 0)


NCCL_ID_BYTES = 128  # CSFS_B200_NCCL_ID_BYTES


def nccl_unique_id() -> bytes:
    """csfs_b200_nccl_unique_id: rank 0 makes it, the other ranks receive it (any channel)."""
    buf = C.create_string_buffer(NCCL_ID_BYTES)
    rc = lib().csfs_b200_nccl_unique_id(buf)
    if rc != OK:
        raise RuntimeError(f"csfs_b200_nccl_unique_id failed with code {rc}")
    return buf.raw


class Engine:
    """One csfs_b200_ctx: one device (default), or a multi-GPU group whose csfmm calls run
    the target-partitioned evaluation with NCCL exchanges (include/csfs_b200.h):

      Engine(device)                          one GPU
      Engine.multi(num_gpus, device_ids)      one process, N devices (ncclCommInitAll)
      Engine.rank(device, nranks, rank, id)   one process per GPU (torchrun), NCCL unique id
      Engine.emulated(device, nranks)         N ranks on one device (partition parity tests)
    """

    def __init__(self, device: int = 0, _handle=None):
        self._lib = lib()
        if _handle is None:
            h = C.c_void_p()
            rc = self._lib.csfs_b200_create(C.byref(h), int(device))
            if rc != OK:
                raise RuntimeError(f"csfs_b200_create(device={device}) failed with code {rc} "
                                   "(needs an sm_100 GPU; there is no CPU fallback)")
            _handle = h
        self._h = _handle
        self.device = device

    @classmethod
    def _made(cls, rc: int, h, device: int, what: str) -> "Engine":
        if rc != OK:
            raise RuntimeError(f"{what} failed with code {rc} (3 = NCCL error; needs sm_100 GPUs)")
        return cls(device, _handle=h)

    @classmethod
    def multi(cls, num_gpus: int, device_ids=None) -> "Engine":
        h = C.c_void_p()
        ids = None
        if device_ids is not None:
            ids = (C.c_int * num_gpus)(*[int(d) for d in device_ids])
        rc = lib().csfs_b200_create_multi(C.byref(h), int(num_gpus), ids)
        return cls._made(rc, h, int(device_ids[0]) if device_ids is not None else 0,
                         f"csfs_b200_create_multi({num_gpus})")

    @classmethod
    def rank(cls, device: int, nranks: int, rank: int, unique_id: bytes) -> "Engine":
        if len(unique_id) != NCCL_ID_BYTES:
            raise ValueError("the NCCL unique id has 128 bytes")
        h = C.c_void_p()
        rc = lib().csfs_b200_create_rank(C.byref(h), int(device), int(nranks), int(rank), unique_id)
        return cls._made(rc, h, device, f"csfs_b200_create_rank(rank {rank} of {nranks})")

    @classmethod
    def emulated(cls, device: int, nranks: int) -> "Engine":
        h = C.c_void_p()
        rc = lib().csfs_b200_create_emulated(C.byref(h), int(device), int(nranks))
        return cls._made(rc, h, device, f"csfs_b200_create_emulated({nranks})")

    def group_info(self) -> dict:
        n, r = C.c_int(), C.c_int()
        self._check(self._lib.csfs_b200_group_info(self._h, C.byref(n), C.byref(r), None, None, None))
        dev = np.empty(n.value, np.int32)
        self._check(self._lib.csfs_b200_group_info(self._h, None, None, _ptr(dev), None, None))
        info = {"nranks": n.value, "rank": r.value, "devices": dev.tolist()}
        tr = np.empty(2 * n.value, np.int64)
        sr = np.empty(2 * n.value, np.int64)
        if self._lib.csfs_b200_group_info(self._h, None, None, None, _ptr(tr), _ptr(sr)) == OK and n.value > 1:
            info["target_ranges"] = tr.reshape(-1, 2).tolist()
            info["source_ranges"] = sr.reshape(-1, 2).tolist()
        return info

    def group_phases(self) -> list[dict]:
        """Per-rank phases of the last partitioned call made with stats (csfs_b200_group_phases)."""
        n = C.c_int()
        self._check(self._lib.csfs_b200_group_phases(self._h, None, 0, C.byref(n)))
        v = np.empty(n.value)
        self._check(self._lib.csfs_b200_group_phases(self._h, _ptr(v), n.value, C.byref(n)))
        keys = ("plan_ms", "upward_ms", "interact_ms", "downward_ms", "finish_ms", "exchange_bytes")
        return [dict(zip(keys, v[i:i + 6].tolist())) for i in range(0, v.size, 6)]

    def leaf_histogram(self, which: int) -> list[int]:
        """TreeStats::leaf_size_histogram of the last call's target (0) / source (1) tree."""
        n = C.c_int()
        self._check(self._lib.csfs_b200_leaf_histogram(self._h, which, None, 0, C.byref(n)))
        h = np.zeros(n.value, np.int32)
        self._check(self._lib.csfs_b200_leaf_histogram(self._h, which, _ptr(h), n.value, C.byref(n)))
        return h.tolist()

    def close(self):
        if getattr(self, "_h", None):
            self._lib.csfs_b200_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc == OK:
            return
        msg = self._lib.csfs_b200_last_error(self._h).decode()
        if rc == INVALID_ARGUMENT:
            raise ValueError(msg)
        if rc == OUT_OF_MEMORY:
            raise MemoryError(msg)
        if rc == NCCL_ERROR:
            raise RuntimeError(f"csfs_b200 NCCL error: {msg}")
        raise RuntimeError(f"csfs_b200 error {rc}: {msg}")

    # --- reference API mirror --------------------------------------------------------
    def csfmm_sum(self, targets: ParticleSet, sources: ParticleSet, kernel: Kernel,
                  config: TraversalConfig, stats: SumStats | None = None,
                  out: np.ndarray | None = None) -> PotentialField:
        """`out` (optional, n*out_dim float64, e.g. a pinned buffer) receives the result."""
        tx = np.ascontiguousarray(targets.positions, dtype=np.float64)
        sx = tx if sources.positions is targets.positions else np.ascontiguousarray(sources.positions, dtype=np.float64)
        sw = np.ascontiguousarray(sources.weights, dtype=np.float64)
        if sw.shape[0] != sx.shape[0]:
            raise ValueError("weight count does not match particle count")
        if out is None:
            out = np.empty(tx.shape[0] * kernel.out_dim())
        assert out.dtype == np.float64 and out.flags.c_contiguous and out.size == tx.shape[0] * kernel.out_dim()
        st = stats if stats is not None else SumStats()
        self._check(self._lib.csfs_b200_csfmm(self._h, _ptr(tx), tx.shape[0], _ptr(sx), _ptr(sw), sx.shape[0],
                                              C.byref(_ckernel(kernel)), C.byref(_cconfig(config)), _ptr(out),
                                              C.byref(st)))
        return PotentialField(kernel.out_dim(), out)

    def direct_sum(self, targets: ParticleSet, sources: ParticleSet, kernel: Kernel,
                   threads: int = 0) -> PotentialField:
        tx = np.ascontiguousarray(targets.positions, dtype=np.float64)
        sx = np.ascontiguousarray(sources.positions, dtype=np.float64)
        sw = np.ascontiguousarray(sources.weights, dtype=np.float64)
        if sw.shape[0] != sx.shape[0]:
            raise ValueError("source weights and positions differ in length")
        out = np.empty(tx.shape[0] * kernel.out_dim())
        self._check(self._lib.csfs_b200_direct(self._h, _ptr(tx), tx.shape[0], _ptr(sx), _ptr(sw), sx.shape[0],
                                               C.byref(_ckernel(kernel)), _ptr(out)))
        return PotentialField(kernel.out_dim(), out)

    def cstc_sum(self, targets: ParticleSet, sources: ParticleSet, kernel: Kernel, config: TraversalConfig,
                 stats: SumStats | None = None) -> PotentialField:
        """csfs::cstc_sum (summation.cpp:308-381): the treecode."""
        tx = np.ascontiguousarray(targets.positions, dtype=np.float64)
        sx = tx if sources.positions is targets.positions else np.ascontiguousarray(sources.positions, dtype=np.float64)
        sw = np.ascontiguousarray(sources.weights, dtype=np.float64)
        if sw.shape[0] != sx.shape[0]:
            raise ValueError("weight count does not match the tree's particle count")
        out = np.empty(tx.shape[0] * kernel.out_dim())
        st = stats if stats is not None else SumStats()
        self._check(self._lib.csfs_b200_cstc(self._h, _ptr(tx), tx.shape[0], _ptr(sx), _ptr(sw), sx.shape[0],
                                             C.byref(_ckernel(kernel)), C.byref(_cconfig(config)), _ptr(out),
                                             C.byref(st)))
        return PotentialField(kernel.out_dim(), out)

    def summed_potential(self, targets, sources, kernel, config, stats=None) -> PotentialField:
        """summation.cpp:423-440: dispatch on config.method."""
        if config.method == Method.Direct:
            if stats is not None:
                import time

                t0 = time.perf_counter()
                f = self.direct_sum(targets, sources, kernel)
                for k, _ in SumStats._fields_:
                    setattr(stats, k, type(getattr(stats, k))())
                stats.t_traversal = stats.t_total = time.perf_counter() - t0
                stats.pp = targets.size() * sources.size()
                return f
            return self.direct_sum(targets, sources, kernel)
        if config.method == Method.Cstc:
            return self.cstc_sum(targets, sources, kernel, config, stats)
        return self.csfmm_sum(targets, sources, kernel, config, stats)

    # --- device-resident entry (torch tensors / raw device pointers) --------------------
    def csfmm_device(self, tgt_xyz_ptr: int, nt: int, src_xyz_ptr: int, src_w_ptr: int, ns: int,
                     kernel: Kernel, config: TraversalConfig, out_ptr: int, stream: int = 0,
                     stats: SumStats | None = None) -> SumStats:
        st = stats if stats is not None else SumStats()
        self._check(self._lib.csfs_b200_csfmm_device(
            self._h, C.c_void_p(tgt_xyz_ptr), nt, C.c_void_p(src_xyz_ptr), C.c_void_p(src_w_ptr), ns,
            C.byref(_ckernel(kernel)), C.byref(_cconfig(config)), C.c_void_p(out_ptr), C.byref(st),
            C.c_void_p(stream)))
        return st

    def direct_device(self, tgt_xyz_ptr, nt, src_xyz_ptr, src_w_ptr, ns, kernel, out_ptr, stream=0):
        self._check(self._lib.csfs_b200_direct_device(
            self._h, C.c_void_p(tgt_xyz_ptr), nt, C.c_void_p(src_xyz_ptr), C.c_void_p(src_w_ptr), ns,
            C.byref(_ckernel(kernel)), C.c_void_p(out_ptr), C.c_void_p(stream)))

    # --- stepwise exports of the last csfmm call ------------------------------------------
    def tree_info(self, which: int) -> tuple[int, int, int, int]:
        ncl, depth, npp = C.c_int(), C.c_int(), C.c_int()
        n = C.c_size_t()
        self._check(self._lib.csfs_b200_tree_info(self._h, which, C.byref(ncl), C.byref(depth), C.byref(n),
                                                  C.byref(npp)))
        return ncl.value, depth.value, n.value, npp.value

    def tree_export(self, which: int) -> dict:
        ncl, depth, n, npp = self.tree_info(which)
        perm = np.empty(n, np.int32)
        ints = np.empty((ncl, 10), np.int32)
        dbls = np.empty((ncl, 8))
        proxy = np.empty((ncl, npp, 3))
        self._check(self._lib.csfs_b200_tree_export(self._h, which, _ptr(perm), _ptr(ints), _ptr(dbls), _ptr(proxy)))
        return {"perm": perm, "ints": ints, "dbls": dbls, "proxy": proxy, "depth": depth}

    def lists_export(self) -> dict:
        counts = (C.c_longlong * 4)()
        self._check(self._lib.csfs_b200_lists_export(self._h, counts, None, None, None, None))
        bufs = [np.empty((max(counts[k], 0), 2), np.int32) for k in range(4)]
        self._check(self._lib.csfs_b200_lists_export(self._h, counts, *[_ptr(b) for b in bufs]))
        return dict(zip(["pp", "pc", "cp", "cc"], bufs))

    # --- barotropic vorticity RK4 step (applications.cpp:378-412, remesh off) ---------
    def bve_step(self, xyz: np.ndarray, zeta: np.ndarray, areas: np.ndarray, omega: float, dt: float,
                 config: TraversalConfig) -> tuple[np.ndarray, np.ndarray, list]:
        """Returns (new positions, new vorticity, per-stage SumStats); inputs untouched."""
        x = np.array(xyz, dtype=np.float64, order="C", copy=True)
        z = np.array(zeta, dtype=np.float64, copy=True)
        a = np.ascontiguousarray(areas, dtype=np.float64)
        st = (SumStats * 4)()
        self._check(self._lib.csfs_b200_bve_step(self._h, _ptr(x), _ptr(z), _ptr(a), x.shape[0], float(omega),
                                                 float(dt), C.byref(_cconfig(config)), st))
        return x, z, list(st)

    def bve_step_device(self, xyz, zeta, areas, n: int, omega: float, dt: float, config: TraversalConfig,
                        stream: int = 0) -> list:
        st = (SumStats * 4)()
        self._check(self._lib.csfs_b200_bve_step_device(self._h, _dptr(xyz), _dptr(zeta), _dptr(areas), n,
                                                        float(omega), float(dt), C.byref(_cconfig(config)), st,
                                                        C.c_void_p(stream)))
        return list(st)

    # --- multi-GPU partition phases (see distributed.py) ------------------------------
    def bve_remesh(self, xyz: np.ndarray, zeta: np.ndarray, grid: np.ndarray, tracer: np.ndarray | None = None,
                   neighbors: int = 12) -> tuple[np.ndarray, np.ndarray, np.ndarray | None]:
        """bve_remesh (applications.cpp:329-371) on the GPU: returns (positions = grid copy,
        fitted zeta, fitted tracer or None); inputs untouched."""
        x = np.array(xyz, dtype=np.float64, order="C", copy=True)
        z = np.array(zeta, dtype=np.float64, copy=True)
        t = None if tracer is None else np.array(tracer, dtype=np.float64, copy=True)
        g = np.ascontiguousarray(grid, dtype=np.float64)
        if g.shape != x.shape or z.shape[0] != x.shape[0] or (t is not None and t.shape[0] != x.shape[0]):
            raise ValueError("positions, zeta, tracer and grid centres must have one entry per particle")
        self._check(self._lib.csfs_b200_bve_remesh(self._h, _ptr(x), _ptr(z), _ptr(t) if t is not None else None,
                                                   _ptr(g), x.shape[0], int(neighbors)))
        return x, z, t

    def bve_remesh_device(self, xyz, zeta, tracer, grid, n: int, neighbors: int = 12, stream: int = 0):
        self._check(self._lib.csfs_b200_bve_remesh_device(self._h, _dptr(xyz), _dptr(zeta),
                                                          _dptr(tracer) if tracer is not None else None,
                                                          _dptr(grid), n, int(neighbors), C.c_void_p(stream)))

    def part_plan(self, tgt_xyz, nt, src_xyz, src_w, ns, kernel, config, stream=0):
        """Arguments are device tensors or raw device addresses."""
        self._check(self._lib.csfs_b200_part_plan(
            self._h, _dptr(tgt_xyz), nt, _dptr(src_xyz), _dptr(src_w), ns,
            C.byref(_ckernel(kernel)), C.byref(_cconfig(config)), C.c_void_p(stream)))

    def part_units(self, which: int):
        n = C.c_int()
        self._check(self._lib.csfs_b200_part_units(self._h, which, C.byref(n), None, None, None))
        b = np.empty(n.value, np.int64)
        e = np.empty(n.value, np.int64)
        c = np.empty(n.value)
        self._check(self._lib.csfs_b200_part_units(self._h, which, C.byref(n), _ptr(b), _ptr(e), _ptr(c)))
        return b, e, c

    def part_sizes(self) -> tuple[int, int]:
        a, b = C.c_size_t(), C.c_size_t()
        self._check(self._lib.csfs_b200_part_sizes(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def part_upward(self, b: int, e: int, pw):
        self._check(self._lib.csfs_b200_part_upward(self._h, b, e, _dptr(pw)))

    def part_eval(self, b: int, e: int, pw, phi):
        self._check(self._lib.csfs_b200_part_eval(self._h, b, e, _dptr(pw), _dptr(phi)))

    def part_finish(self, phi, out):
        self._check(self._lib.csfs_b200_part_finish(self._h, _dptr(phi), _dptr(out)))

    def eval_pairs(self, kernel: Kernel, x, y) -> np.ndarray:
        """Device functor values K(x_i, y_i) (guarded pairs -> 0), shape (n, out_dim)."""
        x = np.ascontiguousarray(x, dtype=np.float64).reshape(-1, 3)
        y = np.ascontiguousarray(y, dtype=np.float64).reshape(-1, 3)
        out = np.empty((x.shape[0], kernel.out_dim()))
        self._check(self._lib.csfs_b200_eval_pairs(self._h, C.byref(_ckernel(kernel)), _ptr(x), _ptr(y),
                                                   x.shape[0], _ptr(out)))
        return out

    def eval_math(self, fn: str, x) -> np.ndarray:
        """Device elementary function (log | rsqrt | rcp | dilog) on host values."""
        code = {"log": 0, "rsqrt": 1, "rcp": 2, "dilog": 3}[fn]
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(self._lib.csfs_b200_eval_math(self._h, code, _ptr(x), x.size, _ptr(out)))
        return out

    def probe_fp64_tflops(self) -> float:
        v = C.c_double()
        self._check(self._lib.csfs_b200_probe_fp64(self._h, C.byref(v)))
        return v.value

    def proxy_weights_export(self) -> np.ndarray:
        ncl, _, _, npp = self.tree_info(1)
        pw = np.empty((ncl, npp))
        self._check(self._lib.csfs_b200_proxy_weights_export(self._h, _ptr(pw)))
        return pw


def kernel_launches() -> int:
    """Engine kernels launched by this process so far."""
    return int(lib().csfs_b200_kernel_launches())


_default: Engine | None = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default


def csfmm_sum(targets, sources, kernel, config, stats=None) -> PotentialField:
    return default_engine().csfmm_sum(targets, sources, kernel, config, stats)


def direct_sum(targets, sources, kernel, threads=0) -> PotentialField:
    return default_engine().direct_sum(targets, sources, kernel, threads)


def summed_potential(targets, sources, kernel, config, stats=None) -> PotentialField:
    return default_engine().summed_potential(targets, sources, kernel, config, stats)


@dataclass
class BveState:  # applications.hpp:58-66
    positions: np.ndarray  # n x 3
    zeta: np.ndarray
    areas: np.ndarray
    grid_centers: np.ndarray
    tracer: np.ndarray | None = None
    omega: float = 2.0 * np.pi
    time: float = 0.0


@dataclass
class BveStepOptions:  # applications.hpp:79-83
    traversal: TraversalConfig = field(default_factory=TraversalConfig)
    remesh: bool = True
    remesh_neighbors: int = 12


def bve_remesh(state: BveState, neighbors: int = 12, engine: Engine | None = None) -> None:
    """applications.hpp:94: positions return to the grid centres, zeta/tracer are refitted."""
    e = engine or default_engine()
    state.positions, state.zeta, state.tracer = e.bve_remesh(state.positions, state.zeta, state.grid_centers,
                                                             state.tracer, neighbors)


def bve_step(state: BveState, dt: float, options: BveStepOptions | None = None,
             engine: Engine | None = None) -> list:
    """applications.hpp:89 / applications.cpp:378-412: one RK4 step (4 Biot-Savart CSFMM sums
    on the GPU), then the remesh when options.remesh.  Returns the per-stage SumStats."""
    o = options or BveStepOptions()
    e = engine or default_engine()
    state.positions, state.zeta, st = e.bve_step(state.positions, state.zeta, state.areas, state.omega, dt,
                                                 o.traversal)
    state.time += dt
    if o.remesh:
        bve_remesh(state, o.remesh_neighbors, e)
    return st
