"""CPU: host-side pieces — the C-ABI library loads and exports exactly what
include/csfs_b200.h declares, the Python mirror of the reference API behaves like the
reference (argument meaning, defaults, error messages), the product fails loudly
without a GPU, and the input generators reproduce the reference's grids bitwise."""
import ctypes
import os
import re

import numpy as np
import pytest

from oracle import ref
from paper_2508_13550_b200 import Kernel, KernelKind, SalParams, TraversalConfig, configs, engine
from paper_2508_13550_b200.grids import cubed_sphere, real_sph_harm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "csfs_b200.h")).read()
    return sorted(set(re.findall(r"CSFS_B200_API\s+[\w\s\*]+?\b(csfs_b200_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 18
    lib = ctypes.CDLL(engine.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in include/csfs_b200.h but not exported"


def test_library_hides_internal_symbols():
    out = os.popen(f"nm -D --defined-only {engine.LIB_PATH}").read()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert exported == set(header_symbols())


def test_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        engine.Engine(0)


def test_reference_api_mirror():
    assert Kernel.parse("laplace").kind == KernelKind.Laplace
    assert Kernel.parse("biot_savart").out_dim() == 3
    assert not Kernel.parse("biharmonic").singular_at_coincidence()
    with pytest.raises(ValueError, match="unknown kernel: fmm3d"):
        Kernel.parse("fmm3d")
    cfg = TraversalConfig()
    assert (cfg.mac, cfg.degree, cfg.n0, cfg.shrink) == (0.7, 6, -1, True)  # summation.hpp:22-31
    assert cfg.resolved_n0() == 144
    assert TraversalConfig(degree=10, n0=256).resolved_n0() == 256
    s = SalParams()
    assert (s.a1, s.b0, s.b1, s.rho_ratio) == (-2.7, -6.21196, 6.1, 1025.0 / 5517.0)  # kernels.hpp:18-23


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("level", [0, 3, 5, 8])
def test_cubed_sphere_matches_reference_bitwise(level):
    xyz, a = cubed_sphere(level)
    rx, ra = ref.grid("cubed_sphere", level)
    np.testing.assert_array_equal(xyz, rx)
    np.testing.assert_array_equal(a, ra)


def test_cubed_sphere_properties():
    xyz, a = cubed_sphere(5)
    assert xyz.shape == (6144, 3)
    np.testing.assert_allclose(np.linalg.norm(xyz, axis=1), 1.0, atol=1e-15)
    assert a.sum() == pytest.approx(4 * np.pi, rel=1e-12)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_real_sph_harm_matches_reference():
    xyz, _ = cubed_sphere(4)
    for l, m in [(1, 0), (4, 3), (7, -5), (32, 17), (20, -20)]:
        np.testing.assert_allclose(real_sph_harm(l, m, xyz), ref.sph_harm(l, m, xyz), rtol=1e-11, atol=1e-13)


def test_configs_deterministic_and_shaped():
    for name, n in [("c1", 6144), ("c2", 6 * 4 ** 5), ("c3", 6 * 4 ** 5), ("c4", 6 * 4 ** 5), ("c5", 6 * 4 ** 5)]:
        a = configs.make(name, level=None if name == "c1" else 5)
        b = configs.make(name, level=None if name == "c1" else 5)
        assert a.n == n
        np.testing.assert_array_equal(a.weights, b.weights)
    c3 = configs.make("c3", level=5)
    assert abs((c3.f * c3.areas).sum()) < 1e-12  # zero mean
    c5 = configs.make("c5", level=5)
    assert 0.65 < c5.meta["ocean_fraction"] < 0.75
    c1 = configs.make("c1")
    assert (c1.kernel, c1.degree, c1.mac, c1.n0) == ("laplace", 8, 0.7, 64)
    c5 = configs.make("c5", level=5)
    assert (c5.kernel, c5.degree, c5.mac, c5.n0) == ("sal", 10, 0.6, 256)


def test_log_table():
    """fastmath.cuh's accurate log table (tools/gen_log_table.c): 4096 intervals of m in
    [hi 0x3fe6a080, +2^20), r_i stored scaled by LAM = fl(1/sqrt 3); the interval holding
    m = 1 (mid-interval) is {LAM, 0}, elsewhere L_i on the 2^-46 grid within 2^-67 of
    -ln(r_i / LAM); |m r_i / LAM - 1| <= 2^-13 on every interval."""
    import struct
    from fractions import Fraction

    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.prec = 160
    src = open(os.path.join(ROOT, "paper_2508_13550_b200", "csrc", "log_table.inc")).read()
    ents = re.findall(r"\{(-?0x[0-9a-fp.+\-]+), (-?0x[0-9a-fp.+\-]+)\}", src)
    n, bits = 4096, 12
    w = 20 - bits
    assert len(ents) == n
    lam = float.fromhex("0x1.279a74590331cp-1")
    assert lam == float(1 / mpmath.sqrt(3))

    def from_hi(h):
        return struct.unpack(">d", struct.pack(">Q", h << 32))[0]

    for i, (a, b) in enumerate(ents):
        r, L = float.fromhex(a), float.fromhex(b)
        lo, hi = from_hi(0x3FE6A080 + (i << w)), from_hi(0x3FE6A080 + ((i + 1) << w))
        if lo <= 1.0 < hi:
            assert (r, L) == (lam, 0.0)
            continue
        assert (Fraction(L) * 2 ** 46).denominator == 1
        assert abs(-mpmath.log(mpmath.mpf(r) / mpmath.mpf(lam)) - mpmath.mpf(L)) < mpmath.mpf(2) ** -67
        rl = Fraction(r) / Fraction(lam)
        assert max(abs(Fraction(lo) * rl - 1), abs(Fraction(hi) * rl - 1)) <= Fraction(1, 8192) * (1 + Fraction(1, 1024))


def test_bve_mirror_defaults_and_sequencing():
    """BveState / BveStepOptions defaults (applications.hpp:58-83) and bve_step's order:
    RK4 step, time += dt, then the remesh only when options.remesh."""
    from paper_2508_13550_b200 import BveState, BveStepOptions, bve_step

    o = BveStepOptions()
    assert o.remesh is True and o.remesh_neighbors == 12 and o.traversal.mac == 0.7
    calls = []

    class Fake:
        def bve_step(self, x, z, a, omega, dt, cfg):
            calls.append(("step", dt, omega))
            return x + 1.0, z + 1.0, ["stats"] * 4

        def bve_remesh(self, x, z, g, t, nb):
            calls.append(("remesh", nb))
            return g.copy(), z * 2.0, t

    g = np.zeros((3, 3))
    st = BveState(positions=g + 0.5, zeta=np.ones(3), areas=np.ones(3), grid_centers=g)
    assert st.omega == 2.0 * np.pi and st.tracer is None
    bve_step(st, 0.25, BveStepOptions(remesh_neighbors=20), Fake())
    assert calls == [("step", 0.25, 2.0 * np.pi), ("remesh", 20)]
    np.testing.assert_array_equal(st.positions, g)
    np.testing.assert_array_equal(st.zeta, 4.0)
    assert st.time == 0.25
    calls.clear()
    bve_step(st, 0.25, BveStepOptions(remesh=False), Fake())
    assert calls == [("step", 0.25, 2.0 * np.pi)] and st.time == 0.5
