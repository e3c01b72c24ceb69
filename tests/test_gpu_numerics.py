"""GPU: the device elementary functions (fastmath.cuh) and kernel functors
(kernels_dev.cuh) against high-precision references and the reference's own
Kernel::try_eval values (golden fixtures, kernels.cpp / summation.cpp:32-77).
Tolerances: log <= 2 ulp + 2e-17 absolute (the truncated degree-3 log1p, <= 9.5e-18,
fastmath.cuh); rsqrt, rcp <= 1 ulp; dilog <= 4e-15 relative to the reference series (+ 2e-17
absolute); kernel values <= 8e-15 relative or 4e-17 absolute (a log enters every scalar
kernel), with identical guard decisions."""
import os

import numpy as np
import pytest

from paper_2508_13550_b200 import Kernel

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
LOG_ABS = 2e-17  # 0.043 h^4 at h = 2^-13 (9.5e-18, the truncated log1p term) + rounding


def test_fast_log(engine):
    rng = np.random.default_rng(3)
    x = np.concatenate([10 ** rng.uniform(-15, 0.35, 200000), 1 + rng.uniform(-1e-3, 1e-3, 20000),
                        [1e-14, 0.5, 1.0, 2.0, 1 - 2 ** -53, 1 + 2 ** -52]])
    got = engine.eval_math("log", x)
    want = np.log(x)  # numpy log is itself within ~1 ulp
    nz = want != 0
    err = np.abs(got - want)[nz]
    assert np.max(err - 2.0 * np.spacing(np.abs(want[nz]))) <= LOG_ABS, np.max(err)
    # |log x| >= 1/2: the absolute truncation term is below 0.1 ulp, so ulp-accurate
    far = nz & (np.abs(want) >= 0.5)
    assert np.max(np.abs(got - want)[far] / np.spacing(np.abs(want[far]))) <= 2.0
    assert got[np.where(x == 1.0)[0][0]] == 0.0
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 40
    sub = np.concatenate([x[:3000], x[200000:201000]])
    g = got[np.r_[0:3000, 200000:201000]]
    # two roundings + the k (ln2 - fl(ln2)) term (<= 0.2 ulp at any k) + the truncated term
    worst = max(float(abs(mpmath.mpf(float(gv)) - mpmath.log(mpmath.mpf(float(v)))))
                - 1.5 * float(np.spacing(abs(np.log(v)))) for v, gv in zip(sub, g) if v != 1.0)
    assert worst <= LOG_ABS, worst


def test_fast_rsqrt_rcp(engine):
    rng = np.random.default_rng(4)
    x = 10 ** rng.uniform(-14, 0.4, 200000)
    rs = engine.eval_math("rsqrt", x)
    want = 1.0 / np.sqrt(x)
    assert np.max(np.abs(rs - want) / np.spacing(want)) <= 2.5
    rc = engine.eval_math("rcp", x)
    want = 1.0 / x
    assert np.max(np.abs(rc - want) / np.spacing(want)) <= 2.5


def test_device_dilog(engine):
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    keep = g["dilog_u"] >= -1e-16
    u, want = g["dilog_u"][keep], g["dilog_v"][keep]
    got = engine.eval_math("dilog", u)
    nz = np.abs(want) > 1e-300
    assert np.max((np.abs(got[nz] - want[nz]) - 2e-17) / np.abs(want[nz])) < 4e-15
    assert np.all(got[~nz] == 0.0)


@pytest.mark.parametrize("kname", ["laplace", "biharmonic", "biot_savart", "sal"])
def test_kernel_values_match_reference(engine, kname):
    g = np.load(os.path.join(GOLD, "kernels.npz"))
    k = Kernel.parse(kname)
    got = engine.eval_pairs(k, g["x"], g["y"])
    ok = g[f"{kname}_ok"]
    want = g[f"{kname}_val"][:, : k.out_dim()]
    assert np.all(got[~ok] == 0.0)  # guarded pairs contribute nothing
    scale = np.maximum(np.abs(want[ok]), 1e-300)
    rel = np.maximum(np.abs(got[ok] - want[ok]) - 4e-17, 0) / np.maximum(
        scale, np.abs(want[ok]).max(axis=-1, keepdims=True) * 1e-3)
    assert rel.max() < 8e-15, rel.max()
