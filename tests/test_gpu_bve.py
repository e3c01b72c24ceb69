"""GPU: config 4 — one barotropic-vorticity RK4 step (4 Biot-Savart CSFMM sums with
advected positions, remesh off; applications.cpp:378-412) against the reference's own
bve_step, and the FMM on ADVECTED (non-grid) positions: data-dependent shrunk-bounds tree,
non-empty PC list, bit-exact topology and lists."""
import numpy as np
import pytest

from oracle import ref
from paper_2508_13550_b200 import Kernel, ParticleSet, SumStats, TraversalConfig, configs

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / np.sum(b ** 2)))


def sorted_pairs(a):
    a = np.asarray(a).reshape(-1, 2)
    return a[np.lexsort((a[:, 1], a[:, 0]))] if a.size else a


@pytest.mark.parametrize("level", [6, 9])
def test_bve_step_matches_reference(engine, level):
    wl = configs.make("c4", level=level)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    omega, dt = wl.meta["omega_per_day"], wl.meta["dt_days"]
    gx, gz, stages = engine.bve_step(wl.xyz, wl.f, wl.areas, omega, dt, cfg)
    rx, rz = ref.bve_step(wl.xyz, wl.f, wl.areas, omega, dt, mac=wl.mac, degree=wl.degree, n0=wl.n0)
    # positions move by ~dt*|u|; compare the displacement, and the vorticity change
    assert rel_l2(gx - wl.xyz, rx - wl.xyz) < 1e-10
    assert rel_l2(gz - wl.f, rz - wl.f) < 1e-10
    np.testing.assert_allclose(np.linalg.norm(gx, axis=1), 1.0, atol=1e-15)
    assert stages[0].pc == 0 and all(s.evals_pp > 0 for s in stages)


def test_fmm_on_advected_positions(engine):
    """Stage-1 positions after one RK4 step: irregular leaves, PC interactions."""
    wl = configs.make("c4", level=7)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    x, z = ref.bve_step(wl.xyz, wl.f, wl.areas, wl.meta["omega_per_day"], wl.meta["dt_days"],
                        mac=wl.mac, degree=wl.degree, n0=wl.n0)
    # a stronger deformation: several steps of the reference
    for _ in range(3):
        x, z = ref.bve_step(x, z, wl.areas, wl.meta["omega_per_day"], 0.05, mac=wl.mac, degree=wl.degree,
                            n0=wl.n0)
    w = z * wl.areas
    for kname in ("biot_savart", "laplace", "sal"):
        st = SumStats()
        p = ParticleSet(x, w)
        g = engine.csfmm_sum(p, p, Kernel.parse(kname), cfg, st).values
        r, rst = ref.csfmm(x, x, w, kname, mac=wl.mac, degree=wl.degree, n0=wl.n0)
        assert rel_l2(g, r) < 1e-10, kname
        assert (st.pp, st.pc, st.cp, st.cc) == tuple(int(v) for v in rst[5:9])
    assert st.pc > 0  # advected trees have PC interactions
    rt = ref.Tree(x, wl.degree, wl.n0)
    re = rt.export()
    ge = engine.tree_export(0)
    np.testing.assert_array_equal(ge["perm"], re["perm"])
    np.testing.assert_array_equal(ge["ints"], re["ints"])
    gl, rl = engine.lists_export(), ref.lists(rt, rt, wl.mac, wl.n0)
    for k in ("pp", "pc", "cp", "cc"):
        np.testing.assert_array_equal(gl[k], sorted_pairs(rl[k]), err_msg=k)
    sizes = re["ints"][:, 2] - re["ints"][:, 1]
    leaf = re["ints"][:, 5] == 0
    assert sizes[leaf & (sizes > 0)].min() != sizes[leaf & (sizes > 0)].max()  # irregular leaves


def test_bve_rejects_nonpositive_dt(engine):
    wl = configs.make("c4", level=3)
    with pytest.raises(ValueError, match="time step must be positive"):
        engine.bve_step(wl.xyz, wl.f, wl.areas, 1.0, 0.0, TraversalConfig())
