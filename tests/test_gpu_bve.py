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


def deformed_state(level, steps=3, dt=0.05):
    """Particles advected by the reference's own RK4 steps (remesh off): a genuinely
    scattered set for the remesh (neighbour sets cross faces and bucket rings)."""
    wl = configs.make("c4", level=level)
    x, z = wl.xyz, wl.f
    for _ in range(steps):
        x, z = ref.bve_step(x, z, wl.areas, wl.meta["omega_per_day"], dt, mac=wl.mac, degree=wl.degree, n0=wl.n0)
    return wl, x, z


@pytest.mark.parametrize("level,neighbors", [(5, 12), (7, 12), (7, 20), (6, 6)])
def test_remesh_matches_reference(engine, level, neighbors):
    """Same neighbour sets, stencils and pivots as the reference; the values agree to the
    conditioning of the 6x6 normal equations.  That conditioning is measured here: the
    reference's own result moves by `sens` when the particle positions move by 1 ulp
    (libdevice vs glibc atan/exp/acos differ by ~1 ulp), and ours must sit within it."""
    wl, x, z = deformed_state(level)
    tracer = np.cos(3 * wl.xyz[:, 0]) * np.sin(2 * wl.xyz[:, 2])
    gx, gz, gt = engine.bve_remesh(x, z, wl.xyz, tracer=tracer, neighbors=neighbors)
    rx, rz, rt = ref.bve_remesh(x, z, wl.xyz, tracer=tracer, neighbors=neighbors)
    np.testing.assert_array_equal(gx, rx)  # positions return to the grid centres exactly
    ulp = np.random.default_rng(level).choice([-1.0, 1.0], size=x.shape) * 2.0 ** -52
    _, pz, pt = ref.bve_remesh(x * (1 + ulp), z, wl.xyz, tracer=tracer, neighbors=neighbors)
    sens_z, sens_t = rel_l2(pz, rz), rel_l2(pt, rt)
    assert rel_l2(gz, rz) <= max(1e-13, 3 * sens_z)
    assert rel_l2(gt, rt) <= max(1e-13, 3 * sens_t)
    if neighbors >= 12:  # over-determined fits: well inside 1e-9 (k = 6 interpolates: ~1e-6)
        assert rel_l2(gz, rz) < 1e-9 and rel_l2(gt, rt) < 1e-9
    # pointwise: no point off by more than the reference's own 1-ulp response allows
    assert np.max(np.abs(gz - rz)) <= max(1e-12, 10 * np.max(np.abs(pz - rz)))


def test_remesh_edge_cases(engine):
    rng = np.random.default_rng(5)
    p = rng.normal(size=(40, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    g = rng.normal(size=(40, 3))
    g /= np.linalg.norm(g, axis=1, keepdims=True)
    z = rng.normal(size=40)
    for n in (1, 3, 5, 6, 7, 40):  # k = min(max(neighbors, 6), n): fewer than 6 -> nearest value
        for nb in (1, 12):
            gx, gz, _ = engine.bve_remesh(p[:n], z[:n], g[:n], neighbors=nb)
            rx, rz, _ = ref.bve_remesh(p[:n], z[:n], g[:n], neighbors=nb)
            np.testing.assert_array_equal(gx, rx)
            np.testing.assert_allclose(gz, rz, rtol=1e-9, atol=1e-12)
    gx, gz, gt = engine.bve_remesh(np.zeros((0, 3)), np.zeros(0), np.zeros((0, 3)))
    assert gx.shape == (0, 3) and gz.shape == (0,) and gt is None
    with pytest.raises(ValueError, match="remesh_neighbors above 64"):
        engine.bve_remesh(p, z, g, neighbors=65)


def test_bve_step_with_remesh_matches_reference(engine):
    """The reference's default BveStepOptions (remesh on, 12 neighbours): RK4 + remesh."""
    from paper_2508_13550_b200 import BveState, BveStepOptions, bve_step

    wl = configs.make("c4", level=6)
    tracer = wl.xyz[:, 2].copy()
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    st = BveState(positions=wl.xyz.copy(), zeta=wl.f.copy(), areas=wl.areas, grid_centers=wl.xyz,
                  tracer=tracer.copy(), omega=wl.meta["omega_per_day"])
    for _ in range(2):
        bve_step(st, 0.05, BveStepOptions(traversal=cfg), engine)
    rx, rz, rt = wl.xyz, wl.f, tracer
    for _ in range(2):
        rx, rz, rt = ref.bve_step_remesh(rx, rz, wl.areas, wl.xyz, wl.meta["omega_per_day"], 0.05, tracer=rt,
                                         mac=wl.mac, degree=wl.degree, n0=wl.n0)
    np.testing.assert_array_equal(st.positions, rx)
    assert rel_l2(st.zeta, rz) < 1e-9 and rel_l2(st.tracer, rt) < 1e-9  # remesh conditioning, see above
    assert abs(st.time - 0.1) < 1e-15
