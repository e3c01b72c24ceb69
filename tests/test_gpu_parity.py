"""GPU parity: the B200 CSFMM (through the C-ABI) against the reference's own csfmm_sum,
direct_sum, ClusterTree, upward_pass and dual_tree_traversal (oracle/_ref) on identical
inputs.  Bars (BASELINE.json north_star): potentials within 1e-10 relative L2, tree
topology / order / interaction lists bit-exact, geometry within a few ulp (glibc vs
libdevice atan/tan).
"""
import numpy as np
import pytest

from oracle import ref
from paper_2508_13550_b200 import Kernel, ParticleSet, SumStats, TraversalConfig, configs

pytestmark = pytest.mark.gpu

PARITY = 1e-10  # north_star: relative L2 vs the reference's own FMM


def rel_l2(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / np.sum(b ** 2)))


def sorted_pairs(a):
    a = np.asarray(a).reshape(-1, 2)
    if a.size == 0:
        return a
    return a[np.lexsort((a[:, 1], a[:, 0]))]


def check_structure(engine, xyz, degree, n0, mac, shrink=True, w=None):
    """Tree (both sides), lists and proxy weights of the last engine call vs the reference."""
    rt = ref.Tree(xyz, degree, n0, shrink)
    re = rt.export()
    for which in (0, 1):
        ge = engine.tree_export(which)
        assert ge["depth"] == re["depth"]
        np.testing.assert_array_equal(ge["perm"], re["perm"])
        np.testing.assert_array_equal(ge["ints"], re["ints"])
        np.testing.assert_allclose(ge["dbls"], re["dbls"], rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(ge["proxy"], re["proxy"], rtol=1e-13, atol=1e-15)
    rl = ref.lists(rt, rt, mac, n0)
    gl = engine.lists_export()
    for k in ("pp", "pc", "cp", "cc"):
        np.testing.assert_array_equal(gl[k], sorted_pairs(rl[k]), err_msg=k)
    if w is not None:
        rpw = rt.upward(w)
        gpw = engine.proxy_weights_export()
        scale = np.abs(rpw).max()
        assert np.abs(gpw - rpw).max() <= 1e-12 * scale


def run_pair(engine, xyz, w, kernel, degree, mac, n0, shrink=True, sal=None):
    cfg = TraversalConfig(mac=mac, degree=degree, n0=n0, shrink=shrink)
    st = SumStats()
    p = ParticleSet(xyz, w)
    g = engine.csfmm_sum(p, p, Kernel.parse(kernel), cfg, st).values
    r, rst = ref.csfmm(xyz, xyz, w, kernel, mac=mac, degree=degree, n0=n0, shrink=shrink)
    return g, r, st, rst


def test_c1_full_parity(engine):
    wl = configs.make("c1")
    g, r, st, rst = run_pair(engine, wl.xyz, wl.weights, wl.kernel, wl.degree, wl.mac, wl.n0)
    assert rel_l2(g, r) < PARITY
    assert (st.pp, st.pc, st.cp, st.cc) == tuple(int(v) for v in rst[5:9])
    assert (st.tgt_depth, st.tgt_clusters, st.tgt_leaves) == tuple(int(v) for v in rst[12:15])
    check_structure(engine, wl.xyz, wl.degree, wl.n0, wl.mac, w=wl.weights)
    # FMM-vs-exact error matches the reference's (same approximation)
    a = wl.areas
    e_g = np.sqrt(np.sum((g - wl.exact) ** 2 * a) / np.sum(wl.exact ** 2 * a))
    e_r = np.sqrt(np.sum((r - wl.exact) ** 2 * a) / np.sum(wl.exact ** 2 * a))
    assert abs(e_g - e_r) <= 1e-8 * e_r


def test_direct_matches_reference(engine):
    wl = configs.make("c1")
    p = ParticleSet(wl.xyz, wl.weights)
    for kname in ("laplace", "biharmonic", "biot_savart", "sal"):
        g = engine.direct_sum(p, p, Kernel.parse(kname)).values
        r = ref.direct(wl.xyz, wl.xyz, wl.weights, kname)
        assert rel_l2(g, r) < 1e-12, kname


@pytest.mark.parametrize("kname", ["laplace", "biharmonic", "biot_savart", "sal"])
@pytest.mark.parametrize("grid,level,degree,mac,n0", [
    ("icosahedral", 4, 6, 0.7, -1),
    ("cubed_sphere", 5, 8, 0.6, 40),
    ("icosahedral", 3, 10, 0.3, 20),
])
def test_kernels_parity(engine, kname, grid, level, degree, mac, n0):
    xyz, a = ref.grid(grid, level)
    w = ref.sph_harm(4, 3, xyz) * a
    g, r, st, rst = run_pair(engine, xyz, w, kname, degree, mac, n0)
    assert rel_l2(g, r) < PARITY
    assert (st.pp, st.pc, st.cp, st.cc) == tuple(int(v) for v in rst[5:9])


def test_targets_differ_from_sources(engine):
    sx, sa = ref.grid("icosahedral", 4)
    sw = ref.sph_harm(4, 3, sx) * sa
    tx, _ = ref.grid("cubed_sphere", 4)
    cfg = TraversalConfig()
    g = engine.csfmm_sum(ParticleSet(tx, np.zeros(len(tx))), ParticleSet(sx, sw), Kernel.parse("laplace"), cfg).values
    r, _ = ref.csfmm(tx, sx, sw, "laplace")
    assert rel_l2(g, r) < PARITY


def test_no_shrink_and_degenerate_mac(engine):
    xyz, a = ref.grid("icosahedral", 3)
    w = ref.sph_harm(4, 3, xyz) * a
    g, r, _, _ = run_pair(engine, xyz, w, "laplace", 6, 0.7, 30, shrink=False)
    assert rel_l2(g, r) < PARITY
    check_structure(engine, xyz, 6, 30, 0.7, shrink=False, w=w)
    # degenerate MAC: CSFMM reduces to the direct sum (test_summation.cpp:100-112)
    cfg = TraversalConfig(mac=1e-9, degree=6)
    p = ParticleSet(xyz, w)
    g = engine.csfmm_sum(p, p, Kernel.parse("laplace"), cfg).values
    d = ref.direct(xyz, xyz, w, "laplace")
    assert np.abs(g - d).max() < 1e-12 * np.abs(d).max()


def test_reference_errors(engine):
    p = ParticleSet(np.array([[0.0, 0.0, 1.0]]), np.array([1.0]))
    empty = ParticleSet(np.zeros((0, 3)), np.zeros(0))
    k = Kernel.parse("laplace")
    with pytest.raises(ValueError, match="cannot build a cluster tree from an empty particle set"):
        engine.csfmm_sum(empty, p, k, TraversalConfig())
    with pytest.raises(ValueError, match="maximum leaf size must be at least 1"):
        engine.csfmm_sum(p, p, k, TraversalConfig(n0=0))
    with pytest.raises(ValueError, match="interpolation degree must be positive"):
        engine.csfmm_sum(p, p, k, TraversalConfig(degree=0))
