"""GPU: the CSTC treecode (csfs::cstc_sum, summation.cpp:308-381) — the second fast
method behind summed_potential — against the reference's own cstc_sum: potentials within
1e-10 relative L2, identical per-target interaction counts (stats pp/pc), degenerate
MAC -> direct sum (test_summation.cpp:100-112), targets != sources."""
import numpy as np
import pytest

from oracle import ref
from paper_2508_13550_b200 import Kernel, Method, ParticleSet, SumStats, TraversalConfig, configs

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.sqrt(np.sum((a - b) ** 2) / np.sum(b ** 2)))


@pytest.mark.parametrize("kname", ["laplace", "biharmonic", "biot_savart", "sal"])
@pytest.mark.parametrize("grid,level,degree,mac,n0", [("icosahedral", 4, 6, 0.7, -1), ("cubed_sphere", 5, 8, 0.6, 40)])
def test_cstc_matches_reference(engine, kname, grid, level, degree, mac, n0):
    xyz, a = ref.grid(grid, level)
    w = ref.sph_harm(4, 3, xyz) * a
    cfg = TraversalConfig(method=Method.Cstc, mac=mac, degree=degree, n0=n0)
    st = SumStats()
    p = ParticleSet(xyz, w)
    g = engine.summed_potential(p, p, Kernel.parse(kname), cfg, st).values
    r, rst = ref.summed(1, xyz, xyz, w, kname, mac=mac, degree=degree, n0=n0)
    assert rel_l2(g, r) < 1e-10
    assert (st.pp, st.pc) == (int(rst[5]), int(rst[6]))
    assert st.pc > 0


def test_cstc_degenerate_mac_is_direct(engine):
    xyz, a = ref.grid("icosahedral", 3)
    w = ref.sph_harm(4, 3, xyz) * a
    p = ParticleSet(xyz, w)
    g = engine.summed_potential(p, p, Kernel.parse("laplace"), TraversalConfig(method=Method.Cstc, mac=1e-9)).values
    d = ref.direct(xyz, xyz, w, "laplace")
    assert np.abs(g - d).max() < 1e-12 * np.abs(d).max()


def test_cstc_targets_differ_and_full_size(engine):
    sx, sa = ref.grid("icosahedral", 4)
    sw = ref.sph_harm(4, 3, sx) * sa
    tx, _ = ref.grid("cubed_sphere", 4)
    cfg = TraversalConfig(method=Method.Cstc)
    g = engine.summed_potential(ParticleSet(tx, np.zeros(len(tx))), ParticleSet(sx, sw), Kernel.parse("laplace"), cfg).values
    r, _ = ref.summed(1, tx, sx, sw, "laplace")
    assert rel_l2(g, r) < 1e-10
    # C2 grid size: 393,216 points (reference treecode, all host threads)
    wl = configs.make("c2")
    cfg = TraversalConfig(method=Method.Cstc, mac=wl.mac, degree=wl.degree, n0=wl.n0)
    p = ParticleSet(wl.xyz, wl.weights)
    st = SumStats()
    g = engine.summed_potential(p, p, Kernel.parse(wl.kernel), cfg, st).values
    r, rst = ref.summed(1, wl.xyz, wl.xyz, wl.weights, wl.kernel, mac=wl.mac, degree=wl.degree, n0=wl.n0)
    print(f"C2 CSTC: GPU {st.t_total*1e3:.1f} ms, rel L2 {rel_l2(g, r):.2e}")
    assert rel_l2(g, r) < 1e-10
    assert (st.pp, st.pc) == (int(rst[5]), int(rst[6]))


@pytest.mark.parametrize("kname", ["laplace", "biharmonic", "biot_savart", "sal"])
def test_cstc_warp_traversal_equals_per_target_traversal(engine, kname, monkeypatch):
    """The warp-cooperative traversal (shared stack of (cluster, lane mask), sources staged
    once per warp) sums every target in the order of its own depth-first traversal: bit for
    bit the one-thread-per-target kernel (CSFS_B200_CSTC=thread), same counts — on a grid
    (targets == sources, tree order), on shuffled separate targets (sparse lane masks) and on
    a target count that is not a multiple of 32."""
    xyz, a = ref.grid("cubed_sphere", 5)
    w = ref.sph_harm(4, 3, xyz) * a
    rng = np.random.default_rng(11)
    tx = xyz[rng.permutation(len(xyz))[:3001]] * 1.0
    k = Kernel.parse(kname)
    cfg = TraversalConfig(method=Method.Cstc, mac=0.6, degree=8, n0=40)
    for tgt in (ParticleSet(xyz, w), ParticleSet(tx, np.zeros(len(tx)))):
        res = {}
        for mode in ("thread", "warp"):
            if mode == "thread":
                monkeypatch.setenv("CSFS_B200_CSTC", "thread")
            else:
                monkeypatch.delenv("CSFS_B200_CSTC", raising=False)
            st = SumStats()
            res[mode] = (engine.summed_potential(tgt, ParticleSet(xyz, w), k, cfg, st).values.copy(), st.pp, st.pc)
        assert res["thread"][1:] == res["warp"][1:]
        assert np.array_equal(res["thread"][0].view(np.uint64), res["warp"][0].view(np.uint64))
