"""Multi-GPU contexts of the C-ABI (include/csfs_b200.h: csfs_b200_create_multi / _rank /
_emulated; paper_2508_13550_b200/csrc/partition.cu).

On one GPU:
  * Emulated groups run R ranks phase by phase on one device with device copies in place
    of the NCCL all-gathers: the partition, the owner-packed proxy-weight exchange and the
    potential exchange are checked BITWISE for R = 1..8 against each other and against
    the single-GPU engine with the same symmetric-pair scope (CSFS_B200_MUTUAL_SCOPE=unit);
  * the NCCL groups (ncclCommInitAll / ncclCommInitRank) run with one rank and must give
    the same bits (their exchanges are real NCCL broadcasts);
  * a multi-device group asking for a device that does not exist fails with code 1.
With two or more GPUs the multi-device group is checked bitwise against the emulation.
"""
import os

import numpy as np
import pytest
import torch

from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs
from paper_2508_13550_b200.engine import nccl_unique_id

pytestmark = pytest.mark.gpu

CASES = [("c2", 7, None), ("c5", 7, None), ("c3", 6, None), ("c4", 6, None)]


def _inputs(name, level, kname):
    wl = configs.make(name, level=level)
    k = Kernel.parse(kname or wl.kernel)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    return wl, k, cfg


def _unit_scope_engine():
    old = os.environ.get("CSFS_B200_MUTUAL_SCOPE")
    os.environ["CSFS_B200_MUTUAL_SCOPE"] = "unit"
    try:
        return Engine(0)
    finally:
        if old is None:
            del os.environ["CSFS_B200_MUTUAL_SCOPE"]
        else:
            os.environ["CSFS_B200_MUTUAL_SCOPE"] = old


@pytest.fixture(scope="module")
def unit_engine():
    e = _unit_scope_engine()
    yield e
    e.close()


@pytest.mark.parametrize("name,level,kname", CASES)
def test_emulated_groups_bitwise(unit_engine, name, level, kname):
    wl, k, cfg = _inputs(name, level, kname)
    p = ParticleSet(wl.xyz, wl.weights)
    want = unit_engine.csfmm_sum(p, p, k, cfg).values.copy()
    for R in (1, 2, 3, 4, 8):
        g = Engine.emulated(0, R)
        st = SumStats()
        got = g.csfmm_sum(p, p, k, cfg, st).values
        np.testing.assert_array_equal(got, want, err_msg=f"{name} R={R}")
        assert st.n_ranks == R
        info = g.group_info()
        assert info["nranks"] == R and info["devices"] == [0] * R
        if R > 1:
            t = [r for r in info["target_ranges"] if r[1] > r[0]]
            assert t[0][0] == 0 and t[-1][1] == wl.n and all(a[1] == b[0] for a, b in zip(t, t[1:]))
            s = [r for r in info["source_ranges"] if r[1] > r[0]]
            assert s[0][0] == 0 and s[-1][1] == wl.n and all(a[1] == b[0] for a, b in zip(s, s[1:]))
            assert st.t_exchange >= 0.0
        g.close()


def test_more_ranks_than_units_bitwise(unit_engine):
    """More ranks than partition units (24 depth-1 subtrees): the extra ranks own no
    targets and no sources — they build only the depth-0 items, send empty segments and
    still receive the full result — and the result is the same bits."""
    wl, k, cfg = _inputs("c2", 5, None)
    p = ParticleSet(wl.xyz, wl.weights)
    want = unit_engine.csfmm_sum(p, p, k, cfg).values.copy()
    g = Engine.emulated(0, 30)
    st = SumStats()
    np.testing.assert_array_equal(g.csfmm_sum(p, p, k, cfg, st).values, want)
    info = g.group_info()
    assert sum(1 for r in info["target_ranges"] if r[1] <= r[0]) >= 6
    u = SumStats()
    unit_engine.csfmm_sum(p, p, k, cfg, u)
    assert st.evals_executed == u.evals_executed
    g.close()


def test_group_executed_evaluations_add_up(unit_engine):
    """The executed evaluations the ranks report sum to the one-rank count (the roofline of
    an N-GPU bench line is this sum / N peaks); grid inputs have no depth-0 target items."""
    wl, k, cfg = _inputs("c5", 7, None)
    p = ParticleSet(wl.xyz, wl.weights)
    one = SumStats()
    Engine.emulated(0, 1).csfmm_sum(p, p, k, cfg, one)
    for R in (2, 4, 8):
        st = SumStats()
        Engine.emulated(0, R).csfmm_sum(p, p, k, cfg, st)
        assert st.evals_executed == one.evals_executed, R
    u = SumStats()
    unit_engine.csfmm_sum(p, p, k, cfg, u)
    assert one.evals_executed == u.evals_executed


def test_nccl_single_rank_groups_bitwise(unit_engine):
    wl, k, cfg = _inputs("c5", 7, None)
    p = ParticleSet(wl.xyz, wl.weights)
    want = unit_engine.csfmm_sum(p, p, k, cfg).values.copy()
    m = Engine.multi(1, [0])
    np.testing.assert_array_equal(m.csfmm_sum(p, p, k, cfg).values, want)
    assert m.group_info()["nranks"] == 1
    m.close()
    r = Engine.rank(0, 1, 0, nccl_unique_id())
    st = SumStats()
    np.testing.assert_array_equal(r.csfmm_sum(p, p, k, cfg, st).values, want)
    assert st.n_ranks == 1
    # device-pointer entry on the caller's stream
    dev = torch.device("cuda", 0)
    xyz = torch.from_numpy(wl.xyz).to(dev)
    w = torch.from_numpy(wl.weights).to(dev)
    out = torch.empty(wl.n, dtype=torch.float64, device=dev)
    r.csfmm_device(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg, out.data_ptr(),
                   torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), want)
    r.close()


def test_multi_refuses_missing_or_repeated_devices():
    n = torch.cuda.device_count()
    with pytest.raises(RuntimeError, match="code 1"):
        Engine.multi(n + 1)
    with pytest.raises(RuntimeError, match="code 1"):
        Engine.multi(2, [0, 0])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_multi_device_group_bitwise():
    n = torch.cuda.device_count()
    for name, level, kname in CASES[:2]:
        wl, k, cfg = _inputs(name, level, kname)
        p = ParticleSet(wl.xyz, wl.weights)
        for R in sorted({2, n}):
            want = Engine.emulated(0, R).csfmm_sum(p, p, k, cfg).values.copy()
            m = Engine.multi(R)
            st = SumStats()
            np.testing.assert_array_equal(m.csfmm_sum(p, p, k, cfg, st).values, want)
            assert st.n_ranks == R
            m.close()


def test_group_bve_step_bitwise():
    """bve_step on a group: four partitioned Biot-Savart sums (3-vector output)."""
    wl, _, _ = _inputs("c4", 6, None)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    zeta = wl.f.copy()
    res = []
    for R in (1, 3):
        g = Engine.emulated(0, R)
        x, z, st = g.bve_step(wl.xyz, zeta, wl.areas, 2 * np.pi, 0.01, cfg)
        res.append((x, z))
        assert all(s.n_ranks == R for s in st)
        g.close()
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1], res[1][1])


def test_leaf_histogram_matches_reference_tree(engine):
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    for name, level in (("c1", 5), ("c5", 6)):
        wl = configs.make(name, level=level)
        p = ParticleSet(wl.xyz, wl.weights)
        cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
        engine.csfmm_sum(p, p, Kernel.parse(wl.kernel), cfg)
        ints = ref.Tree(wl.xyz, wl.degree, wl.n0).export()["ints"]
        leaf = ints[:, 5] == 0
        sizes = (ints[:, 2] - ints[:, 1])[leaf]
        want = np.bincount(sizes).tolist()
        assert engine.leaf_histogram(0) == want
        assert engine.leaf_histogram(1) == want


@pytest.mark.parametrize("kname", ["laplace", "biot_savart"])
def test_groups_targets_differ_from_sources(engine, kname):
    """Separate target and source trees (no symmetric pairs): every rank count gives the
    single-GPU engine's result bit for bit."""
    from paper_2508_13550_b200.grids import cubed_sphere

    tx, _ = cubed_sphere(6)
    rng = np.random.default_rng(5)
    sx = rng.standard_normal((30000, 3))
    sx /= np.linalg.norm(sx, axis=1, keepdims=True)
    sw = rng.standard_normal(30000)
    k = Kernel.parse(kname)
    cfg = TraversalConfig(mac=0.6, degree=7, n0=60)
    t, s = ParticleSet(tx, np.zeros(len(tx))), ParticleSet(sx, sw)
    want = engine.csfmm_sum(t, s, k, cfg).values.copy()
    for R in (1, 2, 5):
        g = Engine.emulated(0, R)
        st = SumStats()
        np.testing.assert_array_equal(g.csfmm_sum(t, s, k, cfg, st).values, want, err_msg=f"R={R}")
        assert st.shared_tree == 0 and st.n_ranks == R
        g.close()
