"""Multi-GPU target partitioning on ONE GPU: the R ranks are emulated one after the other
(each rank's phase is an independent launch; the all-reduces are done here on the device
by summing the per-rank buffers), so nothing waits on another rank.  The result must be
BITWISE identical for every R (each target is evaluated by exactly one rank in a fixed
order; every reduced slot has one non-zero term), and bitwise equal to the single-GPU
csfmm run with the same symmetric-pair scope (CSFS_B200_MUTUAL_SCOPE=unit); the default
single-GPU scope pairs more leaves symmetrically and agrees to rounding."""
import numpy as np
import pytest
import torch

from paper_2508_13550_b200 import Kernel, ParticleSet, TraversalConfig, configs
from paper_2508_13550_b200.distributed import plan_partition

pytestmark = pytest.mark.gpu


def emulate(engine, xyz, w, kernel, cfg, world):
    dev = xyz.device
    s = torch.cuda.current_stream(dev).cuda_stream
    engine.part_plan(xyz.data_ptr(), xyz.shape[0], xyz.data_ptr(), w.data_ptr(), xyz.shape[0], kernel, cfg, s)
    plans = [plan_partition(engine, r, world) for r in range(world)]
    n_pw, n_phi = engine.part_sizes()
    pws = [torch.empty(n_pw, dtype=torch.float64, device=dev) for _ in plans]
    for p, buf in zip(plans, pws):
        engine.part_upward(*p.source_range, buf.data_ptr())
    pw = torch.stack(pws).sum(0)  # the all-reduce
    phis = [torch.empty(n_phi, dtype=torch.float64, device=dev) for _ in plans]
    for p, buf in zip(plans, phis):
        engine.part_eval(*p.target_range, pw.data_ptr(), buf.data_ptr())
    phi = torch.stack(phis).sum(0)
    out = torch.empty(xyz.shape[0] * kernel.out_dim(), dtype=torch.float64, device=dev)
    engine.part_finish(phi.data_ptr(), out.data_ptr())
    return out, plans, pws


@pytest.mark.parametrize("name,level,kname", [("c1", 5, None), ("c3", 6, None), ("c4", 6, None)])
def test_partition_bitwise(engine, name, level, kname):
    wl = configs.make(name, level=level)
    dev = torch.device("cuda", 0)
    xyz = torch.from_numpy(wl.xyz).to(dev)
    w = torch.from_numpy(wl.weights).to(dev)
    k = Kernel.parse(kname or wl.kernel)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    ref_out = torch.empty(wl.n * k.out_dim(), dtype=torch.float64, device=dev)
    engine.csfmm_device(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg, ref_out.data_ptr(),
                        torch.cuda.current_stream().cuda_stream)
    want = ref_out.cpu().numpy()
    want_pw = engine.proxy_weights_export()
    one, _, _ = emulate(engine, xyz, w, k, cfg, 1)
    one = one.cpu().numpy()
    assert np.sqrt(np.sum((one - want) ** 2) / np.sum(want ** 2)) < 1e-14  # global vs unit pair scope
    want = one
    for world in (1, 2, 4, 8):
        got, plans, pws = emulate(engine, xyz, w, k, cfg, world)
        # every proxy weight slot at depth >= 1 has exactly one owner
        nz = torch.stack([(p != 0) for p in pws]).sum(0)
        assert int(nz.max()) <= 1, f"world={world}: a proxy weight has {int(nz.max())} owners"
        np.testing.assert_array_equal(got.cpu().numpy(), want, err_msg=f"world={world}")
        # target ranges tile [0, N) in order
        rngs = [p.target_range for p in plans if p.target_range[1] > p.target_range[0]]
        assert rngs[0][0] == 0 and rngs[-1][1] == wl.n
        assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))


@pytest.mark.parametrize("name,level", [("c5", 7), ("c3", 7), ("c4", 7)])
def test_run_to_run_bitwise(engine, name, level):
    """Every output slot has one owner and a fixed summation order (no atomics on
    floating-point data), so repeated runs are bitwise identical — the reference's
    thread-count independence claim (summation.hpp:19-21) on the GPU, and a race check."""
    wl = configs.make(name, level=level)
    p = ParticleSet(wl.xyz, wl.weights)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    k = Kernel.parse(wl.kernel)
    a = engine.csfmm_sum(p, p, k, cfg).values
    b = engine.csfmm_sum(p, p, k, cfg).values
    np.testing.assert_array_equal(a, b)


def test_unit_scope_single_gpu_equals_partition(monkeypatch):
    """With CSFS_B200_MUTUAL_SCOPE=unit the single-GPU csfmm pairs exactly the leaves the
    partitioned path pairs, and the two are bitwise equal."""
    from paper_2508_13550_b200 import Engine

    monkeypatch.setenv("CSFS_B200_MUTUAL_SCOPE", "unit")
    eng = Engine(0)
    wl = configs.make("c5", level=6)
    dev = torch.device("cuda", 0)
    xyz = torch.from_numpy(wl.xyz).to(dev)
    w = torch.from_numpy(wl.weights).to(dev)
    k = Kernel.parse(wl.kernel)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    ref_out = torch.empty(wl.n, dtype=torch.float64, device=dev)
    eng.csfmm_device(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg, ref_out.data_ptr(),
                     torch.cuda.current_stream().cuda_stream)
    got, _, _ = emulate(eng, xyz, w, k, cfg, 4)
    np.testing.assert_array_equal(got.cpu().numpy(), ref_out.cpu().numpy())
    eng.close()
