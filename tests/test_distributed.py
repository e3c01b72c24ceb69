"""CPU: the multi-GPU host runtime (paper_2508_13550_b200/distributed.py) with world
size 2 and 4 over gloo.  The device engine is replaced by a CPU stand-in that honours the
csfs_b200_part_* ownership contract using the C restatement (oracle/port) — so what is
tested is the partition split, the exchange wiring (two all-reduces) and the final
scatter, i.e. everything the ranks do besides the kernels (which tests/
test_gpu_partition.py checks bitwise on the GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_13550_b200 import Kernel, TraversalConfig, configs
from paper_2508_13550_b200.distributed import owned_range, partitioned_csfmm, split_contiguous


class FakeEngine:
    """CPU stand-in for the part_* entry points (same contract as include/csfs_b200.h)."""

    def part_plan(self, tgt_xyz, nt, src_xyz, src_w, ns, kernel, config, stream):
        from oracle import port

        xyz, w = tgt_xyz.numpy(), src_w.numpy()
        n0 = config.resolved_n0()
        t = port.Tree(xyz, config.degree, n0, config.shrink)
        e = t.export()
        self.perm, ints = e["perm"], e["ints"]
        self.begin, self.end, self.depth, nch = ints[:, 1], ints[:, 2], ints[:, 4], ints[:, 5]
        self.pw_full = t.upward(w)
        self.n, self.dim = nt, kernel.out_dim()
        self.phi_full = port.csfmm(xyz, xyz, w, kernel.name(), mac=config.mac, degree=config.degree,
                                   n0=config.n0, shrink=config.shrink).reshape(nt, self.dim)
        keep = (self.end > self.begin) & ((self.depth == 1) | ((self.depth == 0) & (nch == 0)))
        order = np.argsort(self.begin[keep], kind="stable")
        self.ub, self.ue = self.begin[keep][order], self.end[keep][order]
        # deliberately uneven target costs so the split is exercised
        self.uc = (self.ue - self.ub) * (1.0 + (np.arange(self.ub.size) % 3))

    def part_units(self, which):
        return self.ub, self.ue, (self.uc if which == 0 else (self.ue - self.ub).astype(float))

    def part_sizes(self):
        return self.pw_full.size, self.n * self.dim

    def part_upward(self, b, e, pw):
        pw.zero_()
        own = (self.depth >= 1) & (self.begin >= b) & (self.begin < e)
        pw.view(self.pw_full.shape)[torch.from_numpy(own)] = torch.from_numpy(self.pw_full[own])

    def part_eval(self, b, e, pw, phi):
        deep = self.depth >= 1
        got = pw.view(self.pw_full.shape).numpy()[deep]
        assert np.array_equal(got, self.pw_full[deep]), "proxy-weight exchange incomplete"
        phi.zero_()
        tree = self.phi_full[self.perm]
        phi.view(self.n, self.dim)[b:e] = torch.from_numpy(tree[b:e])

    def part_finish(self, phi, out):
        out.view(self.n, self.dim)[torch.from_numpy(self.perm.astype(np.int64))] = phi.view(self.n, self.dim)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, level, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = configs.make(name, level=level)
        k = Kernel.parse(wl.kernel)
        cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
        xyz = torch.from_numpy(wl.xyz)
        w = torch.from_numpy(wl.weights)
        out = torch.zeros(wl.n * k.out_dim(), dtype=torch.float64)
        eng = FakeEngine()
        plan = partitioned_csfmm(eng, xyz, xyz, w, k, cfg, out)
        want = eng.phi_full.reshape(-1)
        ok = bool(np.array_equal(out.numpy(), want))
        shares = [None] * world
        dist.all_gather_object(shares, (plan.target_range, plan.source_range, plan.target_cost_share))
        if rank == 0:
            result_q.put((ok, shares))
        else:
            result_q.put((ok, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,name,level", [(2, "c1", None), (4, "c4", 5)])
def test_partitioned_runtime_gloo(world, name, level):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, level, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for ok, _ in res), "a rank's output differs from the single-process result"
    shares = next(s for _, s in res if s is not None)
    # target ranges tile the particles in rank order
    rngs = [t for t, _, _ in shares]
    assert rngs[0][0] == 0 and all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
    assert sum(c for _, _, c in shares) == pytest.approx(1.0)


def test_split_contiguous():
    c = np.ones(24)
    for world in (1, 2, 3, 4, 6, 8, 24):
        runs = split_contiguous(c, world)
        assert runs[0][0] == 0 and runs[-1][1] == 24
        assert all(a[1] == b[0] for a, b in zip(runs, runs[1:]))
        sizes = [hi - lo for lo, hi in runs]
        assert max(sizes) - min(sizes) <= 1
    runs = split_contiguous([10, 1, 1, 1, 1, 10], 2)
    assert runs == [(0, 3), (3, 6)]
    assert split_contiguous([5.0], 4)[0] == (0, 0) or split_contiguous([5.0], 4)[-1] == (1, 1)
    assert owned_range(np.array([0, 5, 9]), np.array([5, 9, 12]), (1, 3)) == (5, 12)
    assert owned_range(np.array([0]), np.array([5]), (1, 1)) == (0, 0)
