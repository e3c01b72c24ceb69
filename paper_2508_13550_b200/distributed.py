"""Multi-GPU CSFMM: target partitioning across ranks (one process per GPU).

The paper's parallel CSFMM gives "each MPI rank an equal portion of the interactions
followed by a global reduction".  The B200 design:
every rank builds the full trees and lists (cheap), owns a contiguous run of depth-1
cubed-sphere subtrees (tree order), computes the proxy weights of its source subtrees and
the potentials of its target subtrees, and two NCCL all-reduces (sum) over NVLink
exchange the owned parts (each slot has exactly one non-zero contributor, so the sum is
exact and the result is bitwise identical to one GPU).  The library is
collective-agnostic (include/csfs_b200.h, csfs_b200_part_*); this module is the host
runtime that drives it with torch.distributed.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def split_contiguous(costs, world: int) -> list[tuple[int, int]]:
    """Split units 0..n-1 (in tree order) into `world` contiguous runs of ~equal cost.

    Cut k is placed at the unit boundary whose prefix cost is closest to k*total/world,
    never moving backwards, so every rank gets a (possibly empty) run [lo, hi)."""
    c = np.asarray(costs, dtype=np.float64)
    n = c.size
    pre = np.concatenate([[0.0], np.cumsum(c)])
    total = pre[-1]
    cuts = [0]
    for k in range(1, world):
        goal = total * k / world
        j = int(np.searchsorted(pre, goal))
        cand = [x for x in (j - 1, j) if 0 <= x <= n]
        best = min(cand, key=lambda x: (abs(pre[x] - goal), x))
        cuts.append(max(best, cuts[-1]))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def owned_range(begin, end, run: tuple[int, int]) -> tuple[int, int]:
    lo, hi = run
    if hi <= lo:
        return (0, 0)
    return (int(begin[lo]), int(end[hi - 1]))


@dataclass
class PartitionPlan:
    target_range: tuple[int, int]
    source_range: tuple[int, int]
    target_cost_share: float


def plan_partition(engine, rank: int, world: int) -> PartitionPlan:
    tb, te, tc = engine.part_units(0)
    sb, se, sc = engine.part_units(1)
    trun = split_contiguous(tc, world)[rank]
    srun = split_contiguous(sc, world)[rank]
    share = float(np.sum(tc[trun[0]:trun[1]]) / max(np.sum(tc), 1.0))
    return PartitionPlan(owned_range(tb, te, trun), owned_range(sb, se, srun), share)


class ExchangeBuffers:
    """The two device buffers a rank all-reduces: proxy weights and tree-order potentials."""

    def __init__(self):
        self.pw = None
        self.phi = None

    def ensure(self, n_pw: int, n_phi: int, device):
        import torch

        if self.pw is None or self.pw.numel() < n_pw or self.pw.device != device:
            self.pw = torch.empty(n_pw, dtype=torch.float64, device=device)
        if self.phi is None or self.phi.numel() < n_phi or self.phi.device != device:
            self.phi = torch.empty(n_phi, dtype=torch.float64, device=device)
        return self.pw[:n_pw], self.phi[:n_phi]


def partitioned_csfmm(engine, tgt_xyz, src_xyz, src_w, kernel, config, out, group=None,
                      bufs: ExchangeBuffers | None = None, allreduce=None):
    """One CSFMM evaluation over all ranks of `group`.  Tensors are on this rank's GPU;
    `out` (n_targets x out_dim, input order) is complete on every rank on return.
    `allreduce(tensor)` defaults to torch.distributed.all_reduce(SUM) when world > 1."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if allreduce is None and dist.is_initialized():
        def allreduce(t):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    bufs = bufs if bufs is not None else getattr(engine, "_exchange", None) or ExchangeBuffers()
    engine._exchange = bufs
    dev = tgt_xyz.device
    stream = torch.cuda.current_stream(dev).cuda_stream if dev.type == "cuda" else 0
    engine.part_plan(tgt_xyz, tgt_xyz.shape[0], src_xyz, src_w, src_xyz.shape[0], kernel, config, stream)
    plan = plan_partition(engine, rank, world)
    pw, phi = bufs.ensure(*engine.part_sizes(), dev)
    engine.part_upward(*plan.source_range, pw)
    if allreduce is not None:
        allreduce(pw)
    engine.part_eval(*plan.target_range, pw, phi)
    if allreduce is not None:
        allreduce(phi)
    engine.part_finish(phi, out)
    return plan
