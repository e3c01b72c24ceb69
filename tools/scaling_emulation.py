"""Per-rank cost of the target-partitioned multi-GPU csfmm, emulated on ONE GPU.

csfs_b200_create_emulated(device, W) runs the W ranks of the library's own partitioned
path (partition.cu: replicated plan, owned upward pass, owner-packed proxy-weight
exchange, owned evaluation + downward pass, potential exchange, scatter) phase by phase on
one device, the two all-gathers done as device copies.  Every rank's phases run alone on
the GPU and are timed with CUDA events (csfs_b200_group_phases), so nothing waits on
another rank (B200_PROFILING: no cross-rank spin on one GPU).  The projected step at W
GPUs is the slowest rank's own work plus its all-gather time at NVLink rate: the ranks'
broadcast bytes / NVLINK_GBS (the NCCL exchanges themselves run only on a multi-GPU box).
The result is bitwise the same for every W (checked here against W = 1).

    python tools/scaling_emulation.py [config] [out.json]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs  # noqa: E402

NVLINK_GBS = 450.0  # per-GPU all-gather bus bandwidth assumed for the projection (NVLink 5: 900 GB/s/direction)
REPS = 3


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    out = sys.argv[2] if len(sys.argv) > 2 else None
    wl = configs.make(name)
    k = Kernel.parse(wl.kernel)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    p = ParticleSet(wl.xyz, wl.weights)
    res = {"config": name, "n": wl.n, "nvlink_gbs_assumed": NVLINK_GBS, "worlds": []}
    base = None
    for world in (1, 2, 4, 8):
        g = Engine.emulated(0, world)
        best = None
        for _ in range(REPS + 1):
            st = SumStats()
            phi = g.csfmm_sum(p, p, k, cfg, st).values.copy()
            ph = g.group_phases()
            tot = [r["plan_ms"] + r["upward_ms"] + r["interact_ms"] + r["downward_ms"] + r["finish_ms"] for r in ph]
            if best is None or max(tot) < best[0]:
                best = (max(tot), ph, tot, st.evals_executed)
        if base is None:
            base = phi
        bitwise = bool(np.array_equal(phi, base))
        _, ph, tot, ex = best
        # all-gather time: every rank receives all other ranks' segments; at the bus rate
        # the step pays (total bytes - own) / bandwidth
        total_bytes = sum(r["exchange_bytes"] for r in ph)
        exch_ms = [(total_bytes - r["exchange_bytes"]) / (NVLINK_GBS * 1e9) * 1e3 if world > 1 else 0.0 for r in ph]
        step = max(t + e for t, e in zip(tot, exch_ms))
        rec = {"world": world, "step_ms_projected": step, "pts_per_s_projected": wl.n / (step * 1e-3),
               "bitwise_equal_to_w1": bitwise, "evals_executed_all_ranks": ex,
               "plan_ms_max": max(r["plan_ms"] for r in ph),
               "interact_ms_max": max(r["interact_ms"] for r in ph),
               "interact_ms_min": min(r["interact_ms"] for r in ph),
               "exchange_ms_projected_max": max(exch_ms), "ranks": ph}
        res["worlds"].append(rec)
        print(json.dumps({kk: v for kk, v in rec.items() if kk != "ranks"}), flush=True)
        g.close()
    w1 = res["worlds"][0]["step_ms_projected"]
    for r in res["worlds"]:
        r["efficiency_vs_w1"] = w1 / (r["step_ms_projected"] * r["world"])
    if out:
        json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
