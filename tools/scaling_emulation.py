"""Per-rank cost of the target-partitioned multi-GPU step, emulated on ONE GPU.

For world W in 1, 2, 4, 8 every rank's device work is run one rank after another and timed
with CUDA events: the replicated part (part_plan: trees, lists, items, symmetric pairs),
the rank's owned upward pass, its owned evaluation + downward pass, and the final scatter.
Nothing here waits on another rank (SURVEY/B200_PROFILING: no cross-rank spin on one GPU);
the two all-reduces (proxy weights, tree-order potentials) are not run — their volume is
reported instead.  The projected step time at W GPUs is max over ranks of the rank's own
work; the real multi-GPU run adds the all-reduces over NVLink.

    python tools/scaling_emulation.py [config]
"""
import json
import sys

import torch

REPS = 3  # each rank's phases timed REPS times, min kept (one-off clock dips excluded)

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, TraversalConfig, configs  # noqa: E402
from paper_2508_13550_b200.distributed import plan_partition  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    wl = configs.make(name)
    dev = torch.device("cuda", 0)
    eng = Engine(0)
    xyz = torch.from_numpy(wl.xyz).to(dev)
    w = torch.from_numpy(wl.weights).to(dev)
    k = Kernel.parse(wl.kernel)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    s = torch.cuda.current_stream().cuda_stream
    out = torch.empty(wl.n * k.out_dim(), dtype=torch.float64, device=dev)

    def plan():
        eng.part_plan(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg, s)

    for _ in range(2):
        plan()
    t_plan = min(timed(plan) for _ in range(3))
    n_pw, n_phi = eng.part_sizes()
    pw = torch.zeros(n_pw, dtype=torch.float64, device=dev)
    phi = torch.zeros(n_phi, dtype=torch.float64, device=dev)
    res = {"config": name, "n": wl.n, "part_plan_ms": t_plan, "allreduce_bytes": 8 * (n_pw + n_phi), "worlds": []}
    for world in (1, 2, 4, 8):
        ranks = []
        for r in range(world):
            p = plan_partition(eng, r, world)
            t_up = min(timed(lambda: eng.part_upward(*p.source_range, pw.data_ptr())) for _ in range(REPS))
            t_ev = min(timed(lambda: eng.part_eval(*p.target_range, pw.data_ptr(), phi.data_ptr()))
                       for _ in range(REPS))
            t_fin = min(timed(lambda: eng.part_finish(phi.data_ptr(), out.data_ptr())) for _ in range(REPS))
            ranks.append({"rank": r, "upward_ms": t_up, "eval_ms": t_ev, "finish_ms": t_fin,
                          "total_ms": t_plan + t_up + t_ev + t_fin, "cost_share": p.target_cost_share})
        step = max(x["total_ms"] for x in ranks)
        res["worlds"].append({"world": world, "step_ms_max_rank": step, "pts_per_s": wl.n / (step * 1e-3),
                              "ranks": ranks})
        print(json.dumps({"world": world, "step_ms": step, "pts_per_s": wl.n / (step * 1e-3),
                          "eval_ms": [round(x["eval_ms"], 2) for x in ranks]}), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
