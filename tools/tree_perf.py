"""Phase times (SumStats, median over repeated calls) of one config, with both tree builds
(label-then-sort default and the level-synchronous CSFS_B200_TREE=levels; TREE_MODES=sort
for the default only): python tools/tree_perf.py [config] [reps]"""
import os
import statistics
import sys

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
wl = configs.make(name)
eng = Engine(0)
p = ParticleSet(wl.xyz, wl.weights)
cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
k = Kernel.parse(wl.kernel)
modes = ["" if m == "sort" else m for m in os.environ.get("TREE_MODES", "sort,levels,sort").split(",")]
for mode in modes:
    if mode:
        os.environ["CSFS_B200_TREE"] = mode
    else:
        os.environ.pop("CSFS_B200_TREE", None)
    ph = {f: [] for f in ("t_tree_build", "t_upward", "t_lists", "t_interact", "t_downward", "t_total")}
    for _ in range(reps):
        st = SumStats()
        eng.csfmm_sum(p, p, k, cfg, st)
        for f in ph:
            ph[f].append(getattr(st, f) * 1e3)
    med = {f: statistics.median(v) for f, v in ph.items()}
    print(f"{name} tree={mode or 'sort':7s} build {med['t_tree_build']:.3f} ms (min {min(ph['t_tree_build']):.3f}) "
          f"upward {med['t_upward']:.3f} lists {med['t_lists']:.3f} interact {med['t_interact']:.3f} "
          f"downward {med['t_downward']:.3f} total {med['t_total']:.3f}")
