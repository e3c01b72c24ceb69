"""Tree-build phase time of one config, both builds (label-then-sort default and the
level-synchronous CSFS_B200_TREE=levels), from SumStats over repeated calls:
python tools/tree_perf.py [config] [reps]"""
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
for mode in ("", "levels", ""):
    if mode:
        os.environ["CSFS_B200_TREE"] = mode
    else:
        os.environ.pop("CSFS_B200_TREE", None)
    tb, tl, tt = [], [], []
    for _ in range(reps):
        st = SumStats()
        eng.csfmm_sum(p, p, k, cfg, st)
        tb.append(st.t_tree_build * 1e3)
        tl.append(st.t_lists * 1e3)
        tt.append(st.t_total * 1e3)
    print(f"{name} tree={mode or 'sort':7s} build {statistics.median(tb):.3f} ms (min {min(tb):.3f}) "
          f"lists {statistics.median(tl):.3f} total {statistics.median(tt):.3f}")
