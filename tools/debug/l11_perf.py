"""Steady-state phase times of the C5 setup at a finer level (default, 25.2M points):
python tools/debug/l11_perf.py [level] [reps]"""
import statistics
import sys

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 11
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = configs.make("c5", level=level)
eng = Engine(0)
p = ParticleSet(wl.xyz, wl.weights)
cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
k = Kernel.parse(wl.kernel)
ph = {f: [] for f in ("t_tree_build", "t_upward", "t_lists", "t_interact", "t_downward", "t_total")}
for i in range(reps + 1):
    st = SumStats()
    eng.csfmm_sum(p, p, k, cfg, st)
    if i:
        for f in ph:
            ph[f].append(getattr(st, f) * 1e3)
print(f"c5@L{level} N={wl.n}: " + " ".join(f"{f[2:]} {statistics.median(v):.2f}" for f, v in ph.items()) + " ms")
