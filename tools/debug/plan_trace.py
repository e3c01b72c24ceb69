"""Per-step host-clock trace of the partitioned plan (CSFS_B200_TRACE_PLAN): one emulated
group of R ranks on C5."""
import os, sys
os.environ["CSFS_B200_TRACE_PLAN"] = "1"
sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, TraversalConfig, configs
wl = configs.make(sys.argv[1] if len(sys.argv) > 1 else "c5")
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8
k = Kernel.parse(wl.kernel); cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
p = ParticleSet(wl.xyz, wl.weights)
g = Engine.emulated(0, R)
for _ in range(3):
    g.csfmm_sum(p, p, k, cfg)
    print("----", file=sys.stderr)
