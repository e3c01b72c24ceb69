import os, sys, numpy as np
sys.path.insert(0, ".")
os.environ["CSFS_B200_MUTUAL_SCOPE"] = "unit"
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, TraversalConfig, configs
for name, level in [("c4", 6), ("c2", 7)]:
    wl = configs.make(name, level=level)
    k = Kernel.parse(wl.kernel); cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    p = ParticleSet(wl.xyz, wl.weights)
    e = Engine(0); want = e.csfmm_sum(p, p, k, cfg).values.copy()
    for R in (1, 2, 3, 4, 8):
        g = Engine.emulated(0, R)
        res = [g.csfmm_sum(p, p, k, cfg).values.copy() for _ in range(3)]
        print(name, R, [float(np.abs(r - want).max()) for r in res], [bool(np.array_equal(res[0], r)) for r in res])
        g.close()
