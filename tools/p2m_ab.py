"""A/B of the leaf P2M: FMA kernel vs DMMA kernel (CSFS_B200_P2M=dmma), at C5 size.
Proxy weights against the reference's upward_pass (oracle/_ref) and the upward-phase time
(CUDA events, median of 5).  python tools/p2m_ab.py [fma|dmma] [config]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs  # noqa: E402

variant = sys.argv[1]
name = sys.argv[2] if len(sys.argv) > 2 else "c5"
wl = configs.make(name)
eng = Engine(0)
cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
p = ParticleSet(wl.xyz, wl.weights)
ts = []
for _ in range(6):
    st = SumStats()
    eng.csfmm_sum(p, p, Kernel.parse(wl.kernel), cfg, st)
    ts.append(st.t_upward * 1e3)
gpw = eng.proxy_weights_export()
rpw = ref.Tree(wl.xyz, wl.degree, wl.n0).upward(wl.weights)
err = float(np.abs(gpw - rpw).max() / np.abs(rpw).max())
print(json.dumps({"variant": variant, "config": name, "t_upward_ms_median": statistics.median(ts[1:]),
                  "proxy_weight_max_rel_err_vs_reference": err}))
