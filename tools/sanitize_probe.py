"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck): every
engine entry point on a few thousand points."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, Method, ParticleSet, SumStats, TraversalConfig, configs  # noqa

eng = Engine(0)
wl = configs.make("c1", level=4)
p = ParticleSet(wl.xyz, wl.weights)
for kname in ("laplace", "biharmonic", "biot_savart", "sal"):
    k = Kernel.parse(kname)
    st = SumStats()
    eng.csfmm_sum(p, p, k, TraversalConfig(degree=6, n0=32), st)
    eng.summed_potential(p, p, k, TraversalConfig(method=Method.Cstc, degree=6, n0=32))
    eng.direct_sum(ParticleSet(wl.xyz[:300], wl.weights[:300]), p, k)
    print(kname, st.pp, st.pc, st.cp, st.cc, st.symmetric_pairs, flush=True)
q = ParticleSet(wl.xyz[::2].copy(), wl.weights[::2].copy())
eng.csfmm_sum(q, p, Kernel.parse("sal"), TraversalConfig(degree=8, n0=20))
c4 = configs.make("c4", level=4)
eng.bve_step(c4.xyz, c4.f, c4.areas, 6.28, 0.01, TraversalConfig(mac=0.7, degree=6, n0=40))
eng.eval_math("log", np.linspace(0.1, 2, 100))
print("ok")
