import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import ref
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig
eng = Engine(0)
def unit(v): return v / np.linalg.norm(v, axis=-1, keepdims=True)
def rl2(a, b): return float(np.sqrt(np.sum((a-b)**2)/np.sum(b**2)))
rng = np.random.default_rng(11)
for variant in ("unit", "scatter", "scatter+parallel"):
    x = unit(rng.normal(size=(20000, 3)))
    if variant != "unit":
        x = x * rng.uniform(0.98, 1.02, size=(20000, 1))
    if variant == "scatter+parallel":
        x[:50] = x[50:100] * (1.0 / np.einsum("ij,ij->i", x[50:100], x[50:100]))[:, None]
    w = rng.normal(size=20000)
    p = ParticleSet(x, w)
    for kern in ("laplace", "sal"):
        st = SumStats()
        cfg = TraversalConfig(mac=0.7, degree=6, n0=64)
        g = eng.csfmm_sum(p, p, Kernel.parse(kern), cfg, st).values
        r, rst = ref.csfmm(x, x, w, kern, mac=0.7, degree=6, n0=64)
        gd = eng.direct_sum(p, p, Kernel.parse(kern)).values
        rd = ref.direct(x, x, w, kern)
        print(variant, kern, "fmm", rl2(g, r), "direct", rl2(gd, rd), "lists", (st.pp, st.pc, st.cp, st.cc), tuple(int(v) for v in rst[5:9]), "fmm-vs-direct ref", rl2(r, rd), "gpu", rl2(g, gd), flush=True)
        st2 = SumStats()
