import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import ref
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig
eng = Engine(0)
def unit(v): return v / np.linalg.norm(v, axis=-1, keepdims=True)
def rl2(a, b): return float(np.sqrt(np.sum((a-b)**2)/np.sum(b**2)))
rng = np.random.default_rng(11)
x = unit(rng.normal(size=(20000, 3))) * rng.uniform(0.98, 1.02, size=(20000, 1))
w = rng.normal(size=20000)
p = ParticleSet(x, w)
for mac in (1e-9, 0.3, 0.7):
    cfg = TraversalConfig(mac=mac, degree=6, n0=64)
    st = SumStats()
    g = eng.csfmm_sum(p, p, Kernel.parse("laplace"), cfg, st).values
    r, rst = ref.csfmm(x, x, w, "laplace", mac=mac, degree=6, n0=64)
    rt = ref.Tree(x, 6, 64); re = rt.export(); ge = eng.tree_export(0)
    print("mac", mac, "fmm", rl2(g, r), "perm", np.array_equal(ge["perm"], re["perm"]), "ints", np.array_equal(ge["ints"], re["ints"]),
          "dbls", np.abs(ge["dbls"] - re["dbls"]).max(), "proxy", np.abs(ge["proxy"] - re["proxy"]).max(), flush=True)
    rpw = rt.upward(w); gpw = eng.proxy_weights_export()
    print("   pw", np.abs(gpw - rpw).max() / np.abs(rpw).max(), "lists", (st.pp, st.pc, st.cp, st.cc), tuple(int(v) for v in rst[5:9]))
    bad = np.argsort(-np.abs(g - r))[:5]
    print("   worst", bad, g[bad], r[bad])
