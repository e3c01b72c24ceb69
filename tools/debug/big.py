import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig
eng = Engine(0)
for n in [int(a) for a in sys.argv[1:]]:
    rng = np.random.default_rng(60)
    x = rng.standard_normal((n, 3)); x /= np.linalg.norm(x, axis=1, keepdims=True)
    w = rng.standard_normal(n) * (4 * np.pi / n)
    st = SumStats(); t = time.time()
    p = ParticleSet(x, w)
    k = Kernel.parse("sal")
    g = eng.csfmm_sum(p, p, k, TraversalConfig(mac=0.6, degree=10, n0=256), st).values
    wall = time.time() - t
    idx = np.sort(rng.choice(n, 512, replace=False))
    d = eng.direct_sum(ParticleSet(x[idx], np.zeros(idx.size)), p, k).values
    e = float(np.sqrt(np.sum((g[idx] - d) ** 2) / np.sum(d ** 2)))
    print(n, round(wall, 3), "err", e, {k: v for k, v in st.as_dict().items() if k in ("t_interact", "t_lists", "symmetric_pairs", "symmetric_partials", "evals_executed", "pp")}, flush=True)
