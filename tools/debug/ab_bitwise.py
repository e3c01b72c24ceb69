"""Bitwise A/B of two library builds: python tools/debug/ab_bitwise.py save|check FILE [config]
(run once with CSFS_B200_LIB=<build A> save, once with build B check)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, TraversalConfig, configs  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
name = sys.argv[3] if len(sys.argv) > 3 else "c3"
wl = configs.make(name)
eng = Engine(0)
p = ParticleSet(wl.xyz, wl.weights)
out = eng.csfmm_sum(p, p, Kernel.parse(wl.kernel), TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)).values
if mode == "save":
    np.save(path, out)
    print("saved", out.shape)
else:
    ref = np.load(path)
    same = np.array_equal(ref.view(np.uint64), out.view(np.uint64))
    print(name, "bitwise equal" if same else f"DIFFERENT: max abs diff {np.abs(ref - out).max():.3e}")
    sys.exit(0 if same else 1)
