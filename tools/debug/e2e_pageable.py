"""e2e through the host-pointer C-ABI with pageable vs pinned host buffers (C5)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, TraversalConfig, configs  # noqa: E402

wl = configs.make(sys.argv[1] if len(sys.argv) > 1 else "c5")
eng = Engine(0)
k = Kernel.parse(wl.kernel)
cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
for name in ("pageable", "pinned"):
    if name == "pinned":
        hx = torch.from_numpy(wl.xyz).pin_memory().numpy()
        hw = torch.from_numpy(wl.weights).pin_memory().numpy()
        ho = torch.empty(wl.n * k.out_dim(), dtype=torch.float64).pin_memory().numpy()
    else:
        hx, hw, ho = wl.xyz.copy(), wl.weights.copy(), np.empty(wl.n * k.out_dim())
    p = ParticleSet(hx, hw)
    eng.csfmm_sum(p, p, k, cfg, out=ho)
    t0 = time.perf_counter()
    for _ in range(5):
        eng.csfmm_sum(p, p, k, cfg, out=ho)
    dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {dt * 1e3:.2f} ms per call, {wl.n / dt:.3e} pts/s")
