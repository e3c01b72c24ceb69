"""Developer probe: CSTC (cstc_sum, the §8f treecode) on the GPU vs the reference's cstc_sum
on the host, on a config's grid (device-resident GPU timing from SumStats; the reference on
a bounded sample of targets)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402  (the checker / CPU baseline only)
from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs  # noqa: E402


def main():
    eng = Engine(0)
    for name in sys.argv[1:] or ["c2", "c5"]:
        wl = configs.make(name)
        k = Kernel.parse(wl.kernel)
        cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
        p = ParticleSet(wl.xyz, wl.weights)
        for _ in range(2):
            st = SumStats()
            g = eng.cstc_sum(p, p, k, cfg, st).values
        rng = np.random.default_rng(3)
        m = min(wl.n, 65536)
        idx = np.sort(rng.choice(wl.n, m, replace=False))
        t0 = time.perf_counter()
        r, rst = ref.summed(1, wl.xyz[idx], wl.xyz, wl.weights, wl.kernel, mac=wl.mac, degree=wl.degree, n0=wl.n0)
        t_ref = time.perf_counter() - t0
        e = float(np.sqrt(np.sum((g[idx] - r) ** 2) / np.sum(r ** 2)))
        print(json.dumps({"cfg": name, "n": wl.n, "gpu_total_s": st.t_total, "gpu_pts_per_s": wl.n / st.t_total,
                          "ref_sample": m, "ref_s": t_ref, "ref_pts_per_s": m / t_ref, "threads": os.cpu_count(),
                          "rel_l2_on_sample": e, "pp": st.pp, "pc": st.pc}), flush=True)


if __name__ == "__main__":
    main()
