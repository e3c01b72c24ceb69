"""Developer probe: config 4 — one barotropic-vorticity RK4 step (4 Biot-Savart CSFMM sums)
plus the remesh, on the GPU (device-resident, CUDA-event timed) vs the reference's
bve_step with remesh on (host cores, wall), at C4's L9."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402  (the checker / CPU baseline only)
from paper_2508_13550_b200 import Engine, TraversalConfig, configs  # noqa: E402


def main():
    level = int(sys.argv[1]) if len(sys.argv) > 1 else 9
    wl = configs.make("c4", level=level)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    omega, dt = wl.meta["omega_per_day"], wl.meta["dt_days"]
    eng = Engine(0)
    dev = torch.device("cuda:0")
    s = torch.cuda.current_stream().cuda_stream
    times = []
    for _ in range(3):
        x = torch.from_numpy(wl.xyz).to(dev)
        z = torch.from_numpy(wl.f).to(dev)
        a = torch.from_numpy(wl.areas).to(dev)
        g = torch.from_numpy(wl.xyz).to(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        eng.bve_step_device(x, z, a, wl.n, omega, dt, cfg, s)
        eng.bve_remesh_device(x, z, None, g, wl.n, 12, s)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    gz = z.cpu().numpy()
    t0 = time.perf_counter()
    rx, rz, _ = ref.bve_step_remesh(wl.xyz, wl.f, wl.areas, wl.xyz, omega, dt, mac=wl.mac, degree=wl.degree,
                                    n0=wl.n0)
    t_ref = time.perf_counter() - t0
    e = float(np.sqrt(np.sum((gz - rz) ** 2) / np.sum(rz ** 2)))
    print(json.dumps({"level": level, "n": wl.n, "gpu_step_ms": min(times[1:]), "reference_step_s": t_ref,
                      "reference_threads": os.cpu_count(), "speedup": t_ref / (min(times[1:]) * 1e-3),
                      "rel_l2_zeta_vs_reference": e}))


if __name__ == "__main__":
    main()
