"""Developer probe: bve_remesh at C4's L9 (1.57M particles) on the GPU (device-resident and
through the host-pointer C-ABI) vs the reference's bve_remesh on the host cores."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import ref  # noqa: E402  (the checker / CPU baseline only)
from paper_2508_13550_b200 import Engine, configs  # noqa: E402


def main():
    level = int(sys.argv[1]) if len(sys.argv) > 1 else 9
    wl = configs.make("c4", level=level)
    x, z = ref.bve_step(wl.xyz, wl.f, wl.areas, wl.meta["omega_per_day"], 0.05, mac=wl.mac, degree=wl.degree,
                        n0=wl.n0)
    eng = Engine(0)
    dev = torch.device("cuda:0")
    dx, dz, dg = (torch.from_numpy(a).to(dev) for a in (x, z, wl.xyz))
    s = torch.cuda.current_stream().cuda_stream
    times = []
    for _ in range(5):
        bx, bz = dx.clone(), dz.clone()
        torch.cuda.synchronize()
        t = time.perf_counter()
        eng.bve_remesh_device(bx, bz, None, dg, wl.n, 12, s)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t)
    t0 = time.perf_counter()
    gx, gz, _ = eng.bve_remesh(x, z, wl.xyz)
    t_host = time.perf_counter() - t0
    t0 = time.perf_counter()
    rx, rz, _ = ref.bve_remesh(x, z, wl.xyz)
    t_ref = time.perf_counter() - t0
    e = float(np.sqrt(np.sum((gz - rz) ** 2) / np.sum(rz ** 2)))
    print(json.dumps({"level": level, "n": wl.n, "gpu_device_ms": 1e3 * min(times[1:]),
                      "gpu_host_api_ms": 1e3 * t_host, "reference_ms": 1e3 * t_ref,
                      "reference_threads": os.cpu_count(), "rel_l2": e}))


if __name__ == "__main__":
    main()
