"""Developer probe: run configs through the engine (device-resident) and print SumStats."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, TraversalConfig, configs  # noqa: E402


def main():
    names = sys.argv[1:] or ["c1", "c2", "c5"]
    eng = Engine(0)
    for name in names:
        wl = configs.make(name)
        dev = torch.device("cuda:0")
        xyz = torch.from_numpy(wl.xyz).to(dev)
        w = torch.from_numpy(wl.weights).to(dev)
        k = Kernel.parse(wl.kernel)
        out = torch.empty(wl.n * k.out_dim(), dtype=torch.float64, device=dev)
        cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
        s = torch.cuda.current_stream().cuda_stream
        for it in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            st = eng.csfmm_device(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg,
                                  out.data_ptr(), s)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t
            d = st.as_dict()
            ev = d["evals_pp"] + d["evals_pc"] + d["evals_cp"] + d["evals_cc"]
            print(json.dumps({"cfg": name, "it": it, "wall": dt, "pts_per_s": wl.n / dt,
                              "evals": ev, "evals_per_s": ev / d["t_interact"],
                              **{kk: (round(v, 6) if isinstance(v, float) else v) for kk, v in d.items()}}),
                  flush=True)


if __name__ == "__main__":
    main()
