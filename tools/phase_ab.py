"""A/B helper: median phase times of a config through the device entry (SumStats).
python tools/phase_ab.py [config] [reps]"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, SumStats, TraversalConfig, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 7
wl = configs.make(name)
eng = Engine(0)
dev = torch.device("cuda:0")
xyz = torch.from_numpy(wl.xyz).to(dev)
w = torch.from_numpy(wl.weights).to(dev)
k = Kernel.parse(wl.kernel)
out = torch.empty(wl.n * k.out_dim(), dtype=torch.float64, device=dev)
cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
s = torch.cuda.current_stream().cuda_stream
rows = []
for it in range(reps + 2):
    st = SumStats()
    eng.csfmm_device(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg, out.data_ptr(), s, st)
    if it >= 2:
        rows.append(st.as_dict())
keys = ("t_tree_build", "t_upward", "t_lists", "t_interact", "t_downward", "t_total")
print(json.dumps({"cfg": name, **{kk: round(1e3 * statistics.median(r[kk] for r in rows), 4) for kk in keys}}))
