"""One device-resident csfmm evaluation of a config (for ncu captures):
python tools/prof_once.py [config]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel, TraversalConfig, configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
wl = configs.make(name)
eng = Engine(0)
dev = torch.device("cuda:0")
xyz = torch.from_numpy(wl.xyz).to(dev)
w = torch.from_numpy(wl.weights).to(dev)
k = Kernel.parse(wl.kernel)
out = torch.empty(wl.n * k.out_dim(), dtype=torch.float64, device=dev)
cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
eng.csfmm_device(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg, out.data_ptr(),
                 torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", float(out[:8].sum()))
