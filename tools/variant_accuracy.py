"""Developer probe: accuracy of the device log and kernel values for the library named by
CSFS_B200_LIB (A/B of fastmath variants).  Prints one JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2508_13550_b200 import Engine, Kernel  # noqa: E402

eng = Engine(0)
rng = np.random.default_rng(3)
x = np.concatenate([10 ** rng.uniform(-15, 0.35, 200000), 1 + rng.uniform(-1e-3, 1e-3, 20000)])
got = eng.eval_math("log", x)
want = np.log(x)
nz = want != 0
ulp = np.abs(got - want)[nz] / np.spacing(np.abs(want[nz]))
abserr = np.abs(got - want)
out = {"lib": os.environ.get("CSFS_B200_LIB", ""), "log_max_ulp": float(ulp.max()),
       "log_p999_ulp": float(np.quantile(ulp, 0.999)), "log_max_abs": float(abserr.max())}
g = np.load("tests/golden/kernels.npz")
for kname in ("laplace", "sal"):
    k = Kernel.parse(kname)
    v = eng.eval_pairs(k, g["x"], g["y"])
    ok = g[f"{kname}_ok"]
    w = g[f"{kname}_val"][:, : k.out_dim()]
    scale = np.maximum(np.abs(w[ok]), np.abs(w[ok]).max(axis=-1, keepdims=True) * 1e-3)
    out[f"{kname}_rel"] = float((np.abs(v[ok] - w[ok]) / scale).max())
print(json.dumps(out))
