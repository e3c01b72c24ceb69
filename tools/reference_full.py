"""One FULL run of the reference's csfmm_sum (oracle/_ref) on a BASELINE workload on this
host's cores, with its per-phase SumStats, nproc and the CPU model — and the bounded
sample bench.py times, so the extrapolation can be checked against the real thing.

    python tools/reference_full.py c5 profiles/r02_reference_c5_full.json
"""
import json
import os
import subprocess
import sys
import time

os.environ.setdefault("OMP_WAIT_POLICY", "active")
os.environ.setdefault("OMP_PROC_BIND", "close")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import ref  # noqa: E402
from paper_2508_13550_b200 import configs  # noqa: E402


def main(name, out):
    wl = configs.make(name)
    kw = dict(mac=wl.mac, degree=wl.degree, n0=wl.n0, threads=0)
    ref.csfmm(wl.xyz[:4096], wl.xyz[:4096], wl.weights[:4096], wl.kernel, **kw)  # OpenMP warm-up
    t = time.perf_counter()
    _, st = ref.csfmm(wl.xyz, wl.xyz, wl.weights, wl.kernel, **kw)
    wall = time.perf_counter() - t
    keys = ["t_tree_build", "t_upward", "t_traversal", "t_downward", "t_total", "pp", "pc", "cp", "cc",
            "src_depth", "src_clusters", "src_leaves", "tgt_depth", "tgt_clusters", "tgt_leaves"]
    full = {k: float(v) for k, v in zip(keys, st)}
    sample = bench.cpu_reference(wl, 2, 0)
    ext = [s["extrapolated_full_s"] for s in sample]
    lscpu = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    res = {"workload": bench.workload_config(wl, f"CPU, {os.cpu_count()} threads"),
           "nproc": os.cpu_count(), "cpu_model": bench.cpu_model(),
           "omp": {k: os.environ.get(k) for k in ("OMP_WAIT_POLICY", "OMP_PROC_BIND", "OMP_NUM_THREADS")},
           "full_run": {"wall_s": wall, "sumstats": full, "target_points_per_s": wl.n / wall},
           "bench_sample": sample,
           "extrapolated_over_full": [e / full["t_total"] for e in ext],
           "lscpu": lscpu.splitlines()[:20]}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({"full_s": full["t_total"], "extrapolated_s": ext,
                      "ratio": res["extrapolated_over_full"]}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
