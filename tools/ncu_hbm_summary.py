"""Summarise tools/ncu_hbm.sh captures: per kernel (summed over its launches in one C5 step)
duration, DRAM bytes, achieved GB/s, fraction of the measured HBM bandwidth.
python tools/ncu_hbm_summary.py gpurun_out/hbm_r02_fma.csv [out.json]"""
import csv
import json
import os
import sys
from collections import defaultdict

HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json"))).get("hbm_gbs", 6553.3) if os.path.exists("MEASURED_PEAKS.json") else 6553.3


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    recs = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        d = dict(zip(h, r))
        key = (int(d["ID"]), d["Kernel Name"])
        unit, val = d["Metric Unit"], d["Metric Value"].replace(",", "")
        try:
            v = float(val)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(unit, 1.0)
        recs[key][d["Metric Name"]] = v * scale
    return recs


def main(path, out=None):
    recs = load(path)
    agg = defaultdict(lambda: defaultdict(float))
    for (_, name), m in recs.items():
        short = name.replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
        short = short.replace("csfs_b200::", "").split("(")[0]
        short = short.split("<")[0] if "scan_" not in short else short[:60]
        a = agg[short]
        a["launches"] += 1
        a["time_s"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        a["fp64_pipe_pct_x_time"] += m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0) * m.get("gpu__time_duration.sum", 0.0)
    res = []
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["time_s"]):
        t = a["time_s"]
        res.append({"kernel": k, "launches": int(a["launches"]), "ms": t * 1e3, "dram_mb": a["dram_bytes"] / 1e6,
                    "gbs": a["dram_bytes"] / t / 1e9 if t else None,
                    "frac_of_hbm": a["dram_bytes"] / t / 1e9 / HBM if t else None,
                    "fp64_pipe_pct": a["fp64_pipe_pct_x_time"] / t if t else None})
    tot = sum(r["ms"] for r in res)
    print(f"{'kernel':40s} {'n':>4s} {'ms':>8s} {'MB':>9s} {'GB/s':>8s} {'%HBM':>6s} {'fp64%':>6s}")
    for r in res:
        print(f"{r['kernel'][:40]:40s} {r['launches']:4d} {r['ms']:8.3f} {r['dram_mb']:9.1f} {r['gbs'] or 0:8.1f} "
              f"{100 * (r['frac_of_hbm'] or 0):6.1f} {r['fp64_pipe_pct'] or 0:6.1f}")
    print(f"total {tot:.3f} ms")
    if out:
        json.dump({"source": path, "hbm_gbs_peak": HBM, "total_ms": tot, "kernels": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
