"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
total device time and share (cold-cache, serialised launches: compare SHARES)."""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
         "s": 1.0, "second": 1.0}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
        cnt[name] += 1
    T = sum(tot.values())
    out = [{"kernel": k, "total_ms": v * 1e3, "share": v / T, "launches": cnt[k], "avg_ms": v * 1e3 / cnt[k]}
           for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    return {"total_ms": T * 1e3, "launches": sum(cnt.values()), "kernels": out}


if __name__ == "__main__":
    s = summarise(sys.argv[1])
    if len(sys.argv) > 2:
        json.dump(s, open(sys.argv[2], "w"), indent=1)
    print(f"total {s['total_ms']:.3f} ms over {s['launches']} launches")
    for k in s["kernels"][:20]:
        print(f"{k['total_ms']:10.3f} ms {100 * k['share']:6.2f}%  n={k['launches']:4d}  {k['kernel'][:100]}")
