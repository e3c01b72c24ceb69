"""Per kernel (summed over launches) of an ncu raw-page CSV: launches, total time, and for the
longest launch the issue / occupancy / DRAM figures and the top stall reasons.
ncu -i X.ncu-rep --page raw --csv > raw.csv; python tools/ncu_plan_brief.py raw.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    agg = collections.OrderedDict()
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d["Kernel Name"].split("(")[0][-60:]
        t = float(d["gpu__time_duration.sum"])
        a = agg.setdefault(name, {"n": 0, "t": 0.0, "best": None, "tb": -1.0})
        a["n"] += 1
        a["t"] += t
        if t > a["tb"]:
            a["tb"], a["best"] = t, d
    tot = sum(a["t"] for a in agg.values())
    print(f"total {tot:.1f} us")
    for name, a in sorted(agg.items(), key=lambda x: -x[1]["t"]):
        d = a["best"]

        def g(k):
            try:
                return float(d[k])
            except (KeyError, ValueError):
                return float("nan")
        st = []
        for k in h:
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    st.append((float(d[k]), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        st = ", ".join(f"{n} {v:.1f}" for v, n in sorted(st, reverse=True)[:4] if n != "selected")
        print(f"{a['t']:8.1f} us n={a['n']:3d} max {a['tb']:6.1f}  issue {g('smsp__issue_active.avg.pct_of_peak_sustained_active'):4.0f}% "
              f"warps {g('sm__warps_active.avg.pct_of_peak_sustained_active'):4.0f}% dram {g('dram__throughput.avg.pct_of_peak_sustained_elapsed'):4.0f}% "
              f"grid {d.get('launch__grid_size', '?'):>6s} regs {d.get('launch__registers_per_thread', '?'):>3s}  {name}\n             stalls: {st}")


if __name__ == "__main__":
    main(sys.argv[1])
