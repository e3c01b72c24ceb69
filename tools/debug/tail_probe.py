"""Spread of the persistent evaluation kernels' CTA exit times (the tail): run one config
with a library built with -DCSFS_TAIL_PROBE (CSFS_B200_LIB) and summarise its printf lines
(read from stdin): python tools/debug/tail_probe.py < log"""
import collections
import sys

t = collections.defaultdict(list)
for line in sys.stdin:
    p = line.split()
    if len(p) == 4 and p[0] == "TAIL":
        t[p[1]].append(int(p[3]))
for k, v in t.items():
    v.sort()
    n = len(v)
    print(f"{k}: {n} CTAs, exit spread {(v[-1] - v[0]) / 1e3:.1f} us, median-to-last {(v[-1] - v[n // 2]) / 1e3:.1f} us")
