"""Instruction mix of the hottest loop (the backward branch enclosing the most MUFU) of a
kernel in a cuobjdump -sass listing: python tools/sass_loop.py <sass file> <name substring>."""
import re
import sys
from collections import Counter


def main(path, pat):
    txt = open(path).read()
    for f in re.split(r"\n\s+Function : ", txt):
        name = f.split("\n")[0]
        if pat not in name:
            continue
        addr = []
        for l in f.split("\n"):
            m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
            if m:
                addr.append((int(m.group(1), 16), m.group(2).strip()))
        best = None
        for a, ins in addr:
            m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", ins)
            if m and m.group(1) and int(m.group(1), 16) < a:
                tgt = int(m.group(1), 16)
                body = [x for (b, x) in addr if tgt <= b <= a]
                n = sum("MUFU" in x for x in body)
                if best is None or n > best[0]:
                    best = (n, body)
        n, body = best
        c = Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0] for x in body)
        fp64 = sum(v for k, v in c.items() if k.split(".")[0] in ("DFMA", "DMUL", "DADD", "DSETP"))
        print(name[:110])
        print(f"  MUFU/loop {n}  instructions {len(body)}  fp64 {fp64}  per MUFU: inst {len(body)/max(n,1):.2f} fp64 {fp64/max(n,1):.2f}")
        print("  ", sorted(c.items(), key=lambda kv: -kv[1]))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
