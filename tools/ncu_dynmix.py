"""Dynamic SASS instruction mix of one kernel from an ncu report's source page:
python tools/ncu_dynmix.py <report.ncu-rep> [kernel substring] [top N]
Prints executed warp instructions per opcode and the stall samples per opcode."""
import csv
import io
import re
import subprocess
import sys
from collections import Counter


def main(rep, pat="", top=40):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'(?m)^"Kernel Name",', out)
    for b in blocks[1:]:
        name = b.split("\n", 1)[0]
        if pat not in name:
            continue
        rows = list(csv.DictReader(io.StringIO(b.split("\n", 1)[1])))
        ex, st = Counter(), Counter()
        for r in rows:
            op = re.sub(r"^@!?U?P\w+\s+", "", r["Source"].strip()).split(" ")[0]
            ex[op] += int(r["Instructions Executed"] or 0)
            st[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
        tot = sum(ex.values())
        mufu = ex.get("MUFU.RSQ64H", 0) or 1
        fp64 = sum(v for k, v in ex.items() if k.split(".")[0] in ("DFMA", "DMUL", "DADD", "DSETP"))
        print(name[:100])
        print(f"  executed {tot:.4g} warp inst, {tot / mufu:.2f} per RSQ64H, FP64 {fp64 / mufu:.2f} per RSQ64H")
        for k, v in ex.most_common(int(top)):
            print(f"  {k:28s} {v / mufu:7.3f}  stall {st[k] / max(sum(st.values()), 1):.3f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
