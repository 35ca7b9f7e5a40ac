"""ncu SASS source export -> runs of instructions with equal execution
counts (basic blocks), ranked by executed instructions, with stall share"""
import csv
import sys
from collections import Counter
from itertools import groupby

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [(int(r[ix["Instructions Executed"]] or 0), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0),
         r[ix["Address"]][-5:], r[ix["Source"]].strip()) for r in rows[2:] if len(r) >= len(hdr)]
segs = []
for k, g in groupby(data, key=lambda x: x[0]):
    g = list(g)
    ops = [x[3].split()[1] if x[3].startswith("@") else x[3].split()[0] for x in g]
    segs.append((k, len(g), g[0][2], g[-1][2], sum(x[1] for x in g), ops))
tot = sum(s[0] * s[1] for s in segs)
totst = sum(s[4] for s in segs)
for k, n, a, b, st, ops in sorted(segs, key=lambda s: -s[0] * s[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(k, n, f"{100 * k * n / tot:.1f}%", f"stall {100 * st / totst:.1f}%", a, b,
          Counter(o.split(".")[0] for o in ops).most_common(7))
