"""Summarise an ncu --page source --csv (SASS) export: instructions executed
and warp-stall samples per opcode, and the hottest instructions."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
by_op = defaultdict(lambda: [0, 0])
hot = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ex = int(r[ix["Instructions Executed"]] or 0)
    st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    by_op[op][0] += ex
    by_op[op][1] += st
    hot.append((st, ex, r[ix["Address"]][-5:], src))
tot_ex = sum(v[0] for v in by_op.values())
tot_st = sum(v[1] for v in by_op.values())
print(f"total executed {tot_ex}  stall samples {tot_st}")
for op, (ex, st) in sorted(by_op.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{op:10s} exec {ex:12d} {100*ex/tot_ex:5.1f}%   stall {100*st/max(tot_st,1):5.1f}%")
print("hottest:")
for st, ex, a, src in sorted(hot, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{st:7d} {ex:10d} {a} {src[:90]}")
