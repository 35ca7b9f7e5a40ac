"""top stall-sampled SASS lines of an `ncu --page source --csv` export"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, r in enumerate(rows) if 'Source' in r and any(c.startswith('Warp Stall Sampling') for c in r))
h = rows[hi]
i_s = next(j for j, c in enumerate(h) if c.startswith('Warp Stall Sampling (All'))
i_i = next(j for j, c in enumerate(h) if c.startswith('Instructions Executed'))
data = []
for r in rows[hi + 1:]:
    try:
        data.append((float(r[i_s] or 0), float(r[i_i] or 0), r[0], r[1][:100]))
    except (ValueError, IndexError):
        pass
ts = sum(d[0] for d in data) or 1
ti = sum(d[1] for d in data) or 1
print(f"total instructions {ti:.3g}")
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0] / ts * 100:5.1f}% stall {d[1] / ti * 100:5.1f}% inst  {d[2][-5:]} {d[3]}")
