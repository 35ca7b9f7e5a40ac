"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share (cold-cache,
serialised: compare SHARES, not absolutes)."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':28s} {'launches':>8s} {'total us':>10s} {'share':>6s} {'avg us':>8s}"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{k:28s} {n:8d} {t / 1e3:10.1f} {100 * t / tot:5.1f}% {t / n / 1e3:8.1f}")
    out.append(f"{'TOTAL':28s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.1f}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"== {p}")
        print(summarize(p))
