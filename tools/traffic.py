"""ncu metric CSV of tools/one_step.py -> per-kernel launches, DRAM bytes and
time of the second (measured) step; writes a JSON summary.
usage: traffic.py traffic.csv out.json <launches per step (one_step.py prints it)>"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
recs = defaultdict(dict)
for r in rows[1:]:
    if r[ix["Metric Name"]] not in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        continue
    lid = int(r[ix["ID"]])
    name = r[ix["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
    val = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3,
             "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1)
    recs[lid]["name"] = name
    recs[lid][r[ix["Metric Name"]]] = val * scale
ids = sorted(recs)
per_step = int(sys.argv[3]) if len(sys.argv) > 3 else len(ids) // 2
half = ids[-per_step:]  # the last (second, measured) step
agg = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
for i in half:
    a = agg[recs[i]["name"]]
    a["launches"] += 1
    a["dram_bytes"] += recs[i].get("dram__bytes_read.sum", 0) + recs[i].get("dram__bytes_write.sum", 0)
    a["ms"] += recs[i].get("gpu__time_duration.sum", 0)
out = {k: dict(v, per_launch_bytes=v["dram_bytes"] / v["launches"]) for k, v in agg.items()}
json.dump(out, open(sys.argv[2], "w"), indent=1, sort_keys=True)
tot = sum(v["ms"] for v in out.values())
for k, v in sorted(out.items(), key=lambda x: -x[1]["ms"]):
    print(f"{k:22s} {v['launches']:4d} {v['ms']:8.3f} ms {100 * v['ms'] / tot:5.1f}%  dram {v['dram_bytes'] / 1e6:9.1f} MB")
