"""print step ms and per-kernel ms of bench.py JSON lines (A/B helper)"""
import json
import sys

for path in sys.argv[1:]:
    try:
        d = json.loads(open(path).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(path, "unreadable", e)
        continue
    ks = d.get("kernels", {})
    print(f"{path}: step {d['ms_per_step']:.3f} ms  " +
          "  ".join(f"{k[2:]} {v['ms_per_step']:.3f}" for k, v in sorted(ks.items(), key=lambda kv: -kv[1]['ms_per_step'])))
