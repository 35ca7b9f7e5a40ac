"""One device step of the bench workload (cfg 2: 64 x cfg0 net), direct
launches, after one warm-up step -- the target for per-kernel ncu metric
passes (DRAM traffic of every kernel of the step):
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --csv --log-file traffic.csv python tools/one_step.py
(the first step's launches are the warm-up; tools/traffic.py keeps the second)"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2110_08321_b200 import hegpu as H  # noqa: E402
from paper_2110_08321_b200.workloads import CFG0, net_image, net_weights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = CFG0
ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=2110)
net = H.Net(ctx, cfg, net_weights(cfg, 2110))
taps = np.concatenate([net.encrypt_image(net_image(cfg, i), nonce=i) for i in range(B)])
dt = ctx.ct(B * net.ntaps, net.top, taps, 2.0 ** 40)
out = ctx.ct(B, net.out_level)
for _ in range(2):
    ctx.reset_meter()
    l0 = ctx.launches()
    net.run(dt, out)
    ctx.sync()
print("launches per step", ctx.launches() - l0, flush=True)
