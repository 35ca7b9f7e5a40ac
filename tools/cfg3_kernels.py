"""per-kernel device time of one config-3 step (CIFAR-shaped net, batch 16)"""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_08321_b200 import hegpu as H
from paper_2110_08321_b200.workloads import CFG3, net_image, net_weights
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = CFG3
ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=3)
net = H.Net(ctx, cfg, net_weights(cfg, 3))
taps = np.concatenate([net.encrypt_image(net_image(cfg, i), nonce=i) for i in range(B)])
dt = ctx.ct(B * net.ntaps, net.top, taps, 2.0 ** 40)
out = ctx.ct(B, net.out_level)
net.run(dt, out); ctx.sync()
tot = 0
for k in ["k_hs_diag", "k_hs_imma", "k_drop_ntt", "k_md_ntt", "k_md_intt", "k_ks_modup", "k_conv_mac", "k_intt_rows",
          "k_ks_intt", "k_ks_inner", "k_add", "k_tensor_square", "k_add_plain", "k_sum_parts", "k_merge_c"]:
    ctx.kernel_timer(k)
    net.run(dt, out)
    ms, n, b, o = ctx.kernel_timer_read_ops()
    tot += ms
    print(f"{k:16s} {ms:8.3f} ms {n:4d} launches {b / (ms / 1e3) / 1e9 if ms else 0:8.1f} GB/s {o / (ms / 1e3) / 1e9 if ms else 0:8.1f} Gmodmul/s")
print("sum", tot)
