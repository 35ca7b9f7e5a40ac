"""Timing probe of the HS accumulation kernel alone on the config-2 HS1
shape (100 x 845 at level 4, N = 8192, 64 images): prints the k_hs_imma
kernel-timer ms for the current HEGPU_* environment (HEGPU_HT_DBG runs give
wrong limbs on purpose -- timing only)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_08321_b200 import hegpu as H  # noqa: E402
from paper_2110_08321_b200.workloads import QBITS_45, PBITS_45  # noqa: E402

ctx = H.Context(13, list(QBITS_45), PBITS_45, seed=5)
rng = np.random.default_rng(1)
A = rng.normal(0, 0.05, (100, 845))
plan = ctx.hs_plan(A, 4)
ctx.gen_rotation_keys(plan.rotations())
B = 64
x = rng.uniform(-1, 1, 845)
v = ctx.ct(B, 4, np.concatenate([ctx.encrypt(ctx.encode(x, 2.0 ** 40, 4), 4, i) for i in range(B)]), 2.0 ** 40)
out = ctx.ct(B, 3)
ctx.hs_matvec(plan, v, out)
ctx.kernel_timer("k_hs_imma")
for _ in range(5):
    ctx.hs_matvec(plan, v, out)
ms, n, _ = ctx.kernel_timer_read()
print("HEGPU_HT_DBG=%s k_hs_imma %.4f ms per matvec batch" % (os.environ.get("HEGPU_HT_DBG", "0"), ms / 5))
