import sys, numpy as np
sys.path.insert(0, '.')
from oracle.ckks import Ckks
from paper_2110_08321_b200 import hegpu as H
DELTA = 2.0 ** 40
ctx = H.Context(10, [60, 40, 40, 40, 40], 60, seed=21)
ck = Ckks(10, [60, 40, 40, 40, 40], 60, seed=21)
for (m, n, l, B) in [(100, 300, 4, 16), (100, 400, 4, 16), (100, 400, 4, 33), (128, 128, 4, 16), (100, 400, 3, 16), (64, 400, 4, 16), (100, 400, 2, 16)]:
    rng = np.random.default_rng(m + n + B)
    A = rng.normal(0, 0.05, (m, n))
    cts = [ck.encrypt(ck.encode(rng.uniform(-1, 1, n), DELTA, l), l, 500 + i) for i in range(B)]
    plan = ctx.hs_plan(A, l, True)
    ctx.gen_rotation_keys(plan.rotations())
    got = ctx.hs_matvec(plan, ctx.ct(B, l, np.concatenate(cts), DELTA), ctx.ct(B, l - 1)).download().reshape(B, -1)
    bad = []
    for i in range(B):
        one = ctx.hs_matvec(plan, ctx.ct(1, l, cts[i], DELTA), ctx.ct(1, l - 1)).download()
        if not np.array_equal(got[i], one):
            bad.append((i, int(np.sum(got[i] != one))))
    print((m, n, l, B), "m_eff/folds/kept", plan.m_eff, plan.folds, plan.kept, "bad", bad[:6], flush=True)
