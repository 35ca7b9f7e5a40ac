import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle.ckks import Ckks
from paper_2110_08321_b200 import hegpu as H
DELTA = 2.0 ** 40
qb = [60, 40, 40, 40, 40]
ctx = H.Context(10, qb, 60, seed=21)
ck = Ckks(10, qb, 60, seed=21)
N = 1024
pr = [int(x) for x in ctx.primes]
for (m, n, l, B) in [(64, 400, 4, 16), (100, 300, 4, 16)]:
    rng = np.random.default_rng(m + n + B)
    A = rng.normal(0, 0.05, (m, n))
    cts = [ck.encrypt(ck.encode(rng.uniform(-1, 1, n), DELTA, l), l, 500 + i) for i in range(B)]
    plan = ctx.hs_plan(A, l, True)
    ctx.gen_rotation_keys(plan.rotations())
    dv = ctx.ct(B, l, np.concatenate(cts), DELTA)
    words = ctx.hs_acc_words(plan, B)
    a1 = torch.zeros(words, dtype=torch.int64, device="cuda")
    ctx.hs_matvec_partial(plan, dv, 0, 1, a1); ctx.sync()
    a2 = torch.zeros(words, dtype=torch.int64, device="cuda")
    for p in range(2):
        part = torch.empty(words, dtype=torch.int64, device="cuda")
        ctx.hs_matvec_partial(plan, dv, p, 2, part); ctx.sync(); a2 += part
    a1 = a1.cpu().numpy().view(np.uint64); a2 = a2.cpu().numpy().view(np.uint64)
    na = B * 2 * (l + 1) * N
    acc1 = a1[:na].reshape(B, 2, l + 1, N); acc2 = a2[:na].reshape(B, 2, l + 1, N)
    cac2 = a2[na:].reshape(B, 2, l, N)
    P = pr[-1] if len(pr) > 5 else None
    Pm = pr[len(qb)]
    want = acc2.copy()
    for t in range(l + 1):
        q = pr[t] if t < l else Pm
        w = [int(x) % q for x in acc2[:, :, t, :].ravel()]
        if t < l:
            c = [int(x) for x in cac2[:, 0, t, :].ravel()]
            w0 = [(int(x) + Pm % q * cc) % q for x, cc in zip(acc2[:, 0, t, :].ravel(), c)]
            want[:, 0, t, :] = np.array(w0, dtype=np.uint64).reshape(B, N)
            want[:, 1, t, :] = np.array([int(x) % q for x in acc2[:, 1, t, :].ravel()], dtype=np.uint64).reshape(B, N)
        else:
            want[:, :, t, :] = np.array(w, dtype=np.uint64).reshape(B, 2, N)
    diff = acc1 != want
    print((m, n, l, B), "diff count", diff.sum(), flush=True)
    if diff.sum():
        idx = np.argwhere(diff)
        print(" by b", np.unique(idx[:, 0])[:20], " by p", np.unique(idx[:, 1]), " by t", np.unique(idx[:, 2]))
        ks = np.unique(idx[:, 3]); print(" k count", len(ks), ks[:40], ks[-10:])
