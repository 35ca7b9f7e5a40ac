"""GPU parity at the sizes BASELINE.json states for configs 1, 3 and 4
(ring degree N = 16384): ciphertext limbs from the CUDA path, called through
the C-ABI, are bit-identical to the CPU oracle's on the same keys, nonces
and plaintexts, and the decrypted slots match the cleartext computation.

  config 1: HS matvec m = n = 1024 in full (one ciphertext, and a batch of
            8 on the int8 tensor-core kernel); m = n = 4096 through one
            diagonal range of the partial-sum API (hs_matvec_partial +
            finish, the multi-GPU split) against the oracle's hoisted sum
            over the same range (proj/tests/test_matvec.cpp:110-123 is the
            reference's own at-size HS check);
  config 3: the whole CIFAR-shaped network for one image at L = 6
            (proj/tests/test_netcompile.cpp:173-189 checks execute against
            ref_forward);
  config 4: the conv-pack layer at (c_in, k, c_out) = (32, 5, 64) -- the
            3-maps-per-tile tensor-core conv -- and the reference's
            (3, 3, 18) first-layer case (proj/tests/test_convlower.cpp:63-96).
"""
import numpy as np
import pytest

from oracle import ckks_pipeline as P
from oracle import hesim_oracle as HS
from oracle.ckks import Ckks
from paper_2110_08321_b200 import hegpu as H
from paper_2110_08321_b200.workloads import CFG3, conv_pack_image, hs_sweep_case, net_image, net_weights

pytestmark = pytest.mark.gpu

DELTA = 2.0 ** 40
# N = 16384, one rescale (BASELINE.json configs[1]): the bench's chain
# (45-bit q_0 and P: every limb on the FP64 NTT path) and a 60-bit one (q_0
# and P on the integer path)
CFG1 = (14, [45, 40], 45)
CFG1_60 = (14, [60, 40], 60)


@pytest.fixture(scope="module", params=[CFG1, CFG1_60], ids=["q45", "q60"])
def cfg1(request):
    log_n, qb, pb = request.param
    ctx = H.Context(log_n, qb, pb, seed=1)
    ck = Ckks(log_n, qb, pb, seed=1)
    assert ctx.primes == ck.primes
    return ctx, ck


def _oracle_keys(ck, keys, rights):
    out = []
    for r in rights:
        g = ck.galois_right(r)
        if g not in keys:
            keys[g] = ck.galois_key(g)
        out.append(keys[g])
    return np.concatenate(out) if out else np.zeros(1, dtype=np.uint64)


def test_cfg1_hs_1024_full(cfg1):
    ctx, ck = cfg1
    A, x = hs_sweep_case(1024, 1024)
    v = ck.encrypt(ck.encode(x, DELTA, 2), 2, 1)
    plan = ctx.hs_plan(A, 2)
    assert (plan.m_eff, plan.folds, plan.kept) == (1024, 1, 1024)
    ctx.gen_rotation_keys(plan.rotations())
    out = ctx.ct(1, 1)
    ctx.reset_meter()
    got = ctx.hs_matvec(plan, ctx.ct(1, 2, v, DELTA), out).download()
    assert ctx.total() == (0, 1024, 1024, 0, 1024)  # predict_hs(1024, 1024, 16384): 1024 rotations
    keys = {}
    want = P.hs_matvec(ck, v, 2, A, keys=keys)
    assert np.array_equal(got, want)
    assert np.abs(ck.decrypt_decode(got, 1, DELTA)[:1024] - A @ x).max() < 1e-4
    # a batch of 8 takes the tensor-core kernel (hs_imma.cu) at this size
    B = 8
    rng = np.random.default_rng(5)
    xs = [rng.uniform(-1, 1, 1024) for _ in range(B)]
    cts = [ck.encrypt(ck.encode(z, DELTA, 2), 2, 10 + i) for i, z in enumerate(xs)]
    outb = ctx.ct(B, 1)
    gotb = ctx.hs_matvec(plan, ctx.ct(B, 2, np.concatenate(cts), DELTA), outb).download().reshape(B, -1)
    for i in (0, B - 1):
        assert np.array_equal(gotb[i], P.hs_matvec(ck, cts[i], 2, A, keys=keys)), i
    for i in range(B):
        assert np.abs(ck.decrypt_decode(gotb[i], 1, DELTA)[:1024] - A @ xs[i]).max() < 1e-4


def test_cfg1_hs_64x4096_grouped_folds(cfg1):
    """m = 64, n = 4096: 7 fold doublings, run as two hoisted fold groups
    (4 + 3 doublings: 15 + 7 key inner products instead of 127), limbs ==
    oracle, metering = the reference's 64 + 7 rotations"""
    ctx, ck = cfg1
    A, x = hs_sweep_case(64, 4096)
    v = ck.encrypt(ck.encode(x, DELTA, 2), 2, 3)
    plan = ctx.hs_plan(A, 2)
    assert (plan.m_eff, plan.folds) == (64, 7)
    assert P.fold_groups(7) == [4, 3]
    ctx.gen_rotation_keys(plan.rotations())
    ctx.reset_meter()
    got = ctx.hs_matvec(plan, ctx.ct(1, 2, v, DELTA), ctx.ct(1, 1)).download()
    assert ctx.total() == (0, 70, 64, 0, 70)  # predict_hs(64, 4096, 16384) = 70 (test_matvec.cpp:125-131)
    assert np.array_equal(got, P.hs_matvec(ck, v, 2, A))
    assert np.abs(ck.decrypt_decode(got, 1, DELTA)[:64] - A @ x).max() < 1e-4


def test_cfg1_hs_4096_partial_range(cfg1):
    """m = n = 4096: diagonal range 0 of 8 (512 diagonals) through the
    partial-sum API, finished alone, against the oracle's hoisted sum over
    the same 512 diagonals + rescale + fold"""
    torch = pytest.importorskip("torch")
    ctx, ck = cfg1
    A, x = hs_sweep_case(4096, 4096)
    v = ck.encrypt(ck.encode(x, DELTA, 2), 2, 2)
    plan = ctx.hs_plan(A, 2)
    assert (plan.m_eff, plan.folds, plan.kept) == (4096, 1, 4096)
    ctx.gen_rotation_keys(plan.rotations())
    dv = ctx.ct(1, 2, v, DELTA)
    acc = torch.zeros(ctx.hs_acc_words(plan, 1), dtype=torch.int64, device="cuda")
    nparts, part = 8, 0
    ctx.hs_matvec_partial(plan, dv, part, nparts, acc)
    got = ctx.hs_matvec_finish(plan, dv, acc, 1, ctx.ct(1, 1)).download()
    # oracle: the same kept-diagonal range (capi.cu: kept * part / nparts)
    m_eff, folds, rots, masks = P.hs_masks(ck, A, 2)
    lo, hi = len(rots) * part // nparts, len(rots) * (part + 1) // nparts
    per = 3 * ck.N  # (l + 1) limbs per mask
    keys = {}
    kb = _oracle_keys(ck, keys, [r for r in rots[lo:hi] if r != 0])
    u = ck.hs_hoisted(v, 2, np.array(rots[lo:hi], dtype=np.int64), masks[lo * per:hi * per], kb)
    u = ck.rescale(u, 2)

    def key(g):
        if g not in keys:
            keys[g] = ck.galois_key(g)
        return keys[g]

    want = P.fold_sum(ck, u, 1, m_eff, folds, key)
    assert np.array_equal(got, want)
    # the range's share of A x: rows i of diagonal j contribute A[(j + k) mod m, k]
    sub = np.zeros_like(A)
    for j in rots[lo:hi]:
        k = np.arange(4096)
        sub[(j + k) % 4096, k] = A[(j + k) % 4096, k]
    assert np.abs(ck.decrypt_decode(got, 1, DELTA)[:4096] - sub @ x).max() < 1e-4


def test_cfg3_full_net_limbs_one_image():
    """config 3 at its stated size: N = 16384, L = 6 (Q = 60 + 5 x 40 bits),
    the reference first layer (75 conv_pack taps, 32 maps, 31-rotation
    merge), HS 6272 -> 256, HS 256 -> 10: every output limb equals the
    oracle's, logits within 1e-3 of ref_forward"""
    cfg = CFG3
    ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=33)
    ck = Ckks(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=33)
    w = net_weights(cfg, 3)
    img = net_image(cfg, 7)
    net = H.Net(ctx, cfg, w)
    assert net.tap_cts == 75
    out = ctx.ct(1, net.out_level)
    net.run(ctx.ct(net.tap_cts, net.top, net.encrypt_image(img, nonce=4), DELTA), out)
    got = out.download()
    want, _ = P.run_net(ck, cfg, w, img, nonce=4)
    assert np.array_equal(got, want)
    spec = HS.CnnSpec(cfg.in_c, cfg.in_d, cfg.k, cfg.s, cfg.c_out, cfg.dense, cfg.n_slots)
    assert np.abs(net.decrypt_logits(got) - HS.ref_forward(spec, w, img)).max() < 1e-3


def _conv_np(img, W, b, s=1):
    c_out, c_in, k, _ = W.shape
    d_out = (img.shape[1] - k) // s + 1
    out = np.zeros((c_out, d_out, d_out)) + np.asarray(b)[:, None, None]
    for ci in range(c_in):
        for ky in range(k):
            for kx in range(k):
                win = img[ci, ky:ky + s * d_out:s, kx:kx + s * d_out:s]
                out += W[:, ci, ky, kx][:, None, None] * win[None]
    return out


@pytest.mark.parametrize("c_in,k,c_out,kcb", [(32, 5, 64, None), (3, 3, 18, None), (3, 5, 32, None),
                                               (3, 3, 18, "32"), (3, 3, 18, "96")])
def test_cfg4_conv_layer_at_size(c_in, k, c_out, kcb, monkeypatch):
    """config 4: c_in x 32 x 32 U[0,1], stride 1, N = 16384, taps at level 2
    (the bench's chain); conv_packed_forward + rescale limbs == oracle, HOPs
    k^2 c_in c_out / (k^2 c_in - 1) c_out / c_out, decrypted maps vs the
    FP64 conv.  (3, 5, 32) is config 3's first layer (75 taps: the tcgen05
    conv's tap ring runs in K chunks); kcb forces K chunks of that many bytes
    on the 27-tap case (HEGPU_TC_KCB)"""
    if kcb is not None:
        monkeypatch.setenv("HEGPU_TC_KCB", kcb)
    ctx = H.Context(14, [45, 40], 45, seed=4)
    ck = Ckks(14, [45, 40], 45, seed=4)
    rng = np.random.default_rng(40 + c_in * k + c_out)
    img = rng.uniform(0, 1, (c_in, 32, 32))
    W = rng.normal(0, 0.05, (c_out, c_in, k, k))
    b = rng.normal(0, 0.01, c_out)
    d_out = 32 - k + 1
    w_used = d_out * d_out
    ntaps = k * k * c_in
    taps = conv_pack_image(img, k)
    assert len(taps) == ntaps
    cts = np.concatenate([ck.encrypt(ck.encode(t, DELTA, 2), 2, i) for i, t in enumerate(taps)])
    out = ctx.ct(c_out, 1)
    ctx.reset_meter()
    got = ctx.conv_packed_forward(ctx.ct(ntaps, 2, cts, DELTA), ntaps, W.reshape(c_out, -1), b, w_used,
                                  out).download()
    assert ctx.total() == (c_out, (ntaps - 1) * c_out, ntaps * c_out, 0, 0)
    want = P.conv_layer(ck, cts, ntaps, 2, W.reshape(c_out, -1), b, w_used, DELTA)
    assert np.array_equal(got, want)
    ref = _conv_np(img, W, b)
    per = 2 * ck.N
    for co in (0, c_out // 2, c_out - 1):
        dec = ck.decrypt_decode(got[co * per:(co + 1) * per], 1, DELTA)[:w_used]
        assert np.abs(dec - ref[co].ravel()).max() < 1e-5, co


@pytest.mark.parametrize("l", [7, 8])
def test_hs_tensor_core_at_levels_7_and_8(l):
    """the grouped HS stages of the `ce` builtin run at level 7 (L = 9): the
    tcgen05 HS kernel is instantiated up to level 8 (J = l + 1 <= 9); a
    batch of 8 images equals the single-ciphertext (integer kernel) runs and
    the CPU oracle"""
    from oracle import ckks_pipeline as P
    from oracle.ckks import Ckks
    from paper_2110_08321_b200 import hegpu as H
    qb = [45] + [40] * 8
    ctx = H.Context(11, qb, 45, seed=19)
    ck = Ckks(11, qb, 45, seed=19)
    rng = np.random.default_rng(100 + l)
    m, n, B = 48, 300, 8
    A = rng.normal(0, 0.05, (m, n))
    zs = [rng.uniform(-1, 1, n) for _ in range(B)]
    cts = [ck.encrypt(ck.encode(z, 2.0 ** 40, l), l, 900 + i) for i, z in enumerate(zs)]
    plan = ctx.hs_plan(A, l, True)
    ctx.gen_rotation_keys(plan.rotations())
    got = ctx.hs_matvec(plan, ctx.ct(B, l, np.concatenate(cts), 2.0 ** 40), ctx.ct(B, l - 1)).download().reshape(B, -1)
    for i in (0, B - 1):
        one = ctx.hs_matvec(plan, ctx.ct(1, l, cts[i], 2.0 ** 40), ctx.ct(1, l - 1)).download()
        assert np.array_equal(got[i], one), i
    assert np.array_equal(got[3], P.hs_matvec(ck, cts[3], l, A, True))
    for i in range(B):
        assert np.abs(ck.decrypt_decode(got[i], l - 1, 2.0 ** 40)[:m] - A @ zs[i]).max() < 1e-4
