"""GPU parity: every CUDA op, called through the C-ABI, against the CPU
oracle on identical inputs -- ciphertext limbs must be bit-identical -- and
the decrypted slots against the reference slot semantics (oracle/
hesim_oracle.py, restating proj/src/*.cpp)."""
import numpy as np
import pytest

from oracle import hesim_oracle as HS
from oracle.ckks import Ckks
from paper_2110_08321_b200 import hegpu as H
from paper_2110_08321_b200.workloads import CFG0, hs_sweep_case, net_image, net_weights
from oracle import ckks_pipeline as P

pytestmark = pytest.mark.gpu

SMALL = (10, [60, 40, 40, 40, 40], 60)   # N = 1024, S = 512
DELTA = 2.0 ** 40


@pytest.fixture(scope="module")
def pair():
    log_n, qb, pb = SMALL
    ctx = H.Context(log_n, qb, pb, seed=21)
    ck = Ckks(log_n, qb, pb, seed=21)
    assert ctx.primes == ck.primes
    return ctx, ck


def fresh(ck, rng, level, nonce, n=None, scale=DELTA):
    z = rng.uniform(-1, 1, n or ck.S)
    return z, ck.encrypt(ck.encode(z, scale, level), level, nonce)


def test_upload_download_roundtrip(pair):
    ctx, ck = pair
    rng = np.random.default_rng(0)
    _, c = fresh(ck, rng, 5, 1)
    d = ctx.ct(1, 5, c, DELTA)
    assert np.array_equal(d.download(), c)
    p = ck.encode(rng.uniform(-1, 1, ck.S), DELTA, 3, with_p=True)
    dp = ctx.pt(1, 3, True, p, DELTA)
    assert np.array_equal(dp.download(), p)


def test_compact_upload_regenerates_c1(pair):
    """compact taps (c0 + a-stream keys) expand on the device to exactly the
    oracle's fresh ciphertexts"""
    ctx, ck = pair
    rng = np.random.default_rng(11)
    L = ck.L
    pts = [ck.encode(rng.uniform(-1, 1, ck.S), DELTA, L) for _ in range(3)]
    blob = np.concatenate([ctx.encrypt_compact(p, L, nonce=40 + i) for i, p in enumerate(pts)])
    d = ctx.ct(3, L)
    d.upload_compact(blob, DELTA)
    want = np.concatenate([ck.encrypt(p, L, 40 + i) for i, p in enumerate(pts)])
    assert np.array_equal(d.download(), want)


def test_add_mul_plain(pair):
    ctx, ck = pair
    rng = np.random.default_rng(1)
    l = 4
    za, a = fresh(ck, rng, l, 2)
    zb, b = fresh(ck, rng, l, 3)
    zp = rng.uniform(-1, 1, ck.S)
    p = ck.encode(zp, float(ck.primes[l - 1]), l)
    da, db = ctx.ct(1, l, a, DELTA), ctx.ct(1, l, b, DELTA)
    dp = ctx.pt(1, l, False, p, float(ck.primes[l - 1]))
    out = ctx.ct(1, l)
    assert np.array_equal(ctx.add(da, db, out).download(), ck.add(a, b, l))
    assert np.array_equal(ctx.add_plain(da, dp, out).download(), ck.add_pc(a, p, l))
    got = ctx.mul_plain(da, dp, out).download()
    assert np.array_equal(got, ck.mul_pc(a, p, l))
    r = ctx.ct(1, l - 1)
    ctx.rescale(out, r)
    want = ck.rescale(ck.mul_pc(a, p, l), l)
    assert np.array_equal(r.download(), want)
    assert np.abs(ck.decrypt_decode(want, l - 1, DELTA) - za * zp).max() < 1e-6


@pytest.mark.parametrize("r", [1, 7, 255, 511])
def test_rotate_right_bit_exact(pair, r):
    ctx, ck = pair
    rng = np.random.default_rng(r)
    l = 4
    z, a = fresh(ck, rng, l, 10 + r)
    ctx.gen_rotation_keys([r])
    out = ctx.ct(1, l)
    got = ctx.rotate_right(ctx.ct(1, l, a, DELTA), r, out).download()
    want = ck.rotate(a, l, ck.galois_right(r), ck.galois_key(ck.galois_right(r)))
    assert np.array_equal(got, want)
    # slot semantics: out[j] = v[(j - r) mod S] (proj/src/slotvec.cpp:42-57)
    assert np.abs(ck.decrypt_decode(got, l, DELTA) - np.roll(z, r)).max() < 1e-6


def test_rotate_left_and_zero(pair):
    ctx, ck = pair
    rng = np.random.default_rng(5)
    l = 3
    z, a = fresh(ck, rng, l, 40)
    ctx.gen_rotation_keys([ck.S - 3])
    da, out = ctx.ct(1, l, a, DELTA), ctx.ct(1, l)
    ctx.reset_meter()
    got = ctx.rotate_left(da, 3, out).download()
    want = ck.rotate(a, l, ck.galois_left(3), ck.galois_key(ck.galois_left(3)))
    assert np.array_equal(got, want)
    assert np.abs(ck.decrypt_decode(got, l, DELTA) - np.roll(z, -3)).max() < 1e-6
    assert np.array_equal(ctx.rotate_right(da, 0, out).download(), a)  # free no-op
    assert ctx.total() == (0, 0, 0, 0, 1)
    with pytest.raises(H.RangeError):
        ctx.rotate_right(da, ck.S, out)
    with pytest.raises(H.RangeError):
        ctx.rotate_right(da, -1, out)
    with pytest.raises(H.HegpuError) as e:
        ctx.rotate_right(da, 77, out)
    assert e.value.code == H.ERR_KEY


def test_square_relin_rescale(pair):
    ctx, ck = pair
    rng = np.random.default_rng(6)
    l = 5
    z, a = fresh(ck, rng, l, 50)
    ctx.gen_relin_key()
    out = ctx.ct(1, l - 1)
    got = ctx.square(ctx.ct(1, l, a, DELTA), out).download()
    want = ck.rescale(ck.square(a, l, ck.relin_key()), l)
    assert np.array_equal(got, want)
    s = DELTA * DELTA / ck.primes[l - 1]
    assert abs(out.scale - s) / s < 1e-15
    assert np.abs(ck.decrypt_decode(got, l - 1, s) - z * z).max() < 1e-6


def test_batched_ops_match_per_ciphertext(pair):
    ctx, ck = pair
    rng = np.random.default_rng(7)
    l, B, r = 4, 3, 5
    cts = [fresh(ck, rng, l, 60 + i)[1] for i in range(B)]
    ctx.gen_rotation_keys([r])
    ctx.gen_relin_key()
    d = ctx.ct(B, l, np.concatenate(cts), DELTA)
    out = ctx.ct(B, l)
    got = ctx.rotate_right(d, r, out).download().reshape(B, -1)
    key = ck.galois_key(ck.galois_right(r))
    for i in range(B):
        assert np.array_equal(got[i], ck.rotate(cts[i], l, ck.galois_right(r), key))
    sq = ctx.ct(B, l - 1)
    got = ctx.square(d, sq).download().reshape(B, -1)
    rlk = ck.relin_key()
    for i in range(B):
        assert np.array_equal(got[i], ck.rescale(ck.square(cts[i], l, rlk), l))


@pytest.mark.parametrize("c_out", [4, 7, 11])  # 7, 11: the 3-maps-per-tile layout on the 40-bit limbs
def test_conv_packed_forward(pair, c_out):
    ctx, ck = pair
    rng = np.random.default_rng(8 + c_out)
    # a 1x12x12 image, 3x3 kernel, stride 1 -> d_out 10 (w = 100 slots)
    cfg = type("C", (), dict(in_c=1, in_d=12, k=3, s=1, c_out=c_out))
    img = rng.uniform(0, 1, (1, 12, 12))
    W = rng.normal(0, 0.05, (c_out, 1, 3, 3))
    bias = rng.normal(0, 0.01, c_out)
    L = ck.L
    taps = P.conv_pack_taps(ck, cfg, img, 3, DELTA, merged=False)  # the standalone per-map conv API
    dt = ctx.ct(9, L, taps, DELTA)
    out = ctx.ct(c_out, L - 1)
    ctx.reset_meter()
    got = ctx.conv_packed_forward(dt, 9, W.reshape(c_out, 9), bias, 100, out).download()
    want = P.conv_layer(ck, taps, 9, L, W.reshape(c_out, 9), bias, 100, DELTA)
    assert np.array_equal(got, want)
    assert ctx.total() == (c_out, 8 * c_out, 9 * c_out, 0, 0)   # (c_out, (k^2-1) c_out, k^2 c_out, 0, 0)
    plan = ctx.conv_plan(9, W.reshape(c_out, 9), bias, 100, L, DELTA)  # prepared once, same result
    out2 = ctx.ct(c_out, L - 1)
    assert np.array_equal(ctx.conv_plan_run(plan, dt, out2).download(), want)
    ref = HS.ref_conv(img, W, bias, 1)
    per = 2 * (L - 1) * ck.N
    for co in range(c_out):
        dec = ck.decrypt_decode(got[co * per:(co + 1) * per], L - 1, DELTA)
        assert np.abs(dec[:100] - ref[co].ravel()).max() < 1e-6


def test_merge_maps(pair):
    ctx, ck = pair
    rng = np.random.default_rng(9)
    l, c, w = 4, 5, 100
    zs, cts = [], []
    for j in range(c):
        z, ct = fresh(ck, rng, l, 80 + j, n=w)
        zs.append(z)
        cts.append(ct)
    maps = np.concatenate(cts)
    ctx.gen_rotation_keys([j * w for j in range(1, c)])
    out = ctx.ct(1, l)
    ctx.reset_meter()
    got = ctx.merge_maps(ctx.ct(c, l, maps, DELTA), c, w, out).download()
    assert ctx.total() == (0, 4, 0, 0, 4)   # merge 5 maps: 4 rot + 4 add (test_convlower.cpp:171-188)
    want = P.merge(ck, maps, c, l, w)
    assert np.array_equal(got, want)
    dec = ck.decrypt_decode(got, l, DELTA)
    assert np.abs(dec[: c * w] - np.concatenate(zs)).max() < 1e-6
    with pytest.raises(H.CapacityError):
        ctx.merge_maps(ctx.ct(c, l, maps, DELTA), c, 200, out)


@pytest.mark.parametrize("m,n,skip", [(2, 2, True), (10, 100, True), (32, 300, True), (3, 4, False),
                                      (7, 500, True), (4, 4, True),
                                      (2, 100, True), (2, 300, True),  # 6 / 8 folds: two hoisted fold groups
                                      (300, 200, True)])  # padding branch, 4 diagonal chunks, split CTAs
def test_hs_matvec(pair, m, n, skip):
    ctx, ck = pair
    rng = np.random.default_rng(m * 1000 + n)
    l = 3
    A = rng.normal(0, 0.05, (m, n))
    if (m, n) == (4, 4):
        A = np.eye(4)  # zero diagonals skipped (test_matvec.cpp:99-108)
    z, v = fresh(ck, rng, l, 100 + m, n=n)
    plan = ctx.hs_plan(A, l, skip)
    ctx.gen_rotation_keys(plan.rotations())
    out = ctx.ct(1, l - 1)
    ctx.reset_meter()
    got = ctx.hs_matvec(plan, ctx.ct(1, l, v, DELTA), out).download()
    want = P.hs_matvec(ck, v, l, A, skip)
    assert np.array_equal(got, want)
    dec = ck.decrypt_decode(got, l - 1, DELTA)
    assert np.abs(dec[:m] - A @ z).max() < 1e-5
    # metering equals the reference's hs_matvec on the same matrix
    mc = HS.MeterContext()
    HS.hs_matvec(A, HS.pack(z, ck.S, HS.CIPHERTEXT), mc, skip_zero_diagonals=skip)
    assert ctx.total() == mc.tally.as_tuple()


@pytest.mark.parametrize("m,n,l,B", [(10, 100, 3, 8), (32, 300, 3, 17), (300, 200, 3, 16), (4, 4, 3, 8),
                                     (2, 2, 2, 9), (7, 500, 4, 16), (100, 400, 4, 33), (64, 256, 2, 8), (64, 400, 4, 16),
                                     (50, 60, 5, 8)])
def test_hs_matvec_batched_tensor_core(pair, m, n, l, B):
    """batches of >= 8 ciphertexts take the int8 tensor-core HS kernel
    (hs_imma.cu): every image's limbs == the single-ciphertext (integer
    pipe) run and the CPU oracle"""
    ctx, ck = pair
    rng = np.random.default_rng(11 * m + n + B)
    A = np.eye(4) if (m, n) == (4, 4) else rng.normal(0, 0.05, (m, n))
    cts = [fresh(ck, rng, l, 500 + i, n=n) for i in range(B)]
    plan = ctx.hs_plan(A, l, True)
    ctx.gen_rotation_keys(plan.rotations())
    batch = np.concatenate([c for _, c in cts])
    out = ctx.ct(B, l - 1)
    got = ctx.hs_matvec(plan, ctx.ct(B, l, batch, DELTA), out).download().reshape(B, -1)
    for i in (0, B - 1):
        one = ctx.hs_matvec(plan, ctx.ct(1, l, cts[i][1], DELTA), ctx.ct(1, l - 1)).download()
        assert np.array_equal(got[i], one), i
    assert np.array_equal(got[B // 2], P.hs_matvec(ck, cts[B // 2][1], l, A, True))
    for i in range(B):
        dec = ck.decrypt_decode(got[i], l - 1, DELTA)
        assert np.abs(dec[:m] - A @ cts[i][0]).max() < 1e-4


@pytest.mark.parametrize("kind,m,n,B", [("dense", 1, 1, 1), ("dense", 5, 8, 2), ("dense", 3, 100, 1),
                                         ("stacked", 4, 3, 1), ("stacked", 12, 100, 2), ("stacked", 3, 200, 1),
                                         ("stacked", 300, 2, 1)])
def test_lola_matvec(pair, kind, m, n, B):
    """lola_dense / lola_stacked (proj/src/matvec.cpp:107-166) on the GPU:
    limbs == the CPU oracle composition, decrypted slots == the reference's
    slot vector (A x in slot 0 / at slot_of_row, zeros elsewhere), metering
    == predict_lola_* per input"""
    ctx, ck = pair
    rng = np.random.default_rng(13 * m + n)
    l = 4
    A = rng.normal(0, 0.3, (m, n))
    cts = [fresh(ck, rng, l, 900 + i, n=n) for i in range(B)]
    plan = ctx.lola_plan(kind, A, l)
    ctx.gen_rotation_keys(plan.rotations())
    out = ctx.ct(B * plan.per_input, l - 2)
    ctx.reset_meter()
    got = ctx.lola_matvec(plan, ctx.ct(B, l, np.concatenate([c for _, c in cts]), DELTA), out).download()
    per = plan.per_input
    got = got.reshape(B, per, -1)
    N = ck.N
    if kind == "dense":
        want = P.lola_dense(ck, cts[-1][1], l, A).reshape(per, -1)
        assert np.array_equal(got[-1], want)
        pred = HS.predict_lola_dense(m, n)
        for b in range(B):
            for i in range(m):
                dec = ck.decrypt_decode(got[b][i], l - 2, DELTA)
                assert abs(dec[0] - A[i] @ cts[b][0]) < 1e-4
                assert np.abs(dec[1:]).max() < 1e-4
    else:
        want, sor = P.lola_stacked(ck, cts[-1][1], l, A)
        assert np.array_equal(got[-1][0], want)
        assert plan.slot_of_row() == sor
        pred = HS.predict_lola_stacked(m, n, ck.S)
        for b in range(B):
            dec = ck.decrypt_decode(got[b][0], l - 2, DELTA)
            ref = np.zeros(ck.S)
            ref[sor] = A @ cts[b][0]
            assert np.abs(dec - ref).max() < 1e-4
    assert ctx.total()[2] == B * pred[1] and ctx.total()[4] == B * pred[0] and ctx.total()[1] == B * pred[2]


def test_lola_capacity(pair):
    ctx, ck = pair
    with pytest.raises(H.CapacityError):
        ctx.lola_plan("dense", np.ones((2, ck.S + 1)), 4)
    with pytest.raises(H.CapacityError):
        ctx.lola_plan("stacked", np.ones((ck.S + 1, 2)), 4)


@pytest.mark.parametrize("m,n,nparts", [(300, 200, 3), (32, 300, 2), (10, 100, 8), (4, 4, 5)])
def test_hs_matvec_split_partial_sums(pair, m, n, nparts):
    """config-3 style distributed HS: per-part extended-basis accumulators
    over diagonal ranges, summed element-wise (what the NCCL all-reduce
    does), then one finish == the single-GPU hs_matvec bit for bit, with the
    same total metering"""
    import torch
    ctx, ck = pair
    rng = np.random.default_rng(7 * m + n)
    l = 3
    A = np.eye(4) if (m, n) == (4, 4) else rng.normal(0, 0.05, (m, n))
    z, v = fresh(ck, rng, l, 300 + m, n=n)
    plan = ctx.hs_plan(A, l, True)
    ctx.gen_rotation_keys(plan.rotations())
    dv = ctx.ct(1, l, v, DELTA)
    want = ctx.hs_matvec(plan, dv, ctx.ct(1, l - 1)).download()
    ctx.reset_meter()
    words = ctx.hs_acc_words(plan, 1)
    total = torch.zeros(words, dtype=torch.int64, device="cuda")
    for p in range(nparts):
        part = torch.empty(words, dtype=torch.int64, device="cuda")
        ctx.hs_matvec_partial(plan, dv, p, nparts, part)
        ctx.sync()
        total += part
    out = ctx.ct(1, l - 1)
    ctx.hs_matvec_finish(plan, dv, total, nparts, out)
    assert np.array_equal(out.download(), want)
    mc = HS.MeterContext()
    HS.hs_matvec(A, HS.pack(z, ck.S, HS.CIPHERTEXT), mc, skip_zero_diagonals=True)
    assert ctx.total() == mc.tally.as_tuple()


def test_hs_capacity(pair):
    ctx, ck = pair
    with pytest.raises(H.CapacityError):
        ctx.hs_plan(np.ones((4, ck.S + 1)), 3)


@pytest.fixture(scope="module")
def cfg0():
    cfg = CFG0
    ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=1234)
    ck = Ckks(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=1234)
    w = net_weights(cfg, 0)
    net = H.Net(ctx, cfg, w)
    return cfg, ctx, ck, w, net


def test_cfg0_net_bit_exact_and_logits(cfg0):
    """Config 0 end to end: limbs == oracle pipeline, logits within 1e-3 of
    ref_forward (proj/src/netcompile.cpp:448-503), per-stage HOPs == the
    golden table."""
    cfg, ctx, ck, w, net = cfg0
    B = 2
    imgs = [net_image(cfg, s) for s in range(B)]
    taps = np.concatenate([net.encrypt_image(im, nonce=s) for s, im in enumerate(imgs)])
    dt = ctx.ct(B * net.tap_cts, net.top, taps, DELTA)
    out = ctx.ct(B, net.out_level)
    ctx.reset_meter()
    net.run(dt, out)
    got = out.download().reshape(B, -1)
    spec = HS.CnnSpec(cfg.in_c, cfg.in_d, cfg.k, cfg.s, cfg.c_out, cfg.dense, cfg.n_slots)
    golden = HS.golden_stage_tallies(spec)
    assert dict(ctx.stages()) == {k: tuple(B * x for x in v) for k, v in golden.items()}
    keys = {}
    want, scale = P.run_net(ck, cfg, w, imgs[0], nonce=0, keys=keys)
    assert np.array_equal(got[0], want)
    for b in range(B):
        logits = net.decrypt_logits(got[b])
        ref = HS.ref_forward(spec, w, imgs[b])
        assert np.abs(logits - ref).max() < 1e-3


def test_cfg0_performed_keyswitch_counters(cfg0):
    """hegpu_ks_counters: the key-switch work the engine executes for one
    cfg-0 inference with the reference first layer, next to the reference's
    metered 120 rotations + 2 relinearisations.  Per image: merge 4 ModUps /
    4 inner products / 1 ModDown (lazy sum); each square 1/1/1; HS1 one
    hoisted ModUp, 99 keyed diagonals, 1 ModDown, then its fold as one hoisted
    sum of 2^4 - 1 = 15 rotations (1/15/1); HS2 1/9/1 and fold 1/15/1;
    rescales: 5 conv maps, 2 squares, 2 HS layers."""
    cfg, ctx, ck, w, net = cfg0
    B = 2
    taps = np.concatenate([net.encrypt_image(net_image(cfg, 70 + s), nonce=70 + s) for s in range(B)])
    out = ctx.ct(B, net.out_level)
    dt = ctx.ct(B * net.tap_cts, net.top, taps, DELTA)
    ctx.reset_meter()
    net.run(dt, out)
    got = ctx.ks_counters()
    assert got == {"modups": 10 * B, "key_inner_products": 144 * B, "moddowns": 7 * B, "rescales": 9 * B}, got
    assert ctx.total()[4] == 120 * B  # the reference's metered rotations are unchanged


def test_cfg0_fused_first_layer_bit_exact(cfg0):
    """the fused, region-packed first layer (HEGPU_FIRST_LAYER_FUSED,
    DESIGN.md §4.1c): 7 tap ciphertexts per image instead of 25, limbs ==
    the oracle's fused pipeline, logits within 1e-3 of ref_forward, the same
    per-stage HOPs as the reference layout"""
    cfg, ctx, ck, w, net = cfg0
    fused = H.Net(ctx, cfg, w, first_layer="fused")
    assert (net.tap_cts, fused.tap_cts) == (25, 7)
    assert (net.first_layer, fused.first_layer) == ("reference", "fused")
    B = 2
    imgs = [net_image(cfg, 50 + s) for s in range(B)]
    taps = np.concatenate([fused.encrypt_image(im, nonce=50 + s) for s, im in enumerate(imgs)])
    out = ctx.ct(B, fused.out_level)
    ctx.reset_meter()
    fused.run(ctx.ct(B * fused.tap_cts, fused.top, taps, DELTA), out)
    spec = HS.CnnSpec(cfg.in_c, cfg.in_d, cfg.k, cfg.s, cfg.c_out, cfg.dense, cfg.n_slots)
    golden = HS.golden_stage_tallies(spec)
    assert dict(ctx.stages()) == {k: tuple(B * x for x in v) for k, v in golden.items()}
    # region fold 1/3/1 replaces the merge's 4/4/1; one conv rescale per image
    assert ctx.ks_counters() == {"modups": 7 * B, "key_inner_products": 143 * B, "moddowns": 7 * B,
                                 "rescales": 5 * B}
    got = out.download().reshape(B, -1)
    want, _ = P.run_net(ck, cfg, w, imgs[0], nonce=50, merged=True)
    assert np.array_equal(got[0], want)
    for b in range(B):
        assert np.abs(fused.decrypt_logits(got[b]) - HS.ref_forward(spec, w, imgs[b])).max() < 1e-3


def test_cfg0_net_batch_tensor_core_hs(cfg0):
    """a batch of 9 images: both HS layers run on the tensor-core kernel;
    image 0's limbs == the oracle pipeline, all logits within 1e-3"""
    cfg, ctx, ck, w, net = cfg0
    B = 9
    imgs = [net_image(cfg, 40 + s) for s in range(B)]
    taps = np.concatenate([net.encrypt_image(im, nonce=40 + s) for s, im in enumerate(imgs)])
    out = ctx.ct(B, net.out_level)
    net.run(ctx.ct(B * net.tap_cts, net.top, taps, DELTA), out)
    got = out.download().reshape(B, -1)
    want, _ = P.run_net(ck, cfg, w, imgs[0], nonce=40)
    assert np.array_equal(got[0], want)
    spec = HS.CnnSpec(cfg.in_c, cfg.in_d, cfg.k, cfg.s, cfg.c_out, cfg.dense, cfg.n_slots)
    for b in range(B):
        assert np.abs(net.decrypt_logits(got[b]) - HS.ref_forward(spec, w, imgs[b])).max() < 1e-3


def test_cfg0_net_batch64_two_streams(cfg0):
    """a 64-image batch (config 2's step) runs as two 32-image parts on two
    streams (net.cu run_net), also inside a CUDA-graph capture: every image's
    limbs equal its single-image run"""
    cfg, ctx, ck, w, net = cfg0
    t = [net.encrypt_image(net_image(cfg, 70 + s), nonce=70 + s) for s in range(3)]
    singles = []
    for k in range(3):
        o = ctx.ct(1, net.out_level)
        net.run(ctx.ct(net.tap_cts, net.top, t[k], DELTA), o)
        singles.append(o.download())
    order = [(b * 7 + b // 32) % 3 for b in range(64)]   # a different pattern in each half
    din = ctx.ct(64 * net.tap_cts, net.top, np.concatenate([t[k] for k in order]), DELTA)
    out = ctx.ct(64, net.out_level)
    net.run(din, out)
    got = out.download().reshape(64, -1)
    for b in range(64):
        assert np.array_equal(got[b], singles[order[b]]), b
    out2 = ctx.ct(64, net.out_level)
    graph = ctx.capture(lambda: net.run(din, out2))
    graph()
    graph()
    ctx.sync()
    assert np.array_equal(out2.download().reshape(64, -1), got)


def test_cfg0_run_host_matches_device_run(cfg0):
    cfg, ctx, ck, w, net = cfg0
    B = 3
    taps = np.concatenate([net.encrypt_image(net_image(cfg, 10 + s), nonce=10 + s) for s in range(B)])
    host_out = np.zeros(B * net.out_words, dtype=np.uint64)
    net.run_host(taps, B, host_out)
    out = ctx.ct(B, net.out_level)
    net.run(ctx.ct(B * net.tap_cts, net.top, taps, DELTA), out)
    assert np.array_equal(host_out, out.download())


@pytest.mark.parametrize("chunk", [0, 2, 5])
def test_cfg0_run_host_compact_pipeline(cfg0, chunk):
    """e2e path: compact taps, chunked H2D/compute pipeline == device run"""
    cfg, ctx, ck, w, net = cfg0
    B = 5
    imgs = [net_image(cfg, 30 + s) for s in range(B)]
    compact = np.concatenate([net.encrypt_image_compact(im, nonce=30 + s) for s, im in enumerate(imgs)])
    full = np.concatenate([net.encrypt_image(im, nonce=30 + s) for s, im in enumerate(imgs)])
    host_out = np.zeros(B * net.out_words, dtype=np.uint64)
    net.run_host_compact(compact, B, host_out, chunk)
    out = ctx.ct(B, net.out_level)
    net.run(ctx.ct(B * net.tap_cts, net.top, full, DELTA), out)
    assert np.array_equal(host_out, out.download())


def test_cfg0_run_compact_device_and_submit(cfg0):
    """device-resident compact taps (conv MAC decodes c0 / regenerates c1 on
    the fly) and the pipelined submit/wait serving path == full-ct device run,
    with the same per-stage HOP metering"""
    import torch
    cfg, ctx, ck, w, net = cfg0
    B = 3
    imgs = [net_image(cfg, 60 + s) for s in range(B)]
    compact = np.concatenate([net.encrypt_image_compact(im, nonce=60 + s) for s, im in enumerate(imgs)])
    full = np.concatenate([net.encrypt_image(im, nonce=60 + s) for s, im in enumerate(imgs)])
    ref = ctx.ct(B, net.out_level)
    ctx.reset_meter()
    net.run(ctx.ct(B * net.tap_cts, net.top, full, DELTA), ref)
    want_stages = dict(ctx.stages())
    want = ref.download()
    out = ctx.ct(B, net.out_level)
    ctx.reset_meter()
    net.run_compact(torch.from_numpy(compact).cuda(), B, out)
    assert np.array_equal(out.download(), want)
    assert dict(ctx.stages()) == want_stages
    outs = [np.zeros(B * net.out_words, dtype=np.uint64) for _ in range(2)]
    ctx.reset_meter()
    # passes alternate over the two staging buffers: the first use of each
    # buffer set runs direct, the second is captured into a CUDA graph, later
    # ones replay it (metering re-applied)
    for k in range(6):
        net.submit_host_compact(compact, B, outs[k % 2], 2)
    net.wait()
    for o in outs:
        assert np.array_equal(o, want)
    assert dict(ctx.stages()) == {k: tuple(6 * x for x in v) for k, v in want_stages.items()}


def test_cfg0_net_run_split_dense1(cfg0):
    """the multi-GPU config-3 scheme on one GPU: each "rank" runs the net with
    HS1 restricted to its diagonal range, the partial accumulators are summed
    (here: rank 0's partial is stashed and added by rank 1's reduction), and
    the finished output equals the single-GPU run bit for bit, with the HOP
    tallies of the two parts adding up to one run's"""
    import torch
    cfg, ctx, ck, w, net = cfg0
    B = 2
    imgs = [net_image(cfg, 80 + s) for s in range(B)]
    taps = ctx.ct(B * net.tap_cts, net.top,
                  np.concatenate([net.encrypt_image(im, nonce=80 + s) for s, im in enumerate(imgs)]), DELTA)
    ref = ctx.ct(B, net.out_level)
    ctx.reset_meter()
    net.run(taps, ref)
    one_run = dict(ctx.stages())
    want = ref.download()
    # nparts = 1: plumbing only
    out = ctx.ct(B, net.out_level)
    net.run_split(taps, out, 0, 0, 1, lambda t: None)
    assert np.array_equal(out.download(), want)
    # nparts = 2: rank 0's partial sum is kept for rank 1's reduction
    stash = {}
    ctx.reset_meter()
    net.run_split(taps, ctx.ct(B, net.out_level), 0, 0, 2, lambda t: stash.setdefault("p0", t.clone()))
    net.run_split(taps, out, 0, 1, 2, lambda t: t.add_(stash["p0"]))
    assert np.array_equal(out.download(), want)
    # HS1's MulPC is split over the two parts; every other stage ran twice
    two = dict(ctx.stages())
    assert two["Dense1"][2] == one_run["Dense1"][2]
    for st in one_run:
        if st != "Dense1":
            assert two[st] == tuple(2 * x for x in one_run[st])


@pytest.mark.parametrize("nparts", [2, 3, 5])
def test_cfg0_net_run_split_first_layer(cfg0, nparts):
    """config 3's first-layer split: each "rank" runs the
    conv + merge rotations of its share of the c_out = 5 output maps, the
    (extended-basis, Q-basis) partials are summed by the reduction (here:
    earlier parts stashed and added by the last), every rank finishes the
    merge's ModDown and the rest of the net -- bit-identical to the
    single-GPU run; Conv1 / Flat1 HOPs of the parts add up to one run's"""
    cfg, ctx, ck, w, net = cfg0
    B = 2
    imgs = [net_image(cfg, 90 + s) for s in range(B)]
    taps = ctx.ct(B * net.tap_cts, net.top,
                  np.concatenate([net.encrypt_image(im, nonce=90 + s) for s, im in enumerate(imgs)]), DELTA)
    ref = ctx.ct(B, net.out_level)
    ctx.reset_meter()
    net.run(taps, ref)
    one_run = dict(ctx.stages())
    want = ref.download()
    stash = []
    ctx.reset_meter()
    out = ctx.ct(B, net.out_level)
    for part in range(nparts):
        def red(t, last=part == nparts - 1):
            if last:
                for p in stash:
                    t.add_(p)
            else:
                stash.append(t.clone())
        net.run_split(taps, out if part == nparts - 1 else ctx.ct(B, net.out_level), H.SPLIT_FIRST_LAYER, part,
                      nparts, red)
    assert np.array_equal(out.download(), want)
    parts = dict(ctx.stages())
    for st in ("Conv1", "Flat1"):
        assert parts[st] == one_run[st], st
    for st in one_run:
        if st not in ("Conv1", "Flat1"):
            assert parts[st] == tuple(nparts * x for x in one_run[st])
    with pytest.raises(H.HegpuError):
        net.run_split(taps, out, 7, 0, 2, lambda t: None)
    # both splits in one run (first layer, then HS1): two reductions per run.
    # Every rank needs the full first-layer sum before its HS1 range, so the
    # one-GPU emulation first collects each part's first-layer partial (the
    # run is aborted by a failing reduction), then runs every part with the
    # first reduction completed from the others' partials
    first = {}
    for part in range(nparts):
        def grab(t, part=part):
            first[part] = t.clone()
            raise RuntimeError("stop after the first-layer partial")
        with pytest.raises(H.HegpuError):
            net.run_split(taps, ctx.ct(B, net.out_level), H.split_first_and_dense(0), part, nparts, grab)
    hs1 = []
    out2 = ctx.ct(B, net.out_level)
    for part in range(nparts):
        calls = [0]

        def red2(t, part=part, last=part == nparts - 1):
            k = calls[0]
            calls[0] += 1
            if k == 0:
                for q, p in first.items():
                    if q != part:
                        t.add_(p)
            elif last:
                for p in hs1:
                    t.add_(p)
            else:
                hs1.append(t.clone())
        net.run_split(taps, out2 if part == nparts - 1 else ctx.ct(B, net.out_level), H.split_first_and_dense(0),
                      part, nparts, red2)
        assert calls[0] == 2
    assert np.array_equal(out2.download(), want)


def test_cfg0_net_from_model_files(cfg0, tmp_path):
    """hegpu_net_create_from_model: the cfg-0 net described as a model JSON +
    float32 weights file + float32 input file (the reference's formats)
    computes bit-identical ciphertexts to the net built from arrays"""
    from test_modelio import CFG0_JSON, flat_weights
    cfg, ctx, ck, w, net = cfg0
    model = H.Model.parse(CFG0_JSON)
    model.save_weights(tmp_path / "w.bin", flat_weights(w))
    img = net_image(cfg, 90)
    model.save_input(tmp_path / "x.bin", img)
    x = model.load_input(tmp_path / "x.bin")
    assert np.array_equal(x, img)  # inputs are float32 values already
    net2 = H.Net.from_model(ctx, model, tmp_path / "w.bin")
    t1 = net.encrypt_image(img, nonce=90)
    t2 = net2.encrypt_image(x, nonce=90)
    assert np.array_equal(t1, t2)
    o1, o2 = ctx.ct(1, net.out_level), ctx.ct(1, net2.out_level)
    net.run(ctx.ct(net.tap_cts, net.top, t1, DELTA), o1)
    net2.run(ctx.ct(net2.tap_cts, net2.top, t2, DELTA), o2)
    assert np.array_equal(o1.download(), o2.download())
    spec = HS.CnnSpec(cfg.in_c, cfg.in_d, cfg.k, cfg.s, cfg.c_out, cfg.dense, cfg.n_slots)
    assert np.abs(net2.decrypt_logits(o2.download()) - HS.ref_forward(spec, w, img)).max() < 1e-3


def test_cryptonets_model_lowered_on_gpu(tmp_path):
    """the reference's builtin cryptonets-hs layer list (conv, square,
    avgpool, conv, avgpool, flatten, dense, square, dense) from a model file:
    lower() fuses the linear run into one HS layer; decrypted logits match
    the FP64 forward pass of the layer list; stage labels follow lower()"""
    from test_modelio import cryptonets_weights
    m, w = cryptonets_weights(7)
    m.save_weights(tmp_path / "w.bin", w)
    ctx = H.Context(13, [60, 40, 40, 40, 40, 40], 60, seed=77)
    net = H.Net.from_model(ctx, m, tmp_path / "w.bin")
    per_layer = HS.split_weights(m.layers, m.in_c, m.in_d, w)
    rng = np.random.default_rng(3)
    for s in range(2):
        img = np.zeros((1, 29, 29))
        img[0, :28, :28] = rng.uniform(0, 1, (28, 28)).astype(np.float32)
        out = ctx.ct(1, net.out_level)
        ctx.reset_meter()
        net.run(ctx.ct(net.tap_cts, net.top, net.encrypt_image(img, nonce=s), DELTA), out)
        logits = net.decrypt_logits(out.download())
        want = HS.ref_forward_layers(m.layers, per_layer, img)
        assert np.abs(logits - want).max() < 1e-3
    assert [k for k, _ in ctx.stages()] == ["Conv1", "Flat1", "Square1", "Conv2-Dense1", "Square2", "Dense2"]


def test_cfg3_net_logits_and_hops():
    """Config 3 (CIFAR-shaped, N=16384): conv 5x5/2 3->32 (75 taps), merge 32
    maps (6272 slots), HS 6272->256, HS 256->10; logits vs ref_forward and
    the golden per-inference HOPs (34/2673/2666/2/305)."""
    from paper_2110_08321_b200.workloads import CFG3
    cfg = CFG3
    ctx = H.Context(cfg.log_n, list(cfg.qbits), cfg.pbits, seed=303)
    w = net_weights(cfg, 3)
    net = H.Net(ctx, cfg, w)
    B = 2
    imgs = [net_image(cfg, 100 + s) for s in range(B)]
    taps = np.concatenate([net.encrypt_image(im, nonce=s) for s, im in enumerate(imgs)])
    out = ctx.ct(B, net.out_level)
    ctx.reset_meter()
    net.run(ctx.ct(B * net.tap_cts, net.top, taps, DELTA), out)
    got = out.download().reshape(B, -1)
    spec = HS.CnnSpec(cfg.in_c, cfg.in_d, cfg.k, cfg.s, cfg.c_out, cfg.dense, cfg.n_slots)
    golden = HS.golden_stage_tallies(spec)
    assert dict(ctx.stages()) == {k: tuple(B * x for x in v) for k, v in golden.items()}
    assert tuple(np.sum(list(golden.values()), axis=0)) == (34, 2673, 2666, 2, 305)
    for b in range(B):
        ref = HS.ref_forward(spec, w, imgs[b])
        assert np.abs(net.decrypt_logits(got[b]) - ref).max() < 1e-3


def test_cfg3_shaped_hs_bit_exact():
    """HS 6272 -> 256 at N=16384 (config 3's dense layer, plain branch with 5
    folds) against the oracle, on a 3-prime chain to bound key memory."""
    ctx = H.Context(14, [60, 40, 40], 60, seed=33)
    ck = Ckks(14, [60, 40, 40], 60, seed=33)
    A = np.random.default_rng(0).normal(0, 0.02, (256, 6272))
    x = np.random.default_rng(1).uniform(0, 1, 6272)
    v = ck.encrypt(ck.encode(x, DELTA, 3), 3, 9)
    plan = ctx.hs_plan(A, 3)
    assert (plan.m_eff, plan.folds, plan.kept) == (256, 5, 256)
    ctx.gen_rotation_keys(plan.rotations())
    out = ctx.ct(1, 2)
    got = ctx.hs_matvec(plan, ctx.ct(1, 3, v, DELTA), out).download()
    assert np.array_equal(got, P.hs_matvec(ck, v, 3, A))
    assert np.abs(ck.decrypt_decode(got, 2, DELTA)[:256] - A @ x).max() < 1e-4


def test_cfg1_point_hs(cfg0):
    """Config 1 shape at reduced ring (full sizes run in bench): m=64, n=256."""
    ctx = H.Context(12, [60, 40], 60, seed=3)
    ck = Ckks(12, [60, 40], 60, seed=3)
    A, x = hs_sweep_case(64, 256)
    v = ck.encrypt(ck.encode(x, DELTA, 2), 2, 1)
    plan = ctx.hs_plan(A, 2)
    ctx.gen_rotation_keys(plan.rotations())
    out = ctx.ct(1, 1)
    got = ctx.hs_matvec(plan, ctx.ct(1, 2, v, DELTA), out).download()
    assert np.array_equal(got, P.hs_matvec(ck, v, 2, A))
    assert np.abs(ck.decrypt_decode(got, 1, DELTA)[:64] - A @ x).max() < 1e-5
