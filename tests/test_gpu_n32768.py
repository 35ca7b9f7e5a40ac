"""N = 2^15 (n_slots = 16384, the ring the reference's `ce` builtin declares,
proj/src/netcompile.cpp:612): the NTT rows run as two-CTA clusters (ntt.cu:
first Cooley-Tukey stage on load, last Gentleman-Sande stage through
distributed shared memory).  Every NTT entry point -- row INTT, key-switch
INTT + ModUp, drop-limb NTT (rescale / ModDown), the fused ModDown + rescale
-- is exercised through the C-ABI operators and compared limb for limb with
the CPU oracle."""
import numpy as np
import pytest

from oracle import hesim_oracle as HS
from oracle.ckks import Ckks
from oracle import ckks_pipeline as P
from paper_2110_08321_b200 import hegpu as H

pytestmark = pytest.mark.gpu

BIG = (15, [45, 40, 40, 40], 45)   # N = 32768, S = 16384; every prime on the FP64 butterflies
DELTA = 2.0 ** 40


@pytest.fixture(scope="module")
def pair():
    log_n, qb, pb = BIG
    ctx = H.Context(log_n, qb, pb, seed=33)
    ck = Ckks(log_n, qb, pb, seed=33)
    assert ctx.primes == ck.primes and ctx.N == 32768
    return ctx, ck


def fresh(ck, rng, level, nonce, n=None):
    z = rng.uniform(-1, 1, n or ck.S)
    return z, ck.encrypt(ck.encode(z, DELTA, level), level, nonce)


def test_roundtrip_and_mul_rescale(pair):
    ctx, ck = pair
    rng = np.random.default_rng(0)
    l = 4
    za, a = fresh(ck, rng, l, 1)
    da = ctx.ct(1, l, a, DELTA)
    assert np.array_equal(da.download(), a)
    zp = rng.uniform(-1, 1, ck.S)
    p = ck.encode(zp, float(ck.primes[l - 1]), l)
    out, r = ctx.ct(1, l), ctx.ct(1, l - 1)
    ctx.mul_plain(da, ctx.pt(1, l, False, p, float(ck.primes[l - 1])), out)
    ctx.rescale(out, r)                       # k_intt_rows + k_drop_ntt
    want = ck.rescale(ck.mul_pc(a, p, l), l)
    assert np.array_equal(r.download(), want)
    assert np.abs(ck.decrypt_decode(want, l - 1, DELTA) - za * zp).max() < 1e-5


@pytest.mark.parametrize("r", [1, 4097, 16383])
def test_rotate(pair, r):
    ctx, ck = pair
    rng = np.random.default_rng(r)
    l = 3
    z, a = fresh(ck, rng, l, 10 + r)
    ctx.gen_rotation_keys([r])
    out = ctx.ct(1, l)
    got = ctx.rotate_right(ctx.ct(1, l, a, DELTA), r, out).download()   # k_ks_intt + k_ks_modup + ModDown
    want = ck.rotate(a, l, ck.galois_right(r), ck.galois_key(ck.galois_right(r)))
    assert np.array_equal(got, want)
    assert np.abs(ck.decrypt_decode(got, l, DELTA) - np.roll(z, r)).max() < 1e-5


def test_square_fused_moddown_rescale(pair):
    ctx, ck = pair
    rng = np.random.default_rng(6)
    l = 4
    z, a = fresh(ck, rng, l, 50)
    ctx.gen_relin_key()
    out = ctx.ct(2, l - 1)
    _, b = fresh(ck, rng, l, 51)
    got = ctx.square(ctx.ct(2, l, np.concatenate([a, b]), DELTA), out).download().reshape(2, -1)  # k_md_intt + k_md_ntt
    rlk = ck.relin_key()
    assert np.array_equal(got[0], ck.rescale(ck.square(a, l, rlk), l))
    assert np.array_equal(got[1], ck.rescale(ck.square(b, l, rlk), l))
    s = DELTA * DELTA / ck.primes[l - 1]
    assert np.abs(ck.decrypt_decode(got[0], l - 1, s) - z * z).max() < 1e-5


def test_merge_and_hs(pair):
    ctx, ck = pair
    rng = np.random.default_rng(9)
    l, c, w = 3, 3, 5000
    zs, cts = [], []
    for j in range(c):
        z, ct = fresh(ck, rng, l, 80 + j, n=w)
        zs.append(z)
        cts.append(ct)
    maps = np.concatenate(cts)
    ctx.gen_rotation_keys([j * w for j in range(1, c)])
    out = ctx.ct(1, l)
    got = ctx.merge_maps(ctx.ct(c, l, maps, DELTA), c, w, out).download()
    assert np.array_equal(got, P.merge(ck, maps, c, l, w))
    assert np.abs(ck.decrypt_decode(got, l, DELTA)[: c * w] - np.concatenate(zs)).max() < 1e-5
    for m, n in ((10, 100), (24, 9000)):   # the second: folds across most of the 16384 slots
        A = rng.normal(0, 0.05, (m, n))
        z, v = fresh(ck, rng, l, 100 + m, n=n)
        plan = ctx.hs_plan(A, l, True)
        ctx.gen_rotation_keys(plan.rotations())
        o = ctx.ct(1, l - 1)
        ctx.reset_meter()
        got = ctx.hs_matvec(plan, ctx.ct(1, l, v, DELTA), o).download()
        assert np.array_equal(got, P.hs_matvec(ck, v, l, A, True))
        assert np.abs(ck.decrypt_decode(got, l - 1, DELTA)[:m] - A @ z).max() < 1e-4
        assert ctx.total()[4] == HS.predict_hs(m, n, ck.S)[0]


def test_batched_hs_and_rotate(pair):
    """batches of >= 8 ciphertexts take the tcgen05 HS kernel; a batched
    rotation shares one key"""
    ctx, ck = pair
    rng = np.random.default_rng(21)
    l, B, m, n = 3, 8, 16, 300
    A = rng.normal(0, 0.05, (m, n))
    cts = [fresh(ck, rng, l, 300 + i, n=n) for i in range(B)]
    plan = ctx.hs_plan(A, l, True)
    ctx.gen_rotation_keys(plan.rotations() + [5])
    batch = np.concatenate([c for _, c in cts])
    d = ctx.ct(B, l, batch, DELTA)
    got = ctx.hs_matvec(plan, d, ctx.ct(B, l - 1)).download().reshape(B, -1)
    assert np.array_equal(got[0], P.hs_matvec(ck, cts[0][1], l, A, True))
    one = ctx.hs_matvec(plan, ctx.ct(1, l, cts[B - 1][1], DELTA), ctx.ct(1, l - 1)).download()
    assert np.array_equal(got[B - 1], one)
    for i in range(B):
        assert np.abs(ck.decrypt_decode(got[i], l - 1, DELTA)[:m] - A @ cts[i][0]).max() < 1e-4
    rot = ctx.rotate_right(d, 5, ctx.ct(B, l)).download().reshape(B, -1)
    key = ck.galois_key(ck.galois_right(5))
    for i in (0, B - 1):
        assert np.array_equal(rot[i], ck.rotate(cts[i][1], l, ck.galois_right(5), key))


def test_cluster_kernels_are_deterministic(pair):
    """the DSMEM exchange of the split inverse transform and the two-CTA
    forward halves: 12 repeated key switches / squares of a 16-ciphertext
    batch (enough rows to fill the GPU several times) give identical limbs"""
    ctx, ck = pair
    rng = np.random.default_rng(31)
    l, B = 4, 16
    cts = np.concatenate([fresh(ck, rng, l, 400 + i)[1] for i in range(B)])
    ctx.gen_rotation_keys([123])
    ctx.gen_relin_key()
    d = ctx.ct(B, l, cts, DELTA)
    rot0 = ctx.rotate_right(d, 123, ctx.ct(B, l)).download()
    sq0 = ctx.square(d, ctx.ct(B, l - 1)).download()
    assert np.array_equal(rot0.reshape(B, -1)[3], ck.rotate(cts.reshape(B, -1)[3], l, ck.galois_right(123),
                                                             ck.galois_key(ck.galois_right(123))))
    for _ in range(12):
        assert np.array_equal(ctx.rotate_right(d, 123, ctx.ct(B, l)).download(), rot0)
        assert np.array_equal(ctx.square(d, ctx.ct(B, l - 1)).download(), sq0)


def test_conv_pack_layer(pair):
    ctx, ck = pair
    rng = np.random.default_rng(12)
    cfg = type("C", (), dict(in_c=3, in_d=32, k=3, s=1, c_out=4))   # ce's first layer shape, 4 of its 18 maps
    img = rng.uniform(0, 1, (3, 32, 32))
    W = rng.normal(0, 0.05, (4, 3, 3, 3))
    bias = rng.normal(0, 0.01, 4)
    L = ck.L
    taps = P.conv_pack_taps(ck, cfg, img, 3, DELTA, merged=False)
    out = ctx.ct(4, L - 1)
    got = ctx.conv_packed_forward(ctx.ct(27, L, taps, DELTA), 27, W.reshape(4, 27), bias, 900, out).download()
    assert np.array_equal(got, P.conv_layer(ck, taps, 27, L, W.reshape(4, 27), bias, 900, DELTA))
    ref = HS.ref_conv(img, W, bias, 1)
    per = 2 * (L - 1) * ck.N
    assert np.abs(ck.decrypt_decode(got[:per], L - 1, DELTA)[:900] - ref[0].ravel()).max() < 1e-5


def test_sixty_bit_chain_is_rejected():
    with pytest.raises(H.HegpuError):
        H.Context(15, [60, 40, 40], 60, seed=1)
