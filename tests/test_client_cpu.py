"""CPU-side checks of the product library (no GPU needed):
  - libhegpu.so loads and exports every symbol include/hegpu.h declares;
  - the host client (encode / encrypt / keygen / decrypt) is bit-identical
    to the independent CPU oracle (oracle/ckks_oracle.c);
  - without a device, evaluator contexts fail loudly (no CPU fallback)."""
import ctypes

import numpy as np
import pytest

from oracle.ckks import Ckks
from paper_2110_08321_b200 import hegpu as H

PARAMS = [
    (5, [60, 40, 40], 60),                 # N = 32 (fast)
    (10, [60, 40, 40, 40], 60),            # N = 1024
    (13, [60, 40, 40, 40, 40, 40], 60),    # config 0: N = 8192, 5 rescales
]


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(H.LIB_PATH)
    decl = H.declared_symbols()
    assert len(decl) >= 45
    missing = [s for s in decl if not hasattr(lib, s)]
    assert not missing, missing


def test_device_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(H.HegpuError) as e:
        H.Context(5, [60, 40], 60, device=0)
    assert e.value.code == H.ERR_CUDA
    ctx = H.Context(5, [60, 40], 60, device=H.CLIENT_ONLY)
    with pytest.raises(H.HegpuError) as e:
        ctx.ct(1, 1)
    assert e.value.code == H.ERR_CUDA


@pytest.mark.parametrize("log_n,qbits,pbits", PARAMS)
def test_primes_match_oracle(log_n, qbits, pbits):
    ctx = H.Context(log_n, qbits, pbits, seed=3, device=H.CLIENT_ONLY)
    ck = Ckks(log_n, qbits, pbits, seed=3)
    assert ctx.primes == ck.primes
    for q in ctx.primes:
        assert q % (2 * ctx.N) == 1 and q < 2 ** 61


@pytest.mark.parametrize("log_n,qbits,pbits", PARAMS)
def test_encode_encrypt_bit_exact(log_n, qbits, pbits):
    ctx = H.Context(log_n, qbits, pbits, seed=11, device=H.CLIENT_ONLY)
    ck = Ckks(log_n, qbits, pbits, seed=11)
    rng = np.random.default_rng(log_n)
    L = len(qbits)
    for scale, level, with_p in ((2.0 ** 40, L, False), (2.0 ** 80, L - 1, True), (float(ctx.primes[1]), 2, True)):
        z = rng.uniform(-1, 1, ctx.S // 2 + 1)
        a = ctx.encode(z, scale, level, with_p)
        b = ck.encode(z, scale, level, with_p)
        assert np.array_equal(a, b)
    pt = ck.encode(rng.uniform(-1, 1, ctx.S), 2.0 ** 40, L)
    c1 = ctx.encrypt(pt, L, nonce=77)
    c2 = ck.encrypt(pt, L, nonce=77)
    assert np.array_equal(c1, c2)
    assert np.array_equal(ctx.decrypt(c1, L), ck.decrypt(c2, L))
    d1 = ctx.decode(ctx.decrypt(c1, L), L, 2.0 ** 40)
    d2 = ck.decrypt_decode(c2, L, 2.0 ** 40)
    assert np.abs(d1 - d2).max() < 1e-9


def slot_src(log_n):
    """device slot order: position p < S holds psi^(5^p), p >= S psi^(-5^(p-S));
    wire index brv((e - 1) / 2)"""
    n, s, m2n = 1 << log_n, 1 << (log_n - 1), 2 << log_n
    out = np.empty(n, dtype=np.int64)
    g = 1
    for p in range(s):
        for e, q in ((g, p), (m2n - g, p + s)):
            k = (e - 1) // 2
            out[q] = int(format(k, f"0{log_n}b")[::-1], 2)
        g = g * 5 % m2n
    return out


def unpack_compact(ctx, blob, level):
    """host-side reference unpacking of the compact format (c0 only, back to
    wire order)"""
    off = 8 * level
    perm = slot_src(int(ctx.N).bit_length() - 1)
    c0 = []
    for t in range(level):
        nb = (int(ctx.primes[t]).bit_length() + 7) // 8
        raw = blob[off:off + nb * ctx.N].reshape(ctx.N, nb).astype(np.uint64)
        slot = sum(raw[:, b] << np.uint64(8 * b) for b in range(nb))
        wire = np.empty_like(slot)
        wire[perm] = slot
        c0.append(wire)
        off += nb * ctx.N
    assert off == len(blob)
    return np.concatenate(c0)


@pytest.mark.parametrize("log_n,qbits,pbits", PARAMS)
def test_compact_encryption_matches_full(log_n, qbits, pbits):
    ctx = H.Context(log_n, qbits, pbits, seed=17, device=H.CLIENT_ONLY)
    L = len(qbits)
    pt = ctx.encode(np.random.default_rng(1).uniform(-1, 1, ctx.S), 2.0 ** 40, L)
    full = ctx.encrypt(pt, L, nonce=5)
    blob = ctx.encrypt_compact(pt, L, nonce=5)
    assert len(blob) == ctx.compact_bytes(L)
    assert np.array_equal(unpack_compact(ctx, blob, L), full[: L * ctx.N])
    # config 0: 33 bytes per coefficient instead of 96
    if qbits == [60, 40, 40, 40, 40, 40]:
        assert len(blob) == 8 * L + ctx.N * (8 + 5 * 5)


def test_edge_encodings():
    ctx = H.Context(6, [60, 40], 60, seed=1, device=H.CLIENT_ONLY)
    ck = Ckks(6, [60, 40], 60, seed=1)
    for z in (np.zeros(0), np.zeros(ctx.S), np.full(ctx.S, -3.25), np.array([1e6, -1e6])):
        assert np.array_equal(ctx.encode(z, 2.0 ** 40, 2), ck.encode(z, 2.0 ** 40, 2))
    with pytest.raises(H.CapacityError):
        ctx.encode(np.zeros(ctx.S + 1), 2.0 ** 40, 2)


@pytest.mark.parametrize("log_n,qbits,pbits", PARAMS[:2])
def test_keys_bit_exact(log_n, qbits, pbits):
    ctx = H.Context(log_n, qbits, pbits, seed=5, device=H.CLIENT_ONLY)
    ck = Ckks(log_n, qbits, pbits, seed=5)
    assert np.array_equal(ctx.export_relin_key(), ck.relin_key())
    for r in (1, 3, ctx.S - 1):
        assert np.array_equal(ctx.export_rotation_key(r), ck.galois_key(ck.galois_right(r)))
    with pytest.raises(H.RangeError):
        ctx.export_rotation_key(ctx.S)


def test_cfg0_galois_key_bit_exact():
    ctx = H.Context(13, [60, 40, 40, 40, 40, 40], 60, seed=9, device=H.CLIENT_ONLY)
    ck = Ckks(13, [60, 40, 40, 40, 40, 40], 60, seed=9)
    assert np.array_equal(ctx.export_rotation_key(169), ck.galois_key(ck.galois_right(169)))


def test_oracle_lola_pipelines_decrypt_to_reference_slots():
    """the CPU-oracle LoLa compositions (checkers of the GPU LoLa path)
    decrypt to the reference's slot vectors (proj/src/matvec.cpp:107-166)"""
    import numpy as np
    from oracle import ckks_pipeline as P
    from oracle import hesim_oracle as HS
    from oracle.ckks import Ckks
    ck = Ckks(9, [60, 40, 40, 40], 60, seed=5)
    rng = np.random.default_rng(3)
    for m, n in ((3, 5), (6, 20)):
        A = rng.normal(0, 0.3, (m, n))
        x = rng.uniform(-1, 1, n)
        v = ck.encrypt(ck.encode(x, 2.0 ** 40, 4), 4, 1)
        outs = P.lola_dense(ck, v, 4, A).reshape(m, -1)
        for i in range(m):
            dec = ck.decrypt_decode(outs[i], 2, 2.0 ** 40)
            assert abs(dec[0] - A[i] @ x) < 1e-5 and np.abs(dec[1:]).max() < 1e-5
        res, sor = P.lola_stacked(ck, v, 4, A)
        ctx = HS.MeterContext()
        want, sor_ref = HS.lola_stacked_matvec(A, HS.pack(x, ck.S, HS.CIPHERTEXT), ctx)
        assert sor == sor_ref
        assert np.abs(ck.decrypt_decode(res, 2, 2.0 ** 40) - want.slots).max() < 1e-5


def test_workload_conv_helpers_match_the_oracle():
    """the client-side packing helpers used by bench_configs (config 4)
    equal the oracle's conv_pack / conv_to_matrix restatements"""
    import numpy as np
    from oracle import hesim_oracle as HS
    from paper_2110_08321_b200.workloads import conv_as_matrix, conv_pack_image
    rng = np.random.default_rng(2)
    img = rng.uniform(0, 1, (3, 9, 9))
    W = rng.normal(0, 1, (4, 3, 3, 3))
    for s in (1, 2):
        shape = HS.ConvShape(9, 3, 3, s, 4)
        taps = HS.conv_pack(img, shape, 64)
        mine = conv_pack_image(img, 3, s)
        w = shape.d_out() ** 2
        assert all(np.array_equal(t.slots[:w], m) for t, m in zip(taps, mine))
        assert np.array_equal(HS.conv_to_matrix(shape, W), conv_as_matrix(W, 9, s))
