"""Pins the slot-level oracle (oracle/hesim_oracle.py) against the
reference's own known-answer tests.  Each test cites the reference test it
restates (proj/tests/*.cpp)."""
import numpy as np
import pytest

from oracle import hesim_oracle as H


def ct(vals, n):
    v = np.zeros(n)
    v[: len(vals)] = vals
    return H.SlotVector(v, H.CIPHERTEXT)


def test_power_of_two():  # test_slotvec.cpp:28-32
    H.SlotVector(np.zeros(8), H.CIPHERTEXT)
    with pytest.raises(H.ShapeError):
        H.SlotVector(np.zeros(6), H.CIPHERTEXT)
    with pytest.raises(H.ShapeError):
        H.SlotVector(np.zeros(0), H.PLAINTEXT)


def test_rotate_right_basics():  # test_slotvec.cpp:34-51
    ctx = H.MeterContext()
    v = ct([1, 2, 3, 4], 4)
    assert (H.rotate_right(v, 0, ctx).slots == v.slots).all()
    assert ctx.tally.rot == 0
    assert list(H.rotate_right(v, 1, ctx).slots) == [4, 1, 2, 3]
    assert ctx.tally.rot == 1
    with pytest.raises(IndexError):
        H.rotate_right(v, 4, ctx)
    with pytest.raises(IndexError):
        H.rotate_right(v, -1, ctx)


def test_rotate_left_basics():  # test_slotvec.cpp:53-64
    ctx = H.MeterContext()
    v = ct([1, 2, 3, 4], 4)
    l1 = H.rotate_left(v, 1, ctx)
    assert l1[0] == 2 and l1[3] == 1 and ctx.tally.rot == 1
    assert (H.rotate_left(v, 0, ctx).slots == v.slots).all()
    assert ctx.tally.rot == 1


def test_rotations_compose():  # test_slotvec.cpp:66-82
    rng = np.random.default_rng(7)
    for n in (4, 8, 16, 8192):
        for _ in range(5):
            v = H.SlotVector(rng.uniform(-1, 1, n), H.CIPHERTEXT)
            a, b = int(rng.integers(n)), int(rng.integers(n))
            ctx = H.MeterContext()
            lhs = H.rotate_right(H.rotate_right(v, a, ctx), b, ctx)
            rhs = H.rotate_right(v, (a + b) % n, ctx)
            assert (lhs.slots == rhs.slots).all()
            inv = H.rotate_left(H.rotate_right(v, a, ctx), a, ctx)
            assert (inv.slots == v.slots).all()


def test_plaintext_rotations_free():  # test_slotvec.cpp:84-90
    ctx = H.MeterContext()
    pt = H.pack(np.ones(4), 4, H.PLAINTEXT)
    H.rotate_right(pt, 2, ctx)
    H.rotate_left(pt, 3, ctx)
    assert ctx.tally.rot == 0


def test_add_mul_metering():  # test_slotvec.cpp:92-134
    ctx = H.MeterContext()
    a, b = ct([1, 2], 2), ct([3, 4], 2)
    s = H.add(a, b, ctx)
    assert list(s.slots) == [4, 6] and ctx.tally.add_cc == 1
    z = H.zeros(2, H.PLAINTEXT)
    s2 = H.add(a, z, ctx)
    assert s2.kind == H.CIPHERTEXT and ctx.tally.add_pc == 1
    H.add(z, z, ctx)
    assert ctx.tally.add_pc == 1 and ctx.tally.add_cc == 1
    ctx = H.MeterContext()
    a = ct([2, 3], 2)
    one = H.pack(np.ones(2), 2, H.PLAINTEXT)
    assert (H.mul(a, one, ctx).slots == a.slots).all() and ctx.tally.mul_pc == 1
    sq = H.mul(a, a, ctx)
    assert list(sq.slots) == [4, 9] and ctx.tally.mul_cc == 1


def test_pack_and_masked_prefix():  # test_slotvec.cpp:149-176
    p = H.pack([1, 2, 3], 4, H.CIPHERTEXT)
    assert list(p.slots) == [1, 2, 3, 0]
    assert H.pack([], 4, H.CIPHERTEXT).is_zero()
    with pytest.raises(H.CapacityError):
        H.pack([4, 3, 2, 1], 2, H.CIPHERTEXT)
    m = ct([1, 2, 3, 4], 4).masked_prefix(2)
    assert list(m.slots) == [1, 2, 0, 0]


def test_extract_diagonals_2x2():  # test_matvec.cpp:35-45
    m_eff, masks = H.extract_diagonals(np.array([[1, 2], [3, 4]]), 4)
    assert m_eff == 2
    assert list(masks[0][:2]) == [1, 4] and list(masks[1][:2]) == [3, 2]


def test_extract_diagonals_pad():  # test_matvec.cpp:47-56
    A = np.random.default_rng(1).uniform(-1, 1, (3, 4))
    m_eff, masks = H.extract_diagonals(A, 4)
    assert m_eff == 4 and masks.shape[0] == 4
    assert masks[0][3] == 0 and masks[3][0] == 0


def test_extract_diagonals_identity():  # test_matvec.cpp:58-64
    _, masks = H.extract_diagonals(np.eye(4), 8)
    assert (masks[0][:4] == 1).all()
    assert all(not masks[i].any() for i in range(1, 4))


def test_rotate_and_sum():  # test_matvec.cpp:66-86
    ctx = H.MeterContext()
    s = H.rotate_and_sum(H.pack(np.arange(1, 9), 8, H.CIPHERTEXT), 8, 1, ctx)
    assert s[0] == 36 and ctx.tally.rot == 3
    ctx2 = H.MeterContext()
    v = H.pack(np.arange(1, 5), 8, H.CIPHERTEXT)
    assert (H.rotate_and_sum(v, 4, 4, ctx2).slots == v.slots).all()
    assert ctx2.tally.rot == 0
    ctx3 = H.MeterContext()
    f = H.rotate_and_sum(H.pack([5, 39, 12, 0], 4, H.CIPHERTEXT), 3, 2, ctx3)
    assert f[0] == 17 and f[1] == 39 and ctx3.tally.rot == 1


def test_hs_2x2():  # test_matvec.cpp:88-97
    ctx = H.MeterContext()
    r = H.hs_matvec(np.array([[1, 2], [3, 4]]), H.pack([5, 6], 4, H.CIPHERTEXT), ctx)
    assert r[0] == pytest.approx(17) and r[1] == pytest.approx(39)


def test_hs_identity_skips_zero_diagonals():  # test_matvec.cpp:99-108
    x = np.random.default_rng(3).uniform(-1, 1, 4)
    ctx = H.MeterContext()
    r = H.hs_matvec(np.eye(4), H.pack(x, 8, H.CIPHERTEXT), ctx)
    assert np.allclose(r.slots[:4], x)
    assert ctx.tally.mul_pc == 1 and ctx.tally.rot == 1


def test_hs_fusion_point_100x845():  # test_matvec.cpp:110-123
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (100, 845))
    x = rng.uniform(-1, 1, 845)
    ctx = H.MeterContext()
    r = H.hs_matvec(A, H.pack(x, 8192, H.CIPHERTEXT), ctx)
    want = A @ x
    assert (np.abs(r.slots[:100] - want) / np.maximum(1, np.abs(want))).max() < 1e-9
    assert ctx.tally.mul_pc == 100 and 103 <= ctx.tally.rot <= 104
    # and at the CKKS slot count S = 4096 used for ring N = 8192
    ctx = H.MeterContext()
    r = H.hs_matvec(A, H.pack(x, 4096, H.CIPHERTEXT), ctx)
    assert ctx.tally.as_tuple() == (0, 103, 100, 0, 103)


def test_predict_hs():  # test_matvec.cpp:125-131
    assert H.predict_hs(64, 4096, 16384)[:2] == (70, 64)
    assert H.predict_hs(3, 4, 4)[0] == 3
    assert H.predict_hs(1, 1, 4)[:2] == (0, 1)


def test_hs_random_triples():  # test_matvec.cpp:198-220
    rng = np.random.default_rng(23)
    for _ in range(60):
        m, n = int(rng.integers(1, 25)), int(rng.integers(1, 101))
        N = H.next_power_of_two(max(m + n - 1, 2)) * (2 if rng.integers(2) else 1)
        A = rng.uniform(-1, 1, (m, n))
        x = rng.uniform(-1, 1, n)
        r = H.hs_matvec(A, H.pack(x, N, H.CIPHERTEXT), H.MeterContext())
        want = A @ x
        assert (np.abs(r.slots[:m] - want) / np.maximum(1, np.abs(want))).max() < 1e-9


def test_hs_padding_branch_formula():  # test_matvec.cpp:222-247
    rng = np.random.default_rng(29)
    done = 0
    while done < 40:
        N = 16 << int(rng.integers(3))
        m, n = int(rng.integers(2, N)), int(rng.integers(2, N))
        if N >= m + n - 1 or H.next_power_of_two(m) > N:
            continue
        done += 1
        A = rng.uniform(-1, 1, (m, n))
        x = rng.uniform(-1, 1, n)
        ctx = H.MeterContext()
        r = H.hs_matvec(A, H.pack(x, N, H.CIPHERTEXT), ctx, skip_zero_diagonals=False)
        want = A @ x
        assert (np.abs(r.slots[:m] - want) / np.maximum(1, np.abs(want))).max() < 1e-9
        mp = H.next_power_of_two(m)
        lg = 0
        while (mp << lg) < N:
            lg += 1
        assert ctx.tally.rot == mp - 1 + lg


def test_hs_metering_equals_prediction():  # test_matvec.cpp:249-283 (HS part)
    rng = np.random.default_rng(31)
    for N in (4096, 16384):
        for n in (16, 64, 256, 1024, 4096):
            for m in (4, 16, 64):
                A = rng.uniform(-1, 1, (m, n)) + 2.0
                ctx = H.MeterContext()
                H.hs_matvec(A, H.pack(rng.uniform(-1, 1, n), N, H.CIPHERTEXT), ctx)
                rot, mul_, _ = H.predict_hs(m, n, N)
                assert ctx.tally.rot <= rot and ctx.tally.mul_pc <= mul_
                if N >= m + n - 1:
                    assert (ctx.tally.rot, ctx.tally.mul_pc) == (rot, mul_)


def test_hs_capacity():  # test_matvec.cpp:298-304
    rng = np.random.default_rng(37)
    with pytest.raises(H.CapacityError):
        H.hs_matvec(rng.uniform(-1, 1, (4, 9)), H.pack(rng.uniform(-1, 1, 8), 8, H.CIPHERTEXT),
                    H.MeterContext())


def test_conv_pack_windows():  # test_convlower.cpp:32-41
    img = np.arange(1, 10, dtype=float).reshape(1, 3, 3)
    taps = H.conv_pack(img, H.ConvShape(3, 1, 2, 1, 1), 4)
    assert len(taps) == 4
    assert list(taps[0].slots) == [1, 2, 4, 5]
    assert list(taps[1].slots) == [2, 3, 5, 6]
    assert list(taps[3].slots) == [5, 6, 8, 9]


def test_conv_pack_k1_and_kd():  # test_convlower.cpp:43-61
    rng = np.random.default_rng(1)
    img = rng.uniform(-1, 1, (1, 4, 4))
    taps = H.conv_pack(img, H.ConvShape(4, 1, 1, 1, 1), 16)
    assert len(taps) == 1 and (taps[0].slots == img.ravel()).all()
    img = rng.uniform(-1, 1, (1, 3, 3))
    taps = H.conv_pack(img, H.ConvShape(3, 1, 3, 1, 1), 4)
    assert len(taps) == 9
    for ky in range(3):
        for kx in range(3):
            assert taps[ky * 3 + kx][0] == img[0, ky, kx]


@pytest.mark.parametrize("d_in,c_in,k,s,c_out,mul_pc,add_cc,add_pc", [
    (29, 1, 5, 2, 5, 125, 120, 5),
    (30, 1, 3, 1, 5, 45, 40, 5),
    (32, 3, 3, 1, 18, 486, 468, 18),
])
def test_conv_packed_forward_counts(d_in, c_in, k, s, c_out, mul_pc, add_cc, add_pc):
    # test_convlower.cpp:63-96
    rng = np.random.default_rng(3)
    img = rng.uniform(-1, 1, (c_in, d_in, d_in))
    w = rng.uniform(-1, 1, (c_out, c_in, k, k))
    b = rng.uniform(-1, 1, c_out)
    shape = H.ConvShape(d_in, c_in, k, s, c_out)
    taps = H.conv_pack(img, shape, 1024)
    ctx = H.MeterContext()
    maps = H.conv_packed_forward(taps, w, b, shape, ctx)
    assert (ctx.tally.mul_pc, ctx.tally.add_cc, ctx.tally.add_pc, ctx.tally.rot) == \
        (mul_pc, add_cc, add_pc, 0)
    want = H.ref_conv(img, w, b, s)
    wd = shape.d_out() ** 2
    for co in range(c_out):
        assert np.allclose(maps[co].slots[:wd], want[co].ravel(), rtol=1e-9, atol=1e-12)


def test_conv_to_matrix_oracle():  # test_convlower.cpp:106-123
    rng = np.random.default_rng(5)
    for _ in range(20):
        d, c_in, c_out = int(rng.integers(3, 8)), int(rng.integers(1, 4)), int(rng.integers(1, 4))
        k, s = int(rng.integers(1, 4)), int(rng.integers(1, 3))
        if k > d:
            continue
        img = rng.uniform(-1, 1, (c_in, d, d))
        w = rng.uniform(-1, 1, (c_out, c_in, k, k))
        b = rng.uniform(-1, 1, c_out)
        shape = H.ConvShape(d, c_in, k, s, c_out)
        got = H.conv_to_matrix(shape, w) @ img.ravel() + H.conv_bias_vector(shape, b)
        assert np.abs(got - H.ref_conv(img, w, b, s).ravel()).max() < 1e-9


def test_square_layer():  # test_convlower.cpp:157-169
    ctx = H.MeterContext()
    s = H.square_layer(H.SlotVector(np.array([2, -3, 0, 1.0]), H.CIPHERTEXT), ctx)
    assert list(s.slots[:3]) == [4, 9, 0] and ctx.tally.mul_cc == 1


def test_merge_maps():  # test_convlower.cpp:171-211
    rng = np.random.default_rng(11)
    maps = [H.pack(rng.uniform(-1, 1, 169), 1024, H.CIPHERTEXT) for _ in range(5)]
    ctx = H.MeterContext()
    merged = H.merge_maps(maps, 169, ctx)
    assert ctx.tally.rot == 4 and ctx.tally.add_cc == 4
    for j in range(5):
        assert np.allclose(merged.slots[j * 169:(j + 1) * 169], maps[j].slots[:169])
    ctx = H.MeterContext()
    v = H.pack([1, 2], 4, H.CIPHERTEXT)
    assert (H.merge_maps([v], 2, ctx).slots == v.slots).all() and ctx.tally.total() == 0
    a = H.pack([1], 4, H.CIPHERTEXT)
    b = H.pack([2], 4, H.CIPHERTEXT)
    assert list(H.merge_maps([a, b], 1, ctx).slots[:3]) == [1, 2, 0]
    with pytest.raises(H.CapacityError):
        H.merge_maps([H.zeros(4, H.CIPHERTEXT)] * 5, 1, ctx)


def test_refmodel_hand_values():  # test_refmodel.cpp (dense + square)
    assert list(H.ref_dense(np.array([1.0, 2.0]), np.array([[1, 2], [3, 4.0]]),
                            np.array([0.5, -1.0]))) == [5.5, 10.0]
    x = np.arange(9, dtype=float).reshape(1, 3, 3)
    out = H.ref_conv(x, np.ones((1, 1, 2, 2)), np.array([1.0]), 1)
    assert out[0].tolist() == [[9.0, 13.0], [21.0, 25.0]]


def test_refmodel_conv_ones_2x2():  # test_refmodel.cpp:26-33
    out = H.ref_conv(np.array([[[1.0, 2.0], [3.0, 4.0]]]), np.ones((1, 1, 2, 2)), np.zeros(1), 1)
    assert out.shape == (1, 1, 1) and out[0, 0, 0] == pytest.approx(10.0)


def test_refmodel_delta_filter_crops_shifted_window():  # test_refmodel.cpp:35-47
    img = np.random.default_rng(3).uniform(-1, 1, (1, 5, 5))
    W = np.zeros((1, 1, 3, 3))
    W[0, 0, 1, 2] = 1.0  # tap (ky=1, kx=2)
    out = H.ref_conv(img, W, np.zeros(1), 1)
    assert out.shape == (1, 3, 3)
    for oy in range(3):
        for ox in range(3):
            assert out[0, oy, ox] == pytest.approx(img[0, oy + 1, ox + 2])


def test_refmodel_bias_per_output_channel():  # test_refmodel.cpp:49-57
    out = H.ref_conv(np.ones((1, 2, 2)), np.ones((2, 1, 2, 2)), np.array([0.5, -1.0]), 1)
    assert out[0, 0, 0] == pytest.approx(4.5) and out[1, 0, 0] == pytest.approx(3.0)


def test_refmodel_avgpool():  # test_refmodel.cpp:59-76
    out = H.ref_avgpool(np.array([[[1.0, 2.0], [3.0, 4.0]]]), 2, 2)
    assert out.shape[1] == 1 and out.ravel()[0] == pytest.approx(2.5)
    img = np.random.default_rng(5).uniform(-1, 1, (2, 6, 6))
    out = H.ref_avgpool(img, 3, 2)
    assert out.shape == (2, 2, 2)
    assert out[1, 1, 1] == pytest.approx(img[1, 2:5, 2:5].sum() / 9.0)


def test_refmodel_square():  # test_refmodel.cpp:78-86
    out = H.ref_square(np.array([[[2.0, -3.0, 0.0]]]))
    assert out.ravel().tolist() == [4.0, 9.0, 0.0]
    assert not H.ref_square(np.zeros((2, 3, 3))).any()


def test_refmodel_dense_identity():  # test_refmodel.cpp:88-95
    v = np.random.default_rng(7).uniform(-1, 1, 5)
    assert np.abs(H.ref_dense(v, np.eye(5), np.zeros(5)) - v).max() < 1e-15


def cfg0_spec():
    return H.CnnSpec(in_c=1, in_d=29, k=5, s=2, c_out=5, dense=(100, 10), n_slots=4096)


def test_cfg0_stage_labels_and_golden_hops():
    # stage list of proj/src/netcompile.cpp:106-213 for Conv/Square/Dense/Square/Dense;
    # per-stage golden HOPs of SURVEY.md §8d (totals 604 = 7+240+235+2+120)
    spec = cfg0_spec()
    assert spec.stage_labels() == ["Conv1", "Flat1", "Square1", "Dense1", "Square2", "Dense2"]
    g = H.golden_stage_tallies(spec)
    assert g == {"Conv1": (5, 120, 125, 0, 0), "Flat1": (0, 4, 0, 0, 4),
                 "Square1": (0, 0, 0, 1, 0), "Dense1": (1, 103, 100, 0, 103),
                 "Square2": (0, 0, 0, 1, 0), "Dense2": (1, 13, 10, 0, 13)}
    tot = np.sum([v for v in g.values()], axis=0)
    assert tuple(tot) == (7, 240, 235, 2, 120) and tot.sum() == 604


def test_cfg0_execute_matches_ref_forward():  # test_netcompile.cpp:173-189
    from paper_2110_08321_b200.workloads import cfg0_weights_and_image
    spec = cfg0_spec()
    w, img = cfg0_weights_and_image(seed=3)
    ctx = H.MeterContext()
    got = H.execute(spec, w, img, ctx)
    want = H.ref_forward(spec, w, img)
    assert (np.abs(got - want) / np.maximum(1, np.abs(want))).max() < 1e-7
    rows = {name: t.as_tuple() for name, t in ctx.stages}
    assert rows == H.golden_stage_tallies(spec)


def test_cfg3_golden_totals():  # 5680 HOPs, 305 Rot
    spec = H.CnnSpec(in_c=3, in_d=32, k=5, s=2, c_out=32, dense=(256, 10), n_slots=8192)
    tot = np.sum(list(H.golden_stage_tallies(spec).values()), axis=0)
    assert tuple(tot) == (34, 2673, 2666, 2, 305) and tot.sum() == 5680


# ---- LoLa comparators (proj/src/matvec.cpp:107-211) -------------------------
def test_lola_dense_examples():  # test_matvec.cpp:133-155
    ctx = H.MeterContext()
    out = H.lola_dense_matvec(np.array([[3.0]]), ct([7], 4), ctx)
    assert len(out) == 1 and out[0][0] == 21
    assert ctx.tally.rot == 0
    rng = np.random.default_rng(9)
    B = rng.uniform(-1, 1, (5, 8))
    y = rng.uniform(-1, 1, 8)
    ctx2 = H.MeterContext()
    rows = H.lola_dense_matvec(B, H.pack(y, 16, H.CIPHERTEXT), ctx2)
    want = B @ y
    for i in range(5):
        assert abs(rows[i][0] - want[i]) < 1e-9 * max(1, abs(want[i]))
        assert not np.any(rows[i].slots[1:])  # masked_prefix(1)
    assert ctx2.tally.rot == 5 * 3 and ctx2.tally.mul_pc == 5


def test_predict_lola_dense():  # test_matvec.cpp:157-161
    assert H.predict_lola_dense(64, 4096)[:2] == (768, 64)
    assert H.predict_lola_dense(1, 2)[0] == 1


def test_lola_stacked_4x3_in_8_slots():  # test_matvec.cpp:163-176
    rng = np.random.default_rng(17)
    A = rng.uniform(-1, 1, (4, 3))
    x = rng.uniform(-1, 1, 3)
    ctx = H.MeterContext()
    res, slot_of_row = H.lola_stacked_matvec(A, H.pack(x, 8, H.CIPHERTEXT), ctx)
    want = A @ x
    for i in range(4):
        assert abs(res[slot_of_row[i]] - want[i]) < 1e-9 * max(1, abs(want[i]))
    assert slot_of_row == [0, 4, 1, 5]
    assert ctx.tally.rot == 7 and ctx.tally.mul_pc == 2  # 2*(2+2-1)+1


def test_predict_lola_stacked():  # test_matvec.cpp:178-185
    assert H.predict_lola_stacked(64, 4096, 16384)[:2] == (255, 16)
    assert H.predict_lola_stacked(4, 3, 8)[0] == 7
    assert H.predict_lola_stacked(4, 16, 64)[0] == 4 + 4 - 1
    with pytest.raises(H.CapacityError):
        H.predict_lola_stacked(4, 9, 8)


def test_worked_example_formula_figures():  # test_matvec.cpp:187-196 (formula half)
    assert H.predict_hs(64, 4096, 16384)[:2] == (70, 64)
    assert H.predict_lola_dense(64, 4096)[0] == 768
    assert H.predict_lola_stacked(64, 4096, 16384)[:2] == (255, 16)


def test_all_kernels_match_naive_on_random_triples():  # test_matvec.cpp:198-220
    rng = np.random.default_rng(23)
    for _ in range(150):
        m = 1 + int(rng.integers(24))
        n = 1 + int(rng.integers(100))
        N = H.next_power_of_two(max(m + n - 1, 2))
        if rng.integers(2):
            N *= 2
        A = rng.uniform(-1, 1, (m, n))
        x = rng.uniform(-1, 1, n)
        want = A @ x
        v = H.pack(x, N, H.CIPHERTEXT)
        ctx = H.MeterContext()
        hs = H.hs_matvec(A, v, ctx)
        dn = H.lola_dense_matvec(A, v, ctx)
        st, sor = H.lola_stacked_matvec(A, v, ctx)
        for i in range(m):
            tol = 1e-9 * max(1, abs(want[i]))
            assert abs(hs[i] - want[i]) < tol
            assert abs(dn[i][0] - want[i]) < tol
            assert abs(st[sor[i]] - want[i]) < tol


def test_lola_metering_equals_prediction():  # test_matvec.cpp:249-283 (LoLa part, reduced grid)
    rng = np.random.default_rng(31)
    for N in (4096, 16384):
        for n in (16, 64, 256, 1024):
            for m in (4, 16, 64):
                A = rng.uniform(-1, 1, (m, n)) + 2.0
                v = H.pack(rng.uniform(-1, 1, n), N, H.CIPHERTEXT)
                dn = H.MeterContext()
                H.lola_dense_matvec(A, v, dn)
                assert (dn.tally.rot, dn.tally.mul_pc) == H.predict_lola_dense(m, n)[:2]
                st = H.MeterContext()
                H.lola_stacked_matvec(A, v, st)
                assert (st.tally.rot, st.tally.mul_pc) == H.predict_lola_stacked(m, n, N)[:2]


def test_figure2_regime_hs_dominates():  # test_matvec.cpp:285-296
    for N in (4096, 16384):
        for n in (256, 512, 1024, 2048, 4096):
            for m in (64, 128, 256, 512):
                hs = H.predict_hs(m, n, N)[0]
                assert hs < min(H.predict_lola_dense(m, n)[0], H.predict_lola_stacked(m, n, N)[0])
