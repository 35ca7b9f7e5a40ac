"""The general stage driver: lower() + execute() with
SubConv groups, grouped merges, RepackConv and the LoLa-dense policy
(proj/src/netcompile.cpp:106-213, 291-446).

CPU: the slot-level restatement is pinned to the reference's own tests for
this path (proj/tests/test_netcompile.cpp:40-54 stage labels, :139-152 the
`ce` totals within 5 % of the published breakdown); the C++ lowering
(hegpu_model_lower) equals it stage for stage; the CKKS-level oracle
pipeline decrypts to the FP64 forward pass.
GPU: hegpu_prog runs a scaled-down `ce` (same layer list, shapes that fit
N = 4096) and a LoLa-dense model encrypted: limbs bit-exact against the CPU
oracle, logits within 1e-3 of ref_forward, the per-stage HOP report equal to
the slot-level execute()."""
import numpy as np
import pytest

from oracle import hesim_oracle as HS

L = HS._L

CE_MINI = dict(name="ce-mini", in_c=3, in_d=16, n_slots=2048, layers=[
    L("conv", 3, 1, 6, label="Conv1"), L("square"), L("avgpool", 2, 2, label="Pool1"),
    L("subconv", 3, 1, 6, 3, label="Conv2"), L("conv", 1, 1, 8, policy="convpack", label="Conv3"),
    L("square"), L("avgpool", 2, 2, label="Pool2"), L("conv", 2, 1, 12), L("flatten"),
    L("dense", out=16, label="Dense1"), L("square"), L("dense", out=10, label="Dense2")])
CE_MINI_QBITS = [45] + [40] * 8  # 8 primes consumed (conv, 3 squares, 3 HS, the repack conv)

# no conv-pack first layer (dense input ciphertext), a LoLa-dense stage
LD_MINI = dict(name="ld-mini", in_c=1, in_d=4, n_slots=512, layers=[
    L("flatten"), L("dense", out=6, policy="lola-dense", label="D1"), L("square"),
    L("dense", out=4, label="D2")])
LD_MINI_QBITS = [45] + [40] * 4  # lola-dense 2, square 1, HS 1


def _weights(model, seed, sigma=0.3):
    rng = np.random.default_rng(seed)
    flat = rng.normal(0, sigma, HS.model_weight_count(model)).astype(np.float32).astype(np.float64)
    img = rng.uniform(0, 1, (model["in_c"], model["in_d"], model["in_d"])).astype(np.float32).astype(np.float64)
    return flat, img


def _tallies(ctx):
    return [(lab, (t.add_pc, t.add_cc, t.mul_pc, t.mul_cc, t.rot)) for lab, t in ctx.stages]


# ------------------------------------------------------------------ CPU ---
def test_lower_stage_labels_reference_kats():
    """proj/tests/test_netcompile.cpp:40-54"""
    assert [s["label"] for s in HS.lower(HS.builtin_model("cryptonets-hs"))] == \
        ["Conv1", "Flat1", "Square1", "Conv2-Dense1", "Square2", "Dense2"]
    assert len(HS.lower(HS.builtin_model("me"))) == 6
    ce = HS.lower(HS.builtin_model("ce"))
    assert [s["label"] for s in ce] == ["Conv1", "Flat1", "Square1", "Pool1-Conv2", "Conv3", "Flat2", "Square2",
                                        "Pool2-Dense1", "Square3", "Dense2"]
    assert [s["groups"] for s in ce][:4] == [1, 3, 1, 3]


def test_lower_no_adjacent_linear_layers_unchanged():
    """proj/tests/test_netcompile.cpp:56-72, 74-97"""
    toy = dict(name="toy", in_c=1, in_d=2, n_slots=8,
               layers=[L("dense", out=4, label="D1"), L("square"), L("dense", out=2, label="D2")])
    st = HS.lower(toy)
    assert [s["label"] for s in st] == ["D1", "Square1", "D2"] and st[1]["kind"] == "square"
    unit = dict(name="unit", in_c=1, in_d=1, n_slots=4, layers=[L("dense", out=1, label="D")])
    ctx = HS.MeterContext()
    lg = HS.execute_program(unit, [(np.array([[3.0]]), np.array([1.0]))], np.array([[[2.0]]]), ctx)
    assert lg[0] == pytest.approx(7.0) and ctx.tally.mul_pc == 1 and ctx.tally.rot == 0


def test_ce_totals_within_five_percent_of_published():
    """proj/tests/test_netcompile.cpp:139-152"""
    m = HS.builtin_model("ce")
    flat, img = _weights(m, 1, 0.05)
    w = HS.split_model_weights(m, flat)
    ctx = HS.MeterContext()
    lg = HS.execute_program(m, w, img, ctx)
    rows = dict(_tallies(ctx))
    assert rows["Conv1"] == (18, 468, 486, 0, 0)
    t = ctx.tally
    within = lambda got, want: abs(got - want) * 20 <= want  # noqa: E731
    assert within(t.add_pc + t.add_cc + t.mul_pc + t.mul_cc + t.rot, 11134)
    assert within(t.add_pc, 85) and within(t.add_cc, 4092) and within(t.mul_pc, 4080)
    assert t.mul_cc == 5 and within(t.rot, 2872)
    assert np.abs(lg - HS.ref_forward_model(m, w, img)).max() < 1e-7  # e2e bound, test_netcompile.cpp:173-189


def test_grouped_execute_matches_forward():
    for model in (CE_MINI, LD_MINI):
        flat, img = _weights(model, 3)
        w = HS.split_model_weights(model, flat)
        lg = HS.execute_program(model, w, img, HS.MeterContext())
        assert np.abs(lg - HS.ref_forward_model(model, w, img)).max() < 1e-9


def test_lola_stacked_policy_value_level():
    m = dict(LD_MINI, layers=[L("flatten"), L("dense", out=6, policy="lola-stacked", label="D1"), L("square"),
                              L("dense", out=4, label="D2")])
    flat, img = _weights(m, 4)
    w = HS.split_model_weights(m, flat)
    lg = HS.execute_program(m, w, img, HS.MeterContext())
    assert np.abs(lg - HS.ref_forward_model(m, w, img)).max() < 1e-9


def test_grouped_stage_requires_hs():
    bad = dict(CE_MINI, layers=[dict(l, policy="lola-dense") if l["kind"] == "subconv" else l
                                for l in CE_MINI["layers"]])
    with pytest.raises(HS.ShapeError):
        HS.lower(bad)


def test_cpp_lowering_equals_the_restatement():
    from paper_2110_08321_b200 import hegpu as H
    for model in (HS.builtin_model("cryptonets-hs"), HS.builtin_model("me"), HS.builtin_model("ce"), CE_MINI,
                  LD_MINI):
        got = H.Model.parse(HS.model_json(model)).lower()
        want = HS.lower(model)
        assert [(s["label"], s["kind"], s["groups"]) for s in got] == \
            [(s["label"], s["kind"], s["groups"]) for s in want]
        assert [s["policy"] for s in got if s["kind"] == "linear"] == \
            [s["policy"] for s in want if s["kind"] == "linear"]
        assert H.Model.parse(HS.model_json(model)).weight_floats == HS.model_weight_count(model)


def test_default_policy_changes_the_linear_stages():
    """ModelSpec::default_policy (netcompile.hpp:33-35, netcompile.cpp:178;
    test_netcompile.cpp:190-205): stages without a per-layer policy take it"""
    from paper_2110_08321_b200 import hegpu as H
    me = dict(HS.builtin_model("me"), default_policy="lola-dense")
    want = HS.lower(me)
    assert [s["policy"] for s in want if s["kind"] == "linear"] == ["lola-dense", "lola-dense"]
    m = H.Model.parse(HS.model_json(me))
    assert [s["policy"] for s in m.lower() if s["kind"] == "linear"] == ["hs", "hs"]
    m.set_default_policy("lola-dense")
    assert [(s["label"], s["policy"]) for s in m.lower() if s["kind"] == "linear"] == \
        [(s["label"], s["policy"]) for s in want if s["kind"] == "linear"]
    with pytest.raises(H.ShapeError):
        m.net_spec()   # the batched net is HS only; the general driver takes this model
    flat, img = _weights(me, 3, 0.05)
    w = HS.split_model_weights(me, flat)
    mc = HS.MeterContext()
    lg = HS.execute_program(me, w, img, mc)
    assert mc.tally.rot > 56
    assert np.abs(lg - HS.ref_forward_model(me, w, img)).max() < 1e-7
    m.set_n_slots(16)   # test_netcompile.cpp:207-211: an undersized slot count is a stage-named CapacityError
    with pytest.raises(H.CapacityError):
        m.lower()
    with pytest.raises(HS.CapacityError):
        HS.lower(dict(me, n_slots=16))


def test_workload_builtins_and_forward_match_the_restatement():
    """the product-side builtin model files and FP64 forward used by
    bench_configs.py --model (paper_2110_08321_b200/workloads.py) against the
    restated reference builtins and ref_forward"""
    from paper_2110_08321_b200 import hegpu as H
    from paper_2110_08321_b200.workloads import BUILTIN_MODEL_JSON, model_forward
    for name in ("cryptonets-hs", "me", "ce"):
        m = H.Model.parse(BUILTIN_MODEL_JSON[name])
        ref = H.Model.parse(HS.model_json(HS.builtin_model(name)))
        assert (m.in_c, m.in_d, m.n_slots, m.layers) == (ref.in_c, ref.in_d, ref.n_slots, ref.layers)
    mini = H.Model.parse(BUILTIN_MODEL_JSON["ce-mini"])
    assert mini.layers == H.Model.parse(HS.model_json(CE_MINI)).layers
    for model in (CE_MINI, HS.builtin_model("me"), LD_MINI):
        flat, img = _weights(model, 8, 0.1)
        m = H.Model.parse(HS.model_json(model))
        got = model_forward(m.layers, m.in_c, m.in_d, flat, img)
        want = HS.ref_forward_model(model, HS.split_model_weights(model, flat), img)
        assert np.abs(got - want).max() < 1e-9


def test_cpp_lowering_errors():
    from paper_2110_08321_b200 import hegpu as H
    bad = dict(CE_MINI, n_slots=1024)  # Pool1-Conv2: fused 150 x 1176 exceeds n_slots
    with pytest.raises(H.CapacityError):
        H.Model.parse(HS.model_json(bad)).lower()
    with pytest.raises(HS.CapacityError):
        HS.lower(bad)
    grouped_lola = dict(CE_MINI, layers=[dict(l, policy="lola-dense") if l["kind"] == "subconv" else l
                                         for l in CE_MINI["layers"]])
    with pytest.raises(H.ShapeError):
        H.Model.parse(HS.model_json(grouped_lola)).lower()


def test_ckks_oracle_program_decrypts_to_forward():
    from oracle import ckks_pipeline as P
    from oracle.ckks import Ckks
    for model, qbits, log_n in ((CE_MINI, CE_MINI_QBITS, 12), (LD_MINI, LD_MINI_QBITS, 10)):
        flat, img = _weights(model, 5)
        w = HS.split_model_weights(model, flat)
        ck = Ckks(log_n, qbits, 45, seed=7)
        ct, l, scale, n = P.run_program(ck, model, w, img, nonce=2)
        assert l == 1
        got = np.real(ck.decrypt_decode(ct, l, scale)[:n])
        assert np.abs(got - HS.ref_forward_model(model, w, img)).max() < 1e-3


# ------------------------------------------------------------------ GPU ---
def _run_gpu(model, qbits, log_n, seed):
    from oracle import ckks_pipeline as P
    from oracle.ckks import Ckks
    from paper_2110_08321_b200 import hegpu as H
    flat, img = _weights(model, seed)
    w = HS.split_model_weights(model, flat)
    ctx = H.Context(log_n, qbits, 45, seed=7, device=0)
    prog = H.Program(ctx, H.Model.parse(HS.model_json(model)), flat)
    assert [(s["label"], s["kind"], s["groups"]) for s in prog.stages] == \
        [(s["label"], s["kind"], s["groups"]) for s in HS.lower(model)]
    cts = prog.encrypt_input(img, nonce=2)
    out = ctx.ct(1, prog.out_level)
    ctx.reset_meter()
    launches0 = ctx.launches()
    prog.run(ctx.ct(prog.input_cts, prog.top, cts, 2.0 ** 40), out)
    assert ctx.launches() > launches0
    got = out.download()
    # limbs: the CPU oracle evaluating the same stages
    ck = Ckks(log_n, qbits, 45, seed=7)
    want, l, scale, n = P.run_program(ck, model, w, img, nonce=2)
    assert (l, n) == (prog.out_level, prog.n_logits) and scale == prog.out_scale
    assert np.array_equal(got, want), "GPU limbs differ from the CPU oracle"
    # logits against the FP64 forward pass (BASELINE tolerance 1e-3)
    ref = HS.ref_forward_model(model, w, img)
    logits = prog.decrypt_logits(got)
    assert np.abs(logits - ref).max() < 1e-3
    # the per-stage HOP report is the reference's
    mc = HS.MeterContext()
    HS.execute_program(model, w, img, mc)
    assert [(lab, tuple(t)) for lab, t in ctx.stages()] == _tallies(mc)
    return ctx


@pytest.mark.gpu
def test_prog_ce_mini_bit_exact_and_metered():
    _run_gpu(CE_MINI, CE_MINI_QBITS, 12, 5)


@pytest.mark.gpu
def test_prog_lola_dense_dense_seed():
    _run_gpu(LD_MINI, LD_MINI_QBITS, 10, 6)


@pytest.mark.gpu
@pytest.mark.parametrize("model,qbits,log_n,B", [(CE_MINI, CE_MINI_QBITS, 12, 3), (CE_MINI, CE_MINI_QBITS, 12, 8),
                                                 (LD_MINI, LD_MINI_QBITS, 10, 5)])
def test_prog_batches_match_single_image_runs(model, qbits, log_n, B):
    """B images per run (unit-major batches; from B = 8 the grouped HS stages
    take the tensor-core kernel): every image's limbs equal its own
    single-image run and the CPU oracle, the HOP report is B times one run's"""
    from oracle import ckks_pipeline as P
    from oracle.ckks import Ckks
    from paper_2110_08321_b200 import hegpu as H
    flat, _ = _weights(model, 5)
    w = HS.split_model_weights(model, flat)
    rng = np.random.default_rng(77)
    imgs = rng.uniform(0, 1, (B, model["in_c"], model["in_d"], model["in_d"]))
    ctx = H.Context(log_n, qbits, 45, seed=7, device=0)
    prog = H.Program(ctx, H.Model.parse(HS.model_json(model)), flat)
    cts = np.concatenate([prog.encrypt_input(imgs[b], nonce=10 + b) for b in range(B)])
    out = ctx.ct(B, prog.out_level)
    ctx.reset_meter()
    prog.run(ctx.ct(B * prog.input_cts, prog.top, cts, 2.0 ** 40), out)
    batch_rows = ctx.stages()
    got = out.download().reshape(B, -1)
    per = prog.input_cts * 2 * prog.top * ctx.N
    for b in (0, B - 1):
        one = ctx.ct(1, prog.out_level)
        ctx.reset_meter()
        prog.run(ctx.ct(prog.input_cts, prog.top, cts[b * per:(b + 1) * per], 2.0 ** 40), one)
        assert np.array_equal(got[b], one.download()), b
    assert batch_rows == [(lab, tuple(B * v for v in t)) for lab, t in ctx.stages()]
    ck = Ckks(log_n, qbits, 45, seed=7)
    want, _, _, _ = P.run_program(ck, model, w, imgs[B // 2], nonce=10 + B // 2)
    assert np.array_equal(got[B // 2], want)
    for b in range(B):
        assert np.abs(prog.decrypt_logits(got[b]) - HS.ref_forward_model(model, w, imgs[b])).max() < 1e-3


@pytest.mark.gpu
def test_prog_rejections():
    from paper_2110_08321_b200 import hegpu as H
    flat, _ = _weights(LD_MINI, 1)
    ctx = H.Context(10, LD_MINI_QBITS, 45, seed=7, device=0)
    stacked = dict(LD_MINI, layers=[L("flatten"), L("dense", out=6, policy="lola-stacked", label="D1"), L("square"),
                                    L("dense", out=4, label="D2")])
    with pytest.raises(H.ShapeError):
        H.Program(ctx, H.Model.parse(HS.model_json(stacked)), flat)
    short = H.Context(10, [45, 40, 40], 45, seed=7, device=0)  # chain too short for 4 primes
    with pytest.raises(H.CapacityError):
        H.Program(short, H.Model.parse(HS.model_json(LD_MINI)), flat)
    with pytest.raises(H.ShapeError):
        H.Program(ctx, H.Model.parse(HS.model_json(dict(LD_MINI, n_slots=1024))), flat)
