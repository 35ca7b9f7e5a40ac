"""Model / weights / input files (the reference's
proj/src/modelio.cpp:106-248 behaviour; cases restated from
proj/tests/test_netcompile.cpp "model json round trip and validation" and
"weights and input files round trip").  Host-only: runs without a GPU."""
import numpy as np
import pytest

from oracle import hesim_oracle as HS
from paper_2110_08321_b200 import hegpu as H
from paper_2110_08321_b200.workloads import CFG0, net_weights

TINY = """{
  "name": "tiny",
  "input": [1, 4, 4],
  "n_slots": 32,
  "layers": [
    {"kind": "conv", "k": 3, "s": 1, "out_channels": 2, "label": "Conv1"},
    {"kind": "square"},
    {"kind": "flatten"},
    {"kind": "dense", "units": 3, "label": "Dense1"}
  ]
}"""

CFG0_JSON = """{"name": "cfg0-mnist", "input": [1, 29, 29], "n_slots": 4096, "layers": [
  {"kind": "conv", "k": 5, "s": 2, "out_channels": 5, "policy": "convpack", "label": "Conv1"},
  {"kind": "square"}, {"kind": "flatten"},
  {"kind": "dense", "units": 100, "policy": "hs", "label": "Dense1"},
  {"kind": "square"},
  {"kind": "dense", "units": 10, "label": "Dense2"}]}"""


def test_parse_tiny_model():
    m = H.Model.parse(TINY)
    assert (m.in_c, m.in_d, m.n_slots) == (1, 4, 4 * 8)
    assert [l["kind"] for l in m.layers] == ["conv", "square", "flatten", "dense"]
    assert m.layers[3]["out"] == 3 and m.layers[0]["k"] == 3
    # conv 2x1x3x3 + 2, dense 3 x (2*2*2) + 3
    assert m.weight_floats == 2 * 9 + 2 + 3 * 8 + 3
    spec = m.net_spec()
    assert (spec.k, spec.stride, spec.c_out, spec.n_dense, spec.dense_out[0]) == (3, 1, 2, 1, 3)


@pytest.mark.parametrize("text", [
    '{"name":"x"}',                                                          # missing fields
    '{"name":"x","input":[1,2,2],"n_slots":8,"layers":[],"extra":1}',         # unknown top-level key
    '{"name":"x","input":[1,2,2],"n_slots":8,"layers":[{"kind":"dense","units":1,"typo_field":2}]}',
    '{"name":"x","input":[1,2,3],"n_slots":8,"layers":[]}',                  # non-square input
    '{"name":"x","input":[1,2,2],"n_slots":8,"layers":[{"kind":"maxpool"}]}',  # unknown kind
    '{"name":"x","input":[1,2,2],"n_slots":8,"layers":[{"kind":"dense","policy":"fft"}]}',
    '{"name":"x","input":[1,2,2],"n_slots":8,"layers":[',                     # truncated JSON
])
def test_model_validation_rejects(text):
    with pytest.raises(H.IoError):
        H.Model.parse(text)


def test_pool_inside_a_linear_run_is_lowered():
    m = H.Model.parse('{"name":"p","input":[1,8,8],"n_slots":64,"layers":['
                      '{"kind":"conv","k":3,"out_channels":2},{"kind":"square"},'
                      '{"kind":"avgpool","k":2,"s":2},{"kind":"dense","units":3}]}')
    spec = m.net_spec()   # conv -> square -> [avgpool, dense] fused into one HS layer
    assert (spec.n_dense, spec.dense_out[0]) == (1, 3)
    # a square must follow the conv
    bad = H.Model.parse('{"name":"q","input":[1,8,8],"n_slots":64,"layers":['
                        '{"kind":"conv","k":3,"out_channels":2},{"kind":"dense","units":3}]}')
    with pytest.raises(H.ShapeError):
        bad.net_spec()


def test_load_resolves_model_dir(tmp_path, monkeypatch):
    (tmp_path / "cfg0.json").write_text(CFG0_JSON)
    monkeypatch.setenv("HECNN_MODEL_DIR", str(tmp_path))
    m = H.Model.load("cfg0")
    assert [l["out"] for l in m.layers if l["kind"] == "dense"] == [100, 10]
    assert m.layers[0]["policy"] == "convpack" and m.layers[5]["policy"] is None
    with pytest.raises(H.IoError):
        H.Model.load("no-such-model")


def flat_weights(w):
    parts = [np.ravel(w["conv_w"]), np.ravel(w["conv_b"])]
    for W, b in w["dense"]:
        parts += [np.ravel(W), np.ravel(b)]
    return np.concatenate(parts)


def test_weights_and_input_round_trip(tmp_path):
    m = H.Model.parse(CFG0_JSON)
    w = flat_weights(net_weights(CFG0, 11))
    assert w.size == m.weight_floats
    m.save_weights(tmp_path / "w.bin", w)
    back = m.load_weights(tmp_path / "w.bin")
    assert np.array_equal(back, w.astype(np.float32).astype(np.float64))  # float32 serialisation
    x = np.random.default_rng(11).uniform(0, 1, (1, 29, 29))
    m.save_input(tmp_path / "i.bin", x)
    assert np.array_equal(m.load_input(tmp_path / "i.bin"), x.astype(np.float32).astype(np.float64))
    (tmp_path / "t.bin").write_bytes(b"xy")                 # truncated
    with pytest.raises(H.IoError):
        m.load_weights(tmp_path / "t.bin")
    (tmp_path / "x.bin").write_bytes((tmp_path / "i.bin").read_bytes() + b"\0")  # trailing bytes
    with pytest.raises(H.IoError):
        m.load_input(tmp_path / "x.bin")
    with pytest.raises(H.IoError):
        m.load_weights(tmp_path / "missing.bin")


# the reference's builtin cryptonets-hs layer list (netcompile.cpp:567-585) as
# a model file, with slot count sized for the N = 8192 ring
CRYPTONETS_JSON = """{"name": "cryptonets-hs", "input": [1, 29, 29], "n_slots": 4096, "layers": [
  {"kind": "conv", "k": 5, "s": 2, "out_channels": 5, "label": "Conv1"},
  {"kind": "square"},
  {"kind": "avgpool", "k": 2, "s": 2},
  {"kind": "conv", "k": 5, "s": 1, "out_channels": 50, "label": "Conv2"},
  {"kind": "avgpool", "k": 2, "s": 2},
  {"kind": "flatten"},
  {"kind": "dense", "units": 100, "label": "Dense1"},
  {"kind": "square"},
  {"kind": "dense", "units": 10, "label": "Dense2"}]}"""


def cryptonets_weights(seed=5):
    m = H.Model.parse(CRYPTONETS_JSON)
    rng = np.random.default_rng(seed)
    return m, rng.normal(0, 0.05, m.weight_floats).astype(np.float32).astype(np.float64)


def test_lower_composes_linear_runs():
    """lower(): the avgpool-conv-avgpool-flatten-dense run is one affine map,
    equal to the oracle's compose_run (netcompile.cpp:225-278)"""
    m, w = cryptonets_weights()
    spec = m.net_spec()
    assert (spec.c_out, spec.n_dense, spec.dense_out[0], spec.dense_out[1]) == (5, 2, 100, 10)
    per_layer = HS.split_weights(m.layers, m.in_c, m.in_d, w)
    M, b = m.compose(w, 0)
    Mo, bo = HS.compose_run(m.layers[2:7], per_layer[2:7], 5, 13)
    assert M.shape == (100, 845)
    assert np.abs(M - Mo).max() < 1e-12 and np.abs(b - bo).max() < 1e-12
    M2, b2 = m.compose(w, 1)
    assert np.array_equal(M2, per_layer[8][0]) and np.array_equal(b2, per_layer[8][1])
    # the lowered net computes the reference forward pass in cleartext
    x = np.random.default_rng(1).uniform(0, 1, (1, 29, 29))
    t = HS.ref_square(HS.ref_conv(x, *per_layer[0], 2)).ravel()
    y = M2 @ HS.ref_square(M @ t + b) + b2
    assert np.abs(y - HS.ref_forward_layers(m.layers, per_layer, x)).max() < 1e-10


def test_lower_rejects_outside_family():
    sub = H.Model.parse('{"name":"g","input":[2,8,8],"n_slots":64,"layers":['
                        '{"kind":"conv","k":3,"out_channels":4},{"kind":"square"},'
                        '{"kind":"subconv","k":3,"out_channels":4,"groups":2},{"kind":"dense","units":3}]}')
    with pytest.raises(H.ShapeError):
        sub.net_spec()
    lola = H.Model.parse('{"name":"l","input":[1,8,8],"n_slots":64,"layers":['
                         '{"kind":"conv","k":3,"out_channels":2},{"kind":"square"},'
                         '{"kind":"dense","units":3,"policy":"lola-dense"}]}')
    with pytest.raises(H.ShapeError):
        lola.net_spec()
