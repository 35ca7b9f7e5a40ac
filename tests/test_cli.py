"""hegpu_cli: the reference CLI's commands, exit
codes (0 ok, 1 I/O, 2 capacity/shape, 3 verification) and CSV formats
(proj/tools/hesim.cpp) over the encrypted path."""
import os
import subprocess

import numpy as np
import pytest

from oracle import hesim_oracle as HS
from paper_2110_08321_b200 import build as B
from paper_2110_08321_b200 import hegpu as H

CLI = B.CLI


def cli(*args, **kw):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=kw.get("timeout", 600))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def test_sweep_matches_predictions():
    """cmd_sweep (hesim.cpp:142-208): all three methods by default"""
    r = cli("sweep", "--n-min", "16", "--n-max", "1024", "--m-min", "4", "--m-max", "256", "--n-slots", "4096,16384")
    assert r.returncode == 0, r.stderr
    lines = r.stdout.strip().splitlines()
    assert lines[0] == "method,n,m,N,rotations,multiplications"
    rows = [l.split(",") for l in lines[1:]]
    assert len(rows) == 3 * 7 * 7 * 2
    pred = {"hs": lambda m, n, N: HS.predict_hs(m, n, N), "lola-dense": lambda m, n, N: HS.predict_lola_dense(m, n),
            "lola-stacked": lambda m, n, N: HS.predict_lola_stacked(m, n, N)}
    assert [r[0] for r in rows[::98]] == ["hs", "lola-dense", "lola-stacked"]
    for method, n, m, N, rot, mul in rows:
        want = pred[method](int(m), int(n), int(N))
        assert (int(rot), int(mul)) == (want[0], want[1])


def test_exit_codes_without_gpu(tmp_path):
    assert cli("run", "--model", "/no/such/model.json").returncode == 1   # IoError
    bad = tmp_path / "stacked.json"                                       # a LoLa-stacked stage policy: ShapeError
    bad.write_text('{"name": "s", "input": [1, 4, 4], "n_slots": 512, "layers": [{"kind": "flatten"}, '
                   '{"kind": "dense", "units": 6, "policy": "lola-stacked", "label": "D1"}]}')
    assert cli("count", "--model", str(bad)).returncode == 2
    assert cli("frobnicate").returncode == 2
    assert cli("sweep", "--methods", "lola-sparse").returncode == 2


@pytest.mark.gpu
def test_run_count_verify_on_gpu(tmp_path):
    from test_modelio import CRYPTONETS_JSON, cryptonets_weights
    (tmp_path / "m.json").write_text(CRYPTONETS_JSON)
    m, w = cryptonets_weights(9)
    m.save_weights(tmp_path / "w.bin", w)
    x = np.random.default_rng(9).uniform(0, 1, (1, 29, 29))
    m.save_input(tmp_path / "x.bin", x)
    r = cli("run", "--model", str(tmp_path / "m.json"), "--weights", str(tmp_path / "w.bin"),
            "--input", str(tmp_path / "x.bin"), "--report", str(tmp_path / "r.csv"))
    assert r.returncode == 0, r.stderr
    logits = np.array([float(l.split(",")[2]) for l in r.stdout.splitlines() if l.startswith("logit,")])
    want = HS.ref_forward_layers(m.layers, HS.split_weights(m.layers, 1, 29, w), m.load_input(tmp_path / "x.bin"))
    assert np.abs(logits - want).max() < 1e-3
    rep = (tmp_path / "r.csv").read_text().splitlines()
    assert rep[0] == "layer,total,add_pc,add_cc,mul_pc,mul_cc,rot"
    assert [l.split(",")[0] for l in rep[1:]] == ["Conv1", "Flat1", "Square1", "Conv2-Dense1", "Square2", "Dense2",
                                                  "Total"]
    c = cli("count", "--model", "cryptonets-hs", "--seed", "3")
    assert c.returncode == 0, c.stderr
    assert "Conv2-Dense1" in c.stdout and c.stdout.strip().splitlines()[-1].startswith("Total")
    v = cli("verify", "--cases", "3", timeout=1200)
    assert v.returncode == 0, v.stdout + v.stderr
    assert "verify: PASS" in v.stdout


@pytest.mark.gpu
def test_run_grouped_model_through_the_general_driver(tmp_path):
    """a model with SubConv groups and a stand-alone conv-pack repack (ce's
    stage list, scaled down) runs through hegpu_prog: logits, stage labels
    and the per-stage HOP rows of the reference's execute"""
    from test_program import CE_MINI, _weights
    (tmp_path / "m.json").write_text(HS.model_json(CE_MINI))
    m = H.Model.parse(HS.model_json(CE_MINI))
    flat, img = _weights(CE_MINI, 11)
    m.save_weights(tmp_path / "w.bin", flat)
    m.save_input(tmp_path / "x.bin", img)
    r = cli("run", "--model", str(tmp_path / "m.json"), "--weights", str(tmp_path / "w.bin"),
            "--input", str(tmp_path / "x.bin"), "--report", str(tmp_path / "r.csv"))
    assert r.returncode == 0, r.stderr
    logits = np.array([float(l.split(",")[2]) for l in r.stdout.splitlines() if l.startswith("logit,")])
    w = HS.split_model_weights(CE_MINI, flat)
    assert np.abs(logits - HS.ref_forward_model(CE_MINI, w, img)).max() < 1e-3
    mc = HS.MeterContext()
    HS.execute_program(CE_MINI, w, img, mc)
    rows = [l.split(",") for l in (tmp_path / "r.csv").read_text().splitlines()[1:]]
    assert [(r[0], tuple(int(v) for v in r[2:])) for r in rows[:-1]] == \
        [(lab, (t.add_pc, t.add_cc, t.mul_pc, t.mul_cc, t.rot)) for lab, t in mc.stages]
    c = cli("count", "--model", "ce-mini", "--seed", "3")
    assert c.returncode == 0, c.stderr
    assert "Pool1-Conv2" in c.stdout and "Conv3" in c.stdout


@pytest.mark.gpu
def test_policy_flag_changes_the_accounting(tmp_path):
    """--policy lola-dense (hesim.cpp:43-48): me's linear stages run the
    LoLa-dense kernel -- more rotations than the 56 of the HS pipeline, the
    same logits (proj/tests/test_netcompile.cpp:190-205)"""
    me = HS.builtin_model("me")
    (tmp_path / "m.json").write_text(HS.model_json(me))
    m = H.Model.parse(HS.model_json(me))
    rng = np.random.default_rng(3)
    flat = rng.normal(0, 0.05, HS.model_weight_count(me)).astype(np.float32).astype(np.float64)
    img = rng.uniform(0, 1, (1, 30, 30)).astype(np.float32).astype(np.float64)
    m.save_weights(tmp_path / "w.bin", flat)
    m.save_input(tmp_path / "x.bin", img)
    r = cli("run", "--model", str(tmp_path / "m.json"), "--weights", str(tmp_path / "w.bin"),
            "--input", str(tmp_path / "x.bin"), "--report", str(tmp_path / "r.csv"), "--policy", "lola-dense")
    assert r.returncode == 0, r.stderr
    logits = np.array([float(l.split(",")[2]) for l in r.stdout.splitlines() if l.startswith("logit,")])
    w = HS.split_model_weights(me, flat)
    assert np.abs(logits - HS.ref_forward_model(me, w, img)).max() < 1e-3
    mc = HS.MeterContext()
    HS.execute_program(dict(me, default_policy="lola-dense"), w, img, mc)
    rows = [l.split(",") for l in (tmp_path / "r.csv").read_text().splitlines()[1:]]
    assert [(x[0], tuple(int(v) for v in x[2:])) for x in rows[:-1]] == \
        [(lab, (t.add_pc, t.add_cc, t.mul_pc, t.mul_cc, t.rot)) for lab, t in mc.stages]
    assert int(rows[-1][6]) > 56
    assert cli("count", "--model", "me", "--policy", "lola-stacked").returncode == 2


@pytest.mark.gpu
def test_verify_negative_control_exits_3():
    """--corrupt-kernel perturbs the expected A x, so verify must report FAIL
    and exit 3 (proj/tools/hesim.cpp:212,237,334-337;
    proj/tests/acceptance.cpp:232-238)"""
    v = cli("verify", "--cases", "2", "--corrupt-kernel", timeout=1200)
    assert v.returncode == 3, v.stdout + v.stderr
    assert "verify: FAIL" in v.stdout


@pytest.mark.gpu
def test_sweep_measure_on_gpu():
    """sweep --measure (hesim.cpp:119-140): every method runs on the GPU and
    its metered rotations / multiplications equal the prediction for dense
    matrices (test_matvec.cpp:249-283)"""
    r = cli("sweep", "--n-min", "16", "--n-max", "64", "--m-min", "4", "--m-max", "16", "--n-slots", "4096",
            "--measure")
    assert r.returncode == 0, r.stderr
    rows = [l.split(",") for l in r.stdout.strip().splitlines()[1:]]
    assert len(rows) == 3 * 3 * 3
    for method, n, m, N, rot, mul, mrot, mmul in rows:
        assert (mrot, mmul) == (rot, mul), (method, n, m, N)
