"""The reference's `ce` builtin (proj/src/netcompile.cpp:607-628; ten stages,
three SubConv groups, the 1x1 conv-pack repack, n_slots = 16384 -> N = 2^15)
encrypted end to end through `hegpu_cli run`: logits within 1e-3 of the FP64
forward pass, per-stage HOP rows equal to the reference's execute
(proj/tests/test_netcompile.cpp:139-152 bounds its totals).  Runs last (file
name): ~1200 rotation keys and the fused key tables take ~140 GB of HBM."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_ce_builtin_runs_encrypted():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "run_ce.py"), "--model", "ce"],
                       capture_output=True, text=True, timeout=1500)
    assert r.returncode == 0, r.stdout + r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["max_abs_logit_err"] < 1e-3 and d["hops_equal_reference"]
    assert d["stages"] == ["Conv1", "Flat1", "Square1", "Pool1-Conv2", "Conv3", "Flat2", "Square2", "Pool2-Dense1",
                           "Square3", "Dense2"]
    total = int(d["total"][0])
    assert abs(total - 11134) * 20 <= 11134   # within 5 % of the published breakdown
