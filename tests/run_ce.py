"""Run the reference's `ce` builtin (proj/src/netcompile.cpp:607-628: CIFAR-shaped,
n_slots = 16384 -> N = 2^15, SubConv groups, the 1x1 conv-pack repack, ten
stages) encrypted through `hegpu_cli run` and compare the logits with the
FP64 forward pass and the per-stage HOP report with the slot-level execute.

    python tests/run_ce.py [--model ce] [--seed 1] [--sigma 0.05]

Needs a GPU with ~150 GB free (about 1200 rotation keys of 47 MB and the
fused key x mask tables of the 845-diagonal grouped HS stages)."""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import hesim_oracle as HS  # noqa: E402  (the checker)
from paper_2110_08321_b200 import build as B  # noqa: E402
from paper_2110_08321_b200 import hegpu as H  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="ce")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sigma", type=float, default=0.05)
    a = ap.parse_args()
    model = HS.builtin_model(a.model)
    rng = np.random.default_rng(a.seed)
    flat = rng.normal(0, a.sigma, HS.model_weight_count(model)).astype(np.float32).astype(np.float64)
    img = rng.uniform(0, 1, (model["in_c"], model["in_d"], model["in_d"])).astype(np.float32).astype(np.float64)
    w = HS.split_model_weights(model, flat)
    want = HS.ref_forward_model(model, w, img)
    mc = HS.MeterContext()
    HS.execute_program(model, w, img, mc)
    with tempfile.TemporaryDirectory() as d:
        mp, wp, xp, rp = (os.path.join(d, n) for n in ("m.json", "w.bin", "x.bin", "r.csv"))
        open(mp, "w").write(HS.model_json(model))
        m = H.Model.parse(HS.model_json(model))
        m.save_weights(wp, flat)
        m.save_input(xp, img)
        t = time.time()
        r = subprocess.run([B.CLI, "run", "--model", mp, "--weights", wp, "--input", xp, "--report", rp,
                            "--seed", str(a.seed)], capture_output=True, text=True)
        dt = time.time() - t
        if r.returncode:
            print(json.dumps({"model": a.model, "exit": r.returncode, "stderr": r.stderr.strip()[-400:]}))
            sys.exit(r.returncode)
        logits = np.array([float(l.split(",")[2]) for l in r.stdout.splitlines() if l.startswith("logit,")])
        rows = [l.split(",") for l in open(rp).read().splitlines()[1:]]
    got = [(x[0], tuple(int(v) for v in x[2:])) for x in rows[:-1]]
    ref = [(lab, (t.add_pc, t.add_cc, t.mul_pc, t.mul_cc, t.rot)) for lab, t in mc.stages]
    err = float(np.abs(logits - want).max())
    timing = [l for l in r.stderr.splitlines() if l.startswith("timing:")]
    print(json.dumps({"model": a.model, "n_slots": model["n_slots"], "wall_s": round(dt, 1),
                      "timing": timing[-1][8:] if timing else None,
                      "max_abs_logit_err": err, "logits": [round(float(v), 6) for v in logits],
                      "want": [round(float(v), 6) for v in want], "hops_equal_reference": got == ref,
                      "total": rows[-1][1:], "stages": [x[0] for x in rows[:-1]]}))
    sys.exit(0 if err < 1e-3 and got == ref else 3)


if __name__ == "__main__":
    main()
