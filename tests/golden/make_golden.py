"""Generates the committed golden fixtures of tests/golden/ (run from the repo
root: python tests/golden/make_golden.py).

reference_kats.json -- the reference's own known-answer vectors for the hot
    path, restated literally from its tests (file:line in each entry) and the
    golden HOP tables of SURVEY.md §8d; tests/test_golden.py checks the
    slot-level oracle (oracle/hesim_oracle.py) against every entry.
ckks_small.json -- CKKS limb fixtures at N = 2^10 from the CPU oracle
    (oracle/ckks.py, builder-authored: no CKKS exists in the reference):
    sha256 of each op's output limbs + decrypted slots.  tests/test_golden.py
    checks the oracle against them on CPU and the CUDA path against them on
    the GPU, so GPU parity does not depend on the oracle at run time.
ckks_programs.json -- the general stage driver: the reference's lowering
    KATs (stage labels, the `ce` totals) and, from the CPU oracle, the output
    ciphertext hash, logits and per-stage HOP rows of the scaled-down `ce`
    and the LoLa-dense model (tests/test_program.py).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

SMALL = {"log_n": 10, "qbits": [60, 40, 40, 40, 40], "pbits": 60, "seed": 77}
DELTA = 2.0 ** 40


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint64).tobytes()).hexdigest()


def reference_kats():
    return {
        "rotate": {"src": "proj/tests/test_slotvec.cpp:34-64", "v": [1, 2, 3, 4],
                   "right1": [4, 1, 2, 3], "left1": [2, 3, 4, 1]},
        "diagonals_2x2": {"src": "proj/tests/test_matvec.cpp:35-45", "A": [[1, 2], [3, 4]],
                          "masks": [[1, 4], [3, 2]]},
        "hs_2x2": {"src": "proj/tests/test_matvec.cpp:88-97", "A": [[1, 2], [3, 4]], "x": [5, 6], "Ax": [17, 39]},
        "rotate_and_sum": {"src": "proj/tests/test_matvec.cpp:66-86",
                           "v8": [1, 2, 3, 4, 5, 6, 7, 8], "sum8": 36, "rot8": 3,
                           "w": [5, 39, 12, 0], "span": 3, "block": 2, "head": [17, 39], "rotw": 1},
        "hs_100x845": {"src": "proj/tests/test_matvec.cpp:110-123", "m": 100, "n": 845, "N": 8192,
                       "mul_pc": 100, "rot_range": [103, 104]},
        "predict_hs": {"src": "proj/tests/test_matvec.cpp:125-131", "m": 64, "n": 4096, "N": 16384, "rot": 70},
        "lola": {"src": "proj/tests/test_matvec.cpp:157-196",
                 "dense_64_4096": [768, 64], "dense_1_2_rot": 1, "stacked_64_4096_16384": [255, 16],
                 "stacked_4_3_8_rot": 7, "stacked_4_16_64_rot": 7},
        "conv_taps_3x3_k2": {"src": "proj/tests/test_convlower.cpp:32-41 (taps 0, 1, 3; tap 2 by conv_pack's rule)",
                             "img": [[1, 2, 3], [4, 5, 6], [7, 8, 9]], "n_slots": 4,
                             "taps": [[1, 2, 4, 5], [2, 3, 5, 6], [4, 5, 7, 8], [5, 6, 8, 9]]},
        "conv_counts": {"src": "proj/tests/test_convlower.cpp:63-96",
                        "cases": [{"d_in": 29, "c_in": 1, "k": 5, "s": 2, "c_out": 5, "mul_pc": 125, "add_cc": 120,
                                   "add_pc": 5},
                                  {"d_in": 30, "c_in": 1, "k": 3, "s": 1, "c_out": 5, "mul_pc": 45, "add_cc": 40,
                                   "add_pc": 5},
                                  {"d_in": 32, "c_in": 3, "k": 3, "s": 1, "c_out": 18, "mul_pc": 486,
                                   "add_cc": 468, "add_pc": 18}]},
        "merge_5x169": {"src": "proj/tests/test_convlower.cpp:171-188", "c": 5, "w": 169, "N": 1024,
                        "rot": 4, "add_cc": 4},
        "cfg0_stage_hops": {"src": "SURVEY.md §8d (derived from proj/src/netcompile.cpp:291-446)",
                            "order": ["add_pc", "add_cc", "mul_pc", "mul_cc", "rot"],
                            "stages": {"Conv1": [5, 120, 125, 0, 0], "Flat1": [0, 4, 0, 0, 4],
                                       "Square1": [0, 0, 0, 1, 0], "Dense1": [1, 103, 100, 0, 103],
                                       "Square2": [0, 0, 0, 1, 0], "Dense2": [1, 13, 10, 0, 13]},
                            "total": 604},
        "cfg3_totals": {"src": "SURVEY.md §8d", "hops": [34, 2673, 2666, 2, 305], "total": 5680},
    }


def ckks_fixtures():
    from oracle import ckks_pipeline as P
    from oracle.ckks import Ckks
    ck = Ckks(SMALL["log_n"], SMALL["qbits"], SMALL["pbits"], seed=SMALL["seed"])
    rng = np.random.default_rng(5)
    l = 4
    z = rng.uniform(-1, 1, ck.S)
    pt = ck.encode(z, DELTA, l)
    ct = ck.encrypt(pt, l, 3)
    w = rng.uniform(-1, 1, ck.S)
    wpt = ck.encode(w, DELTA, l)
    keys = {}
    g = ck.galois_right(3)
    rot = ck.rotate(ct, l, g, ck.galois_key(g))
    mul = ck.mul_pc(ct, wpt, l)
    resc = ck.rescale(mul, l)
    sq = ck.rescale(ck.square(ct, l, ck.relin_key()), l)
    A = rng.normal(0, 0.05, (10, 100))
    zx = rng.uniform(-1, 1, 100)
    ctx_ = ck.encrypt(ck.encode(zx, DELTA, l), l, 4)
    hs = P.hs_matvec(ck, ctx_, l, A, True, keys)
    out = {"params": SMALL, "level": l, "z_seed": 5,
           "primes": [int(p) for p in ck.primes],
           "pt": sha(pt), "ct": sha(ct), "rot3": sha(rot), "mul_pc": sha(mul), "rescale": sha(resc),
           "square_rescale": sha(sq), "hs_10x100": sha(hs),
           "dec_rot3_head": [float(x) for x in ck.decrypt_decode(rot, l, DELTA)[:4]],
           "dec_hs_head": [float(x) for x in ck.decrypt_decode(hs, l - 1, DELTA)[:10]]}
    return out


def program_fixtures():
    """the general stage driver (SubConv groups, RepackConv, LoLa-dense): the
    CPU oracle's output ciphertext of the scaled-down `ce` and the LoLa-dense
    model of tests/test_program.py, plus the reference KATs of the lowering
    (proj/tests/test_netcompile.cpp:40-54, :139-152)"""
    from oracle import ckks_pipeline as P
    from oracle import hesim_oracle as HS
    from oracle.ckks import Ckks
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import test_program as T
    out = {"lowering_kats": {
        "src": "proj/tests/test_netcompile.cpp:40-54,139-152",
        "cryptonets-hs": ["Conv1", "Flat1", "Square1", "Conv2-Dense1", "Square2", "Dense2"],
        "me_stages": 6,
        "ce": ["Conv1", "Flat1", "Square1", "Pool1-Conv2", "Conv3", "Flat2", "Square2", "Pool2-Dense1", "Square3",
               "Dense2"],
        "ce_conv1": [18, 468, 486, 0, 0],
        "ce_published_totals": {"total": 11134, "add_pc": 85, "add_cc": 4092, "mul_pc": 4080, "mul_cc": 5,
                                "rot": 2872, "tolerance_pct": 5}}}
    for name, model, qbits, log_n, seed in (("ce_mini", T.CE_MINI, T.CE_MINI_QBITS, 12, 5),
                                            ("ld_mini", T.LD_MINI, T.LD_MINI_QBITS, 10, 6)):
        flat, img = T._weights(model, seed)
        w = HS.split_model_weights(model, flat)
        ck = Ckks(log_n, qbits, 45, seed=7)
        ct, l, scale, n = P.run_program(ck, model, w, img, nonce=2)
        mc = HS.MeterContext()
        HS.execute_program(model, w, img, mc)
        out[name] = {"log_n": log_n, "qbits": qbits, "pbits": 45, "ctx_seed": 7, "weights_seed": seed, "nonce": 2,
                     "level": l, "scale": scale, "n_logits": n, "out_ct": sha(ct),
                     "logits": [float(x) for x in np.real(ck.decrypt_decode(ct, l, scale)[:n])],
                     "stages": [[lab, [t.add_pc, t.add_cc, t.mul_pc, t.mul_cc, t.rot]] for lab, t in mc.stages]}
    return out


if __name__ == "__main__":
    with open(os.path.join(HERE, "ckks_programs.json"), "w") as f:
        json.dump(program_fixtures(), f, indent=1)
    with open(os.path.join(HERE, "reference_kats.json"), "w") as f:
        json.dump(reference_kats(), f, indent=1)
    with open(os.path.join(HERE, "ckks_small.json"), "w") as f:
        json.dump(ckks_fixtures(), f, indent=1)
    print("wrote", os.listdir(HERE))
