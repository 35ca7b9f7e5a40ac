"""Seeded synthetic workloads for the BASELINE.json configs.

There is no public dataset on this path (BASELINE.json names "MNIST-sized"
and "CIFAR-10-shaped synthetic" inputs only); these generators stand in with
the stated shapes and distributions:
  - images U[0,1], MNIST 28x28 zero-padded bottom/right to 29x29
    (proj/src/netcompile.cpp:571 pads to 29 without naming the side);
  - weights N(0, sigma^2) (0.05 MNIST-sized, 0.02 CIFAR-shaped), biases
    N(0, 0.01^2), all rounded to f32 like the reference weight format
    (proj/src/modelio.cpp:54-70 reads little-endian f32 as double).
numpy's PCG64 is used so every host produces identical values.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class NetConfig:
    name: str
    in_c: int
    img_d: int        # unpadded image side
    in_d: int         # padded side fed to the conv
    k: int
    s: int
    c_out: int
    dense: tuple      # output units of the HS layers
    log_n: int        # ring degree N = 2^log_n; slots S = N/2
    qbits: tuple      # Q chain (q_0 first); len-1 rescales
    pbits: int        # special prime P
    w_sigma: float
    b_sigma: float = 0.01
    log_scale: int = 40

    @property
    def n_slots(self):
        return 1 << (self.log_n - 1)

    @property
    def d_out(self):
        return (self.in_d - self.k) // self.s + 1

    @property
    def n_taps(self):
        return self.k * self.k * self.in_c


# The benchmark prime chain: q_0 and P of 45 bits, five
# 40-bit primes for the five rescales at Delta = 2^40.  Every prime is below
# 2^45, so every NTT row runs on the FP64 butterflies (§5.1); q_0 leaves 4
# bits above Delta for the logits (|logit| < 16) and P >= q_0 bounds the
# hybrid key-switch noise.  The integer (64-bit Shoup) path stays for primes
# up to 2^60 (the 60-bit chains of the unit tests and the CLI).
QBITS_45 = (45, 40, 40, 40, 40, 40)
PBITS_45 = 45
# BASELINE.json configs[0] (and [2] = 64 of these)
CFG0 = NetConfig("cfg0-mnist", 1, 28, 29, 5, 2, 5, (100, 10), 13, QBITS_45, PBITS_45, 0.05)
# BASELINE.json configs[3]
CFG3 = NetConfig("cfg3-cifar", 3, 32, 32, 5, 2, 32, (256, 10), 14, QBITS_45, PBITS_45, 0.02)


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def net_weights(cfg: NetConfig, seed: int):
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x5EED]))
    w = {
        "conv_w": f32(rng.normal(0.0, cfg.w_sigma, (cfg.c_out, cfg.in_c, cfg.k, cfg.k))),
        "conv_b": f32(rng.normal(0.0, cfg.b_sigma, cfg.c_out)),
        "dense": [],
    }
    n = cfg.c_out * cfg.d_out ** 2
    for m in cfg.dense:
        W = f32(rng.normal(0.0, cfg.w_sigma, (m, n)))
        b = f32(rng.normal(0.0, cfg.b_sigma, m))
        w["dense"].append((W, b))
        n = m
    return w


def net_image(cfg: NetConfig, seed: int):
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x1A6E]))
    img = np.zeros((cfg.in_c, cfg.in_d, cfg.in_d))
    img[:, : cfg.img_d, : cfg.img_d] = f32(rng.uniform(0.0, 1.0, (cfg.in_c, cfg.img_d, cfg.img_d)))
    return img


def cfg0_weights_and_image(seed: int = 0):
    return net_weights(CFG0, seed), net_image(CFG0, seed)


def hs_sweep_case(m: int, n: int, seed: int = 0):
    """BASELINE.json configs[1]: A ~ N(0, 0.05^2) (m x n), v ~ U[-1, 1]^n."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, m, n]))
    return f32(rng.normal(0.0, 0.05, (m, n))), f32(rng.uniform(-1.0, 1.0, n))


# ---- client-side cleartext packing for the conv sweep (config 4) ----------
def conv_pack_image(image, k, s=1):
    """conv_pack (proj/src/convlower.cpp:9-37) on the client: tap t = (ci k +
    ky) k + kx holds img[ci, oy s + ky, ox s + kx] at slot oy d_out + ox"""
    image = np.asarray(image, dtype=np.float64)
    c_in, d_in = image.shape[0], image.shape[1]
    d_out = (d_in - k) // s + 1
    taps = []
    for ci in range(c_in):
        for ky in range(k):
            for kx in range(k):
                taps.append(image[ci, ky: ky + s * (d_out - 1) + 1: s, kx: kx + s * (d_out - 1) + 1: s].ravel())
    return taps


def conv_as_matrix(weights, d_in, s=1):
    """conv_to_matrix (proj/src/convlower.cpp:76-102): the conv as a
    (d_out^2 c_out) x (d_in^2 c_in) matrix for the HS formulation"""
    weights = np.asarray(weights, dtype=np.float64)
    c_out, c_in, k, _ = weights.shape
    d_out = (d_in - k) // s + 1
    A = np.zeros((d_out * d_out * c_out, d_in * d_in * c_in))
    oy, ox = np.meshgrid(np.arange(d_out), np.arange(d_out), indexing="ij")
    for co in range(c_out):
        rows = (co * d_out + oy) * d_out + ox
        for ci in range(c_in):
            for ky in range(k):
                for kx in range(k):
                    cols = (ci * d_in + oy * s + ky) * d_in + ox * s + kx
                    A[rows.ravel(), cols.ravel()] += weights[co, ci, ky, kx]
    return A


def plain_forward(cfg: NetConfig, weights, image):
    """the cleartext network (conv -> square -> dense -> square -> dense ...)
    in vectorised FP64 -- bench.py's sanity check on decrypted logits (the
    reference-order oracle ref_forward lives under oracle/ and is for tests)"""
    x = np.asarray(image, dtype=np.float64)
    W, b = np.asarray(weights["conv_w"]), np.asarray(weights["conv_b"])
    taps = conv_pack_image(x, cfg.k, cfg.s)  # [k^2 c_in] windows of d_out^2
    t = np.einsum("ot,tp->op", W.reshape(cfg.c_out, -1), np.stack(taps)) + b[:, None]
    flat = t.ravel()
    for Wd, bd in weights["dense"]:
        flat = np.asarray(Wd) @ (flat * flat) + np.asarray(bd)
    return flat


# ---- the reference's builtin layer lists (proj/src/netcompile.cpp:567-628) as
# model files, plus ce-mini (ce's ten stages scaled to N = 4096) -------------
BUILTIN_MODEL_JSON = {
    "cryptonets-hs": """{"name": "cryptonets-hs", "input": [1, 29, 29], "n_slots": 8192, "layers": [
        {"kind": "conv", "k": 5, "s": 2, "out_channels": 5, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 2, "s": 2}, {"kind": "conv", "k": 5, "s": 1, "out_channels": 50, "label": "Conv2"},
        {"kind": "avgpool", "k": 2, "s": 2}, {"kind": "flatten"}, {"kind": "dense", "units": 100, "label": "Dense1"},
        {"kind": "square"}, {"kind": "dense", "units": 10, "label": "Dense2"}]}""",
    "me": """{"name": "me", "input": [1, 30, 30], "n_slots": 8192, "layers": [
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 5, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 3, "s": 2}, {"kind": "conv", "k": 3, "s": 1, "out_channels": 50, "label": "Conv2"},
        {"kind": "avgpool", "k": 3, "s": 2}, {"kind": "flatten"}, {"kind": "dense", "units": 32, "label": "Dense1"},
        {"kind": "square"}, {"kind": "dense", "units": 10, "label": "Dense2"}]}""",
    "ce": """{"name": "ce", "input": [3, 32, 32], "n_slots": 16384, "layers": [
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 18, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool1"},
        {"kind": "subconv", "k": 3, "s": 1, "out_channels": 15, "groups": 3, "label": "Conv2"},
        {"kind": "conv", "k": 1, "s": 1, "out_channels": 64, "policy": "convpack", "label": "Conv3"},
        {"kind": "square"}, {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool2"},
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 64}, {"kind": "flatten"},
        {"kind": "dense", "units": 256, "label": "Dense1"}, {"kind": "square"},
        {"kind": "dense", "units": 10, "label": "Dense2"}]}""",
    "ce-mini": """{"name": "ce-mini", "input": [3, 16, 16], "n_slots": 2048, "layers": [
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 6, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool1"},
        {"kind": "subconv", "k": 3, "s": 1, "out_channels": 6, "groups": 3, "label": "Conv2"},
        {"kind": "conv", "k": 1, "s": 1, "out_channels": 8, "policy": "convpack", "label": "Conv3"},
        {"kind": "square"}, {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool2"},
        {"kind": "conv", "k": 2, "s": 1, "out_channels": 12}, {"kind": "flatten"},
        {"kind": "dense", "units": 16, "label": "Dense1"}, {"kind": "square"},
        {"kind": "dense", "units": 10, "label": "Dense2"}]}""",
}


def _conv_fp64(x, W, b, s):
    c_out, c_in, k, _ = W.shape
    d = (x.shape[1] - k) // s + 1
    out = np.empty((c_out, d, d))
    o = np.arange(d) * s
    for co in range(c_out):
        acc = np.full((d, d), float(b[co]))
        for ci in range(c_in):
            for ky in range(k):
                for kx in range(k):
                    acc += W[co, ci, ky, kx] * x[ci][np.ix_(o + ky, o + kx)]
        out[co] = acc
    return out


def model_forward(layers, in_c, in_d, flat_weights, image):
    """the cleartext forward pass of a model's layer list (conv / subconv /
    avgpool / square / flatten / dense; the float32-stream weight order of
    proj/src/modelio.cpp:169-202) in FP64 -- the sanity check on decrypted
    logits of bench_configs.py --model (the reference-order oracle lives under
    oracle/ and is for tests); layers as paper_2110_08321_b200.hegpu.Model.layers"""
    w = np.asarray(flat_weights, dtype=np.float64)
    t = np.asarray(image, dtype=np.float64).reshape(in_c, in_d, in_d)
    o = 0
    for l in layers:
        kind = l["kind"]
        if kind in ("conv", "subconv"):
            g = max(1, l.get("groups") or 1) if kind == "subconv" else 1
            ci, co, k = t.shape[0] // g, l["out"] // g, l["k"]
            parts = []
            for i in range(g):
                n = co * ci * k * k
                parts.append(_conv_fp64(t[i * ci:(i + 1) * ci], w[o:o + n].reshape(co, ci, k, k), w[o + n:o + n + co],
                                        l.get("s") or 1))
                o += n + co
            t = np.concatenate(parts)
        elif kind == "avgpool":
            k, s = l["k"], l.get("s") or 1
            d = (t.shape[1] - k) // s + 1
            idx = np.arange(d) * s
            t = sum(t[:, idx + ky][:, :, idx + kx] for ky in range(k) for kx in range(k)) / (k * k)
        elif kind == "square":
            t = t * t
        elif kind == "flatten":
            t = t.reshape(-1)
        elif kind == "dense":
            x = t.reshape(-1)
            n = l["out"] * x.size
            t = w[o:o + n].reshape(l["out"], x.size) @ x + w[o + n:o + n + l["out"]]
            o += n + l["out"]
    assert o == w.size
    return np.asarray(t).reshape(-1)
