"""oracle/hesim_oracle.py -- TEST INFRASTRUCTURE ONLY.

numpy restatement of the reference `hesim` slot simulator for the hot path
(the cleartext/slot-level oracle).  Every function cites the reference
file:line it follows; tests/test_oracle_hesim.py pins it against the
reference's own known-answer tests (proj/tests/*.cpp).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.

Parity status: pinned (slot values, HOP counts, stage labels) against the
reference's golden expectations; the reference itself cannot be built here
(Eigen3 + vendor/ absent).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

CIPHERTEXT, PLAINTEXT = "ct", "pt"


class CapacityError(RuntimeError):
    """proj/include/hesim/errors.hpp:9-12"""


class ShapeError(RuntimeError):
    """proj/include/hesim/errors.hpp:14-17"""


# ----------------------------------------------------------------- meter ---
@dataclass
class OpTally:
    """proj/include/hesim/meter.hpp:12-31"""
    add_pc: int = 0
    add_cc: int = 0
    mul_pc: int = 0
    mul_cc: int = 0
    rot: int = 0

    def total(self):
        return self.add_pc + self.add_cc + self.mul_pc + self.mul_cc + self.rot

    def as_tuple(self):
        return (self.add_pc, self.add_cc, self.mul_pc, self.mul_cc, self.rot)


@dataclass
class MeterContext:
    """proj/include/hesim/meter.hpp:36-70 (begin_stage re-enters rows)."""
    tally: OpTally = field(default_factory=OpTally)
    stages: list = field(default_factory=list)
    _cur: int = -1

    def begin_stage(self, label):
        for i, (name, _) in enumerate(self.stages):
            if name == label:
                self._cur = i
                return
        self.stages.append((label, OpTally()))
        self._cur = len(self.stages) - 1

    def bump(self, f):
        setattr(self.tally, f, getattr(self.tally, f) + 1)
        if self._cur >= 0:
            t = self.stages[self._cur][1]
            setattr(t, f, getattr(t, f) + 1)


# --------------------------------------------------------------- slotvec ---
def is_power_of_two(x):
    return x > 0 and (x & (x - 1)) == 0


class SlotVector:
    """proj/include/hesim/slotvec.hpp:14-33; ctor proj/src/slotvec.cpp:12-18"""

    def __init__(self, slots, kind):
        slots = np.asarray(slots, dtype=np.float64)
        if not is_power_of_two(slots.size):
            raise ShapeError(f"slot count must be a power of two, got {slots.size}")
        self.slots = slots
        self.kind = kind

    @property
    def n_slots(self):
        return self.slots.size

    def __getitem__(self, i):
        return self.slots[i]

    def is_zero(self):
        return not np.any(self.slots)

    def masked_prefix(self, keep):  # proj/src/slotvec.cpp:20-24
        out = self.slots.copy()
        out[keep:] = 0.0
        return SlotVector(out, self.kind)


def pack(values, n_slots, kind):
    """proj/src/slotvec.cpp:26-36"""
    values = np.asarray(values, dtype=np.float64).ravel()
    if values.size > n_slots:
        raise CapacityError(f"pack: {values.size} values exceed {n_slots} slots")
    s = np.zeros(n_slots)
    s[: values.size] = values
    return SlotVector(s, kind)


def zeros(n_slots, kind):
    """proj/src/slotvec.cpp:38-40"""
    return SlotVector(np.zeros(n_slots), kind)


def rotate_right(v, r, ctx):
    """proj/src/slotvec.cpp:42-57: out[j] = v[(j - r) mod N]; r=0 free;
    only ciphertext rotations are metered."""
    n = v.n_slots
    if r < 0 or r >= n:
        raise IndexError(f"rotate: amount {r} outside [0, {n})")
    if r == 0:
        return v
    if v.kind == CIPHERTEXT:
        ctx.bump("rot")
    return SlotVector(np.roll(v.slots, r), v.kind)


def rotate_left(v, r, ctx):
    """proj/src/slotvec.cpp:59-66"""
    n = v.n_slots
    if r < 0 or r >= n:
        raise IndexError(f"rotate: amount {r} outside [0, {n})")
    return rotate_right(v, 0 if r == 0 else n - r, ctx)


def _meter_binary(a, b, ctx, cc, pc):
    """proj/src/slotvec.cpp:76-86"""
    n_ct = (a.kind == CIPHERTEXT) + (b.kind == CIPHERTEXT)
    if n_ct == 2:
        ctx.bump(cc)
    elif n_ct == 1:
        ctx.bump(pc)


def _result_kind(a, b):
    return CIPHERTEXT if CIPHERTEXT in (a.kind, b.kind) else PLAINTEXT


def _check_shapes(a, b):  # proj/src/slotvec.cpp:88-93
    if a.n_slots != b.n_slots:
        raise ShapeError(f"slot count mismatch: {a.n_slots} vs {b.n_slots}")


def add(a, b, ctx):
    """proj/src/slotvec.cpp:97-102"""
    _check_shapes(a, b)
    _meter_binary(a, b, ctx, "add_cc", "add_pc")
    return SlotVector(a.slots + b.slots, _result_kind(a, b))


def mul(a, b, ctx):
    """proj/src/slotvec.cpp:104-109"""
    _check_shapes(a, b)
    _meter_binary(a, b, ctx, "mul_cc", "mul_pc")
    return SlotVector(a.slots * b.slots, _result_kind(a, b))


# ---------------------------------------------------------------- matvec ---
def next_power_of_two(x):
    """proj/src/matvec.cpp:10-14"""
    p = 1
    while p < x:
        p <<= 1
    return p


def _ceil_div(a, b):
    return (a + b - 1) // b


def _ceil_log2(x):
    b = 0
    while (1 << b) < x:
        b += 1
    return b


def plain_branch_fits(m, n, n_slots):
    """proj/src/matvec.cpp:29-33"""
    if n_slots < m + n - 1:
        return False
    b = _ceil_log2(_ceil_div(m + n - 1, m))
    return (m << b) <= n_slots


def _check_dims(m, n, n_slots):  # proj/src/matvec.cpp:35-41
    if m > n_slots or n > n_slots:
        raise CapacityError(f"matrix {m}x{n} exceeds {n_slots} slots")


def extract_diagonals(A, n_slots):
    """proj/src/matvec.cpp:45-65 -> (m_eff, masks[m_eff][n_slots])"""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    _check_dims(m, n, n_slots)
    m_eff = m if plain_branch_fits(m, n, n_slots) else next_power_of_two(m)
    if m_eff > n_slots:
        raise CapacityError(f"padded row count {m_eff} exceeds {n_slots} slots")
    masks = np.zeros((m_eff, n_slots))
    j = np.arange(n)
    for i in range(m_eff):
        row = (i + j) % m_eff
        ok = row < m
        masks[i, j[ok]] = A[row[ok], j[ok]]
    return m_eff, masks


def hs_folds(m, n, n_slots, m_eff):
    """fold count of proj/src/matvec.cpp:88-91"""
    padded = m_eff != m or not plain_branch_fits(m, n, n_slots)
    return _ceil_log2(n_slots // m_eff) if padded else _ceil_log2(_ceil_div(m + n - 1, m))


def rotate_and_sum(v, span, block, ctx):
    """proj/src/matvec.cpp:67-80"""
    if block < 1 or block > v.n_slots:
        raise IndexError("rotate_and_sum: block out of range")
    folds = _ceil_log2(_ceil_div(span, block))
    s = v
    for t in range(folds - 1, -1, -1):
        s = add(s, rotate_left(s, block << t, ctx), ctx)
    return s


def hs_matvec(A, v, ctx, skip_zero_diagonals=True):
    """proj/src/matvec.cpp:82-105"""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    N = v.n_slots
    _check_dims(m, n, N)
    m_eff, masks = extract_diagonals(A, N)
    folds = hs_folds(m, n, N, m_eff)
    s = zeros(N, CIPHERTEXT)
    first = True
    for i in range(m_eff):
        if skip_zero_diagonals and not np.any(masks[i]):
            continue
        t = rotate_right(mul(SlotVector(masks[i], PLAINTEXT), v, ctx), i, ctx)
        s = t if first else add(s, t, ctx)
        first = False
    for t in range(folds - 1, -1, -1):
        s = add(s, rotate_left(s, m_eff << t, ctx), ctx)
    return s


def lola_dense_matvec(A, v, ctx):
    """proj/src/matvec.cpp:107-123: one ciphertext per row i, slot 0 = A[i] . x
    (product with the packed row, rotate-and-sum over next_pow2(n) slots,
    the fold residue cleared at the value level)"""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    N = v.n_slots
    _check_dims(m, n, N)
    delta = next_power_of_two(n)
    out = []
    for i in range(m):
        row = pack(A[i], N, PLAINTEXT)
        p = rotate_and_sum(mul(row, v, ctx), delta, 1, ctx)
        out.append(p.masked_prefix(1))
    return out


def lola_stacked_matvec(A, v, ctx):
    """proj/src/matvec.cpp:125-166: k = N / next_pow2(n) rows per batch; the
    input is re-stacked k times per batch (k-1 rotations + additions), one
    product, rotate-and-sum, segment starts kept (free), batches combined by
    right rotations by the batch index.  Returns (ct, slot_of_row)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    N = v.n_slots
    _check_dims(m, n, N)
    delta = next_power_of_two(n)
    if delta > N:
        raise CapacityError(f"stacked: padded width {delta} exceeds {N} slots")
    k = N // delta
    batches = _ceil_div(m, k)
    vd = v.masked_prefix(n)
    res = zeros(N, CIPHERTEXT)
    slot_of_row = [0] * m
    for b in range(batches):
        stacked = vd
        for j in range(1, k):
            stacked = add(stacked, rotate_right(vd, j * delta, ctx), ctx)
        rows_pt = np.zeros(N)
        for j in range(k):
            if b * k + j < m:
                rows_pt[j * delta: j * delta + n] = A[b * k + j]
        p = mul(SlotVector(rows_pt, PLAINTEXT), stacked, ctx)
        p = rotate_and_sum(p, delta, 1, ctx)
        clean = np.zeros(N)
        for j in range(k):
            if b * k + j < m:
                clean[j * delta] = p[j * delta]
                slot_of_row[b * k + j] = j * delta + b
        batch = SlotVector(clean, CIPHERTEXT)
        res = batch if b == 0 else add(res, rotate_right(batch, b, ctx), ctx)
    return res, slot_of_row


def predict_lola_dense(m, n):
    """proj/src/matvec.cpp:189-195 -> (rotations, multiplications, additions)"""
    lg = _ceil_log2(n)
    return m * lg, m, m * lg


def predict_lola_stacked(m, n, n_slots):
    """proj/src/matvec.cpp:197-211 -> (rotations, multiplications, additions)"""
    delta = next_power_of_two(n)
    if delta > n_slots:
        raise CapacityError("stacked: padded width exceeds slot count")
    k = n_slots // delta
    batches = _ceil_div(m, k)
    r = batches * (k + _ceil_log2(n) - 1) + batches - 1
    return r, batches, r


def predict_hs(m, n, n_slots):
    """proj/src/matvec.cpp:168-187 -> (rotations, multiplications, additions)"""
    _check_dims(m, n, n_slots)
    if plain_branch_fits(m, n, n_slots):
        folds = _ceil_log2(_ceil_div(m + n - 1, m))
        return (m - 1 + folds, m, m - 1 + folds)
    mp = next_power_of_two(m)
    if mp > n_slots:
        raise CapacityError("padded row count exceeds slot count")
    folds = _ceil_log2(n_slots // mp)
    return (mp - 1 + folds, mp, mp - 1 + folds)


# -------------------------------------------------------------- convlower ---
@dataclass
class ConvShape:
    """proj/include/hesim/convlower.hpp:13-17"""
    d_in: int
    c_in: int
    kernel_k: int
    stride: int
    c_out: int

    def d_out(self):
        return (self.d_in - self.kernel_k) // self.stride + 1


def conv_pack(image, shape, n_slots):
    """proj/src/convlower.cpp:9-37; image [c][h][w]; tap t=(ci*k+ky)*k+kx"""
    image = np.asarray(image, dtype=np.float64)
    d_out = shape.d_out()
    if d_out * d_out > n_slots:
        raise CapacityError("conv_pack: output positions exceed slots")
    if image.shape[0] != shape.c_in or image.shape[1] != shape.d_in:
        raise ShapeError("conv_pack: image does not match shape")
    k, s = shape.kernel_k, shape.stride
    taps = []
    o = np.arange(d_out) * s
    for ci in range(shape.c_in):
        for ky in range(k):
            for kx in range(k):
                v = np.zeros(n_slots)
                v[: d_out * d_out] = image[ci][np.ix_(o + ky, o + kx)].ravel()
                taps.append(SlotVector(v, CIPHERTEXT))
    return taps


def conv_packed_forward(taps, weights, bias, shape, ctx):
    """proj/src/convlower.cpp:39-74; weights [c_out][c_in][k][k]"""
    k = shape.kernel_k
    n_taps = k * k * shape.c_in
    weights = np.asarray(weights, dtype=np.float64)
    if len(taps) != n_taps or weights.shape != (shape.c_out, shape.c_in, k, k):
        raise ShapeError("conv_packed_forward: filter/tap shape mismatch")
    N = taps[0].n_slots
    w = shape.d_out() ** 2
    maps = []
    for co in range(shape.c_out):
        acc = None
        for t in range(n_taps):
            ci, ky, kx = t // (k * k), (t // k) % k, t % k
            pt = np.zeros(N)
            pt[:w] = weights[co, ci, ky, kx]
            prod = mul(SlotVector(pt, PLAINTEXT), taps[t], ctx)
            acc = prod if t == 0 else add(acc, prod, ctx)
        bpt = np.zeros(N)
        bpt[:w] = bias[co] if bias is not None and len(bias) else 0.0
        maps.append(add(acc, SlotVector(bpt, PLAINTEXT), ctx))
    return maps


def conv_to_matrix(shape, weights):
    """proj/src/convlower.cpp:76-102 (dense form)"""
    weights = np.asarray(weights, dtype=np.float64)
    d_out, d_in, k, s = shape.d_out(), shape.d_in, shape.kernel_k, shape.stride
    A = np.zeros((d_out * d_out * shape.c_out, d_in * d_in * shape.c_in))
    for co in range(shape.c_out):
        for oy in range(d_out):
            for ox in range(d_out):
                r = (co * d_out + oy) * d_out + ox
                for ci in range(shape.c_in):
                    for ky in range(k):
                        for kx in range(k):
                            col = (ci * d_in + oy * s + ky) * d_in + ox * s + kx
                            A[r, col] += weights[co, ci, ky, kx]
    return A


def conv_bias_vector(shape, bias):
    """proj/src/convlower.cpp:104-113"""
    w = shape.d_out() ** 2
    return np.repeat(np.asarray(bias, dtype=np.float64), w)


def pool_to_matrix(c, d_in, k, stride):
    """proj/src/convlower.cpp:115-139 (dense form)"""
    d_out = (d_in - k) // stride + 1
    A = np.zeros((d_out * d_out * c, d_in * d_in * c))
    for ci in range(c):
        for oy in range(d_out):
            for ox in range(d_out):
                r = (ci * d_out + oy) * d_out + ox
                for ky in range(k):
                    for kx in range(k):
                        A[r, (ci * d_in + oy * stride + ky) * d_in + ox * stride + kx] += 1.0 / (k * k)
    return A


def square_layer(v, ctx):
    """proj/src/convlower.cpp:141-143"""
    return mul(v, v, ctx)


def merge_maps(maps, w, ctx):
    """proj/src/convlower.cpp:145-160"""
    if not maps:
        raise ShapeError("merge_maps: no maps")
    N = maps[0].n_slots
    c = len(maps)
    if c * w > N:
        raise CapacityError(f"merge_maps: {c} maps of {w} slots exceed {N} slots")
    out = maps[0]
    for j in range(1, c):
        out = add(out, rotate_right(maps[j], j * w, ctx), ctx)
    return out


# -------------------------------------------------------------- refmodel ---
def ref_conv(x, weights, bias, stride):
    """proj/src/refmodel.cpp:21-46 (same accumulation order)"""
    x = np.asarray(x, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    c_out, c_in, k, _ = weights.shape
    if x.shape[0] != c_in:
        raise ShapeError("conv: channel mismatch")
    if k > x.shape[1]:
        raise ShapeError("window larger than input")
    d_out = (x.shape[1] - k) // stride + 1
    out = np.zeros((c_out, d_out, d_out))
    for co in range(c_out):
        for oy in range(d_out):
            for ox in range(d_out):
                acc = bias[co] if bias is not None and len(bias) else 0.0
                for ci in range(c_in):
                    for ky in range(k):
                        for kx in range(k):
                            acc += weights[co, ci, ky, kx] * x[ci, oy * stride + ky, ox * stride + kx]
                out[co, oy, ox] = acc
    return out


def ref_avgpool(x, k, stride):
    """proj/src/refmodel.cpp:48-66"""
    x = np.asarray(x, dtype=np.float64)
    c, d = x.shape[0], x.shape[1]
    if k > d:
        raise ShapeError("window larger than input")
    d_out = (d - k) // stride + 1
    out = np.zeros((c, d_out, d_out))
    for oy in range(d_out):
        for ox in range(d_out):
            out[:, oy, ox] = x[:, oy * stride:oy * stride + k, ox * stride:ox * stride + k].sum(axis=(1, 2)) * (
                1.0 / (k * k))
    return out


def ref_square(x):
    """proj/src/refmodel.cpp:68-72"""
    return np.asarray(x) * np.asarray(x)


def ref_dense(v, W, b):
    """proj/src/refmodel.cpp:74-80"""
    W = np.asarray(W, dtype=np.float64)
    if W.shape[1] != len(v) or W.shape[0] != len(b):
        raise ShapeError("dense: dimension mismatch")
    return W @ v + b


# -------------------------------------------------- the CNN (stage driver) ---
@dataclass
class CnnSpec:
    """The hot-path model family: Conv(k, s, c_out) -> Square -> Dense(m1) ->
    Square -> Dense(m2) (BASELINE configs 0/2/3; the cryptonets-style L' net
    after fusion, proj/src/netcompile.cpp:106-213)."""
    in_c: int
    in_d: int
    k: int
    s: int
    c_out: int
    dense: tuple
    n_slots: int

    def shape(self):
        return ConvShape(self.in_d, self.in_c, self.k, self.s, self.c_out)

    def stage_labels(self):
        """lower() output for this layer list (netcompile.cpp:106-213)."""
        labels = ["Conv1", "Flat1"]
        for i, _ in enumerate(self.dense):
            labels.append(f"Square{i + 1}")
            labels.append(f"Dense{i + 1}")
        return labels


def execute(spec, weights, image, ctx):
    """proj/src/netcompile.cpp:291-446 restricted to ConvPack / Merge /
    Square / Linear(HS) stages.  weights = dict(conv_w, conv_b, dense=[(W,b)])
    Returns the logits (first m_last slots of the output ciphertext)."""
    shape = spec.shape()
    N = spec.n_slots
    ctx.begin_stage("Conv1")
    taps = conv_pack(image, shape, N)
    maps = conv_packed_forward(taps, weights["conv_w"], weights["conv_b"], shape, ctx)
    ctx.begin_stage("Flat1")
    ct = merge_maps(maps, shape.d_out() ** 2, ctx)
    for i, (W, b) in enumerate(weights["dense"]):
        ctx.begin_stage(f"Square{i + 1}")
        ct = square_layer(ct, ctx)
        ctx.begin_stage(f"Dense{i + 1}")
        out = hs_matvec(W, ct, ctx)
        out = add(out, pack(b, N, PLAINTEXT), ctx)
        ct = out.masked_prefix(np.asarray(W).shape[0])
    return ct.slots[: np.asarray(weights["dense"][-1][0]).shape[0]].copy()


def ref_forward(spec, weights, image):
    """proj/src/netcompile.cpp:448-503 for the same layer list."""
    t = ref_conv(image, weights["conv_w"], weights["conv_b"], spec.s)
    flat = None
    for i, (W, b) in enumerate(weights["dense"]):
        if flat is None:
            t = ref_square(t)
            flat = t.ravel()
        else:
            flat = ref_square(flat)
        flat = ref_dense(flat, W, b)
    return flat


# ------------------------------------------ model files (layer lists) ---
def split_weights(layers, in_c, in_d, flat):
    """the float32 weights stream of proj/src/modelio.cpp:169-202 -> per-layer
    (W, b); layers: dicts with kind, k, s, out"""
    out, o, c, d = [], 0, in_c, in_d
    for l in layers:
        if l["kind"] == "conv":
            n = l["out"] * c * l["k"] ** 2
            out.append((flat[o:o + n].reshape(l["out"], c, l["k"], l["k"]), flat[o + n:o + n + l["out"]]))
            o += n + l["out"]
            c, d = l["out"], (d - l["k"]) // l["s"] + 1
        elif l["kind"] == "dense":
            n = l["out"] * c * d * d
            out.append((flat[o:o + n].reshape(l["out"], c * d * d), flat[o + n:o + n + l["out"]]))
            o += n + l["out"]
            c, d = l["out"], 1
        else:
            out.append(None)
            if l["kind"] == "avgpool":
                d = (d - l["k"]) // l["s"] + 1
    assert o == len(flat)
    return out


def compose_run(layers, weights, c, d):
    """proj/src/netcompile.cpp:225-278 (dense): the affine map (M, b) of one
    linear run of conv / avgpool / flatten / dense layers on a (c, d, d) input"""
    M, b = None, None

    def fold(A, bias):
        nonlocal M, b
        if M is None:
            M, b = A, bias
        else:
            M, b = A @ M, A @ b + bias

    for l, w in zip(layers, weights):
        if l["kind"] == "conv":
            shape = ConvShape(d, c, l["k"], l["s"], l["out"])
            fold(conv_to_matrix(shape, w[0]), conv_bias_vector(shape, w[1]))
            c, d = l["out"], shape.d_out()
        elif l["kind"] == "avgpool":
            d_out = (d - l["k"]) // l["s"] + 1
            fold(pool_to_matrix(c, d, l["k"], l["s"]), np.zeros(c * d_out * d_out))
            d = d_out
        elif l["kind"] == "dense":
            fold(np.asarray(w[0], dtype=np.float64), np.asarray(w[1], dtype=np.float64))
            c, d = l["out"], 1
    return M, b


def ref_forward_layers(layers, weights, image):
    """proj/src/netcompile.cpp:448-503 over a general layer list"""
    t = np.asarray(image, dtype=np.float64)
    for l, w in zip(layers, weights):
        if l["kind"] == "conv":
            t = ref_conv(t, w[0], w[1], l["s"])
        elif l["kind"] == "avgpool":
            t = ref_avgpool(t, l["k"], l["s"])
        elif l["kind"] == "square":
            t = ref_square(t)
        elif l["kind"] == "flatten":
            t = t.ravel()
        elif l["kind"] == "dense":
            t = ref_dense(np.ravel(t), w[0], w[1])
    return np.ravel(t)


def golden_stage_tallies(spec):
    """Closed-form per-stage HOPs (add_pc, add_cc, mul_pc, mul_cc, rot) for
    dense weights with no zero diagonals."""
    shape = spec.shape()
    taps = shape.kernel_k ** 2 * shape.c_in
    rows = {"Conv1": (shape.c_out, (taps - 1) * shape.c_out, taps * shape.c_out, 0, 0),
            "Flat1": (0, shape.c_out - 1, 0, 0, shape.c_out - 1)}
    n = shape.c_out * shape.d_out() ** 2
    for i, m in enumerate(spec.dense):
        rows[f"Square{i + 1}"] = (0, 0, 0, 1, 0)
        rot, mul_, add_ = predict_hs(m, n, spec.n_slots)
        rows[f"Dense{i + 1}"] = (1, add_, mul_, 0, rot)
        n = m
    return rows


# ------------------------------------- general lower() / execute() ---------
# The full stage driver of the reference (SubConv groups, grouped merges,
# the stand-alone ConvPack repack and the LoLa policies), restated from
# proj/src/netcompile.cpp:14-446.  Layers are dicts {kind, k, s, out, groups,
# policy, label} (kind in conv / subconv / avgpool / square / flatten /
# dense; policy None or convpack / hs / lola-dense / lola-stacked).
_LINEAR = ("conv", "subconv", "avgpool", "flatten", "dense")


def _lget(l, key, default):
    v = l.get(key, default)
    return default if v is None else v


def _is_standalone_convpack(l):  # netcompile.cpp:21-24
    return l["kind"] == "conv" and l.get("policy") == "convpack"


def _apply_layer(shape, l, where):
    """netcompile.cpp:34-69; shape = (c, d, flat, flat_len)"""
    c, d, flat, flat_len = shape
    kind = l["kind"]
    if kind in ("conv", "subconv"):
        if flat:
            raise ShapeError(where + ": convolution after flatten")
        g = _lget(l, "groups", 1)
        if kind == "subconv" and (c % g or l["out"] % g):
            raise ShapeError(f"{where}: channels not divisible into {g} groups")
        return (l["out"], (d - l["k"]) // _lget(l, "s", 1) + 1, flat, flat_len)
    if kind == "avgpool":
        if flat:
            raise ShapeError(where + ": pooling after flatten")
        return (c, (d - l["k"]) // _lget(l, "s", 1) + 1, flat, flat_len)
    if kind == "flatten":
        return (c, d, True, _shape_size(shape))
    if kind == "dense":
        return (c, d, True, l["out"])
    return shape


def _shape_size(shape):
    c, d, flat, flat_len = shape
    return flat_len if flat else c * d * d


def _lookahead_groups(layers, frm):  # netcompile.cpp:71-91
    for j in range(frm, len(layers)):
        l = layers[j]
        if l["kind"] == "square":
            continue
        if _is_standalone_convpack(l):
            return 1
        if l["kind"] == "subconv":
            return _lget(l, "groups", 1)
        if l["kind"] in _LINEAR:
            r = j
            while r < len(layers) and layers[r]["kind"] in _LINEAR and not _is_standalone_convpack(layers[r]):
                if layers[r]["kind"] == "subconv":
                    return _lget(layers[r], "groups", 1)
                r += 1
            return 1
    return 1


def lower(model):
    """proj/src/netcompile.cpp:106-213.  model = dict(name, in_c, in_d,
    n_slots, layers, default_policy='hs').  Returns the stage list: dicts
    {kind (convpack / merge / square / repackconv / linear), label,
    layer_idx, groups, policy}."""
    layers = model["layers"]
    N = model["n_slots"]
    if not layers:
        raise ShapeError("model has no layers")
    if not is_power_of_two(N):
        raise ShapeError("n_slots must be a power of two")
    stages = []
    shape = (model["in_c"], model["in_d"], False, 0)
    idx, flat_n, square_n, linear_n, maps_layout = 0, 0, 0, 0, False
    l0 = layers[0]
    if l0["kind"] == "conv" and l0.get("policy") in (None, "convpack"):
        label = l0.get("label") or "Conv1"
        nxt = _apply_layer(shape, l0, label)
        if nxt[1] * nxt[1] > N:
            raise CapacityError(f"{label}: d_out^2 = {nxt[1] * nxt[1]} > n_slots = {N}")
        stages.append(dict(kind="convpack", label=label, layer_idx=[0], groups=1, policy="hs"))
        shape, maps_layout, idx = nxt, True, 1
    while idx < len(layers):
        l = layers[idx]
        if l["kind"] == "square":
            if maps_layout:
                flat_n += 1
                g = _lookahead_groups(layers, idx + 1)
                label = f"Flat{flat_n}"
                if shape[0] % g:
                    raise ShapeError(f"{label}: {shape[0]} maps not divisible into {g} groups")
                if (shape[0] // g) * shape[1] * shape[1] > N:
                    raise CapacityError(f"{label}: group footprint {(shape[0] // g) * shape[1] ** 2} > n_slots = {N}")
                stages.append(dict(kind="merge", label=label, layer_idx=[], groups=g, policy="hs"))
                maps_layout = False
            square_n += 1
            stages.append(dict(kind="square", label=f"Square{square_n}", layer_idx=[idx], groups=1, policy="hs"))
            idx += 1
            continue
        if l["kind"] not in _LINEAR:
            raise ShapeError(f"unsupported layer kind at index {idx}")
        if _is_standalone_convpack(l):
            label = l.get("label") or f"Conv{idx}"
            stages.append(dict(kind="repackconv", label=label, layer_idx=[idx], groups=1, policy="hs"))
            shape = _apply_layer(shape, l, label)
            maps_layout = True
            idx += 1
            continue
        st = dict(kind="linear", label="", layer_idx=[], groups=1, policy=model.get("default_policy", "hs"))
        j = idx
        while j < len(layers) and layers[j]["kind"] in _LINEAR and not _is_standalone_convpack(layers[j]):
            st["layer_idx"].append(j)
            if layers[j]["kind"] == "subconv":
                st["groups"] = _lget(layers[j], "groups", 1)
            if layers[j].get("policy"):
                st["policy"] = layers[j]["policy"]
            j += 1
        linear_n += 1
        st["label"] = "-".join(layers[r]["label"] for r in st["layer_idx"] if layers[r].get("label")) \
            or f"Linear{linear_n}"
        if st["groups"] > 1 and st["policy"] != "hs":
            raise ShapeError(st["label"] + ": grouped stages require the HS kernel")
        if maps_layout:
            flat_n += 1
            stages.append(dict(kind="merge", label=f"Flat{flat_n}", layer_idx=[], groups=st["groups"], policy="hs"))
            maps_layout = False
        run_shape = shape
        for r in st["layer_idx"]:
            run_shape = _apply_layer(run_shape, layers[r], st["label"])
        m, n = _shape_size(run_shape), _shape_size(shape)
        if m > N or n > N:
            raise CapacityError(f"{st['label']}: fused {m}x{n} exceeds n_slots = {N}")
        stages.append(st)
        shape, idx = run_shape, j
    return stages


def split_model_weights(model, flat):
    """the float32 weights stream (proj/src/modelio.cpp:169-202) -> per layer
    (W [out][c][k][k], b) for conv, [(W, b)] * groups for subconv, (W [m][n],
    b) for dense, None otherwise"""
    flat = np.asarray(flat, dtype=np.float64)
    out, o = [], 0
    shape = (model["in_c"], model["in_d"], False, 0)
    for l in model["layers"]:
        c, d = shape[0], shape[1]
        if l["kind"] == "conv":
            n = l["out"] * c * l["k"] ** 2
            out.append((flat[o:o + n].reshape(l["out"], c, l["k"], l["k"]), flat[o + n:o + n + l["out"]]))
            o += n + l["out"]
        elif l["kind"] == "subconv":
            g = _lget(l, "groups", 1)
            po, pi = l["out"] // g, c // g
            banks = []
            for _ in range(g):
                n = po * pi * l["k"] ** 2
                banks.append((flat[o:o + n].reshape(po, pi, l["k"], l["k"]), flat[o + n:o + n + po]))
                o += n + po
            out.append(banks)
        elif l["kind"] == "dense":
            n_in = _shape_size(shape)
            n = l["out"] * n_in
            out.append((flat[o:o + n].reshape(l["out"], n_in), flat[o + n:o + n + l["out"]]))
            o += n + l["out"]
        else:
            out.append(None)
        shape = _apply_layer(shape, l, "shape inference")
    if o != len(flat):
        raise ShapeError(f"weights: the model needs {o} values, got {len(flat)}")
    return out


def model_weight_count(model):
    shape, o = (model["in_c"], model["in_d"], False, 0), 0
    for l in model["layers"]:
        c = shape[0]
        if l["kind"] == "conv":
            o += l["out"] * c * l["k"] ** 2 + l["out"]
        elif l["kind"] == "subconv":
            g = _lget(l, "groups", 1)
            o += g * ((l["out"] // g) * (c // g) * l["k"] ** 2 + l["out"] // g)
        elif l["kind"] == "dense":
            o += l["out"] * _shape_size(shape) + l["out"]
        shape = _apply_layer(shape, l, "shape inference")
    return o


def compose_group(model, weights, idxs, group, n_groups, shape):
    """compose_run (proj/src/netcompile.cpp:225-278): the affine map (M, b)
    of one linear run restricted to channel group `group` of `n_groups`"""
    c, d = shape[0] // n_groups, shape[1]
    M, b = None, None

    def fold(A, bias):
        nonlocal M, b
        if M is None:
            M, b = A, np.asarray(bias, dtype=np.float64)
        else:
            M, b = A @ M, A @ b + bias

    for i in idxs:
        l, w = model["layers"][i], weights[i]
        if l["kind"] in ("conv", "subconv"):
            W, bias = w[group] if l["kind"] == "subconv" else w
            cs = ConvShape(d, c, l["k"], _lget(l, "s", 1), np.asarray(W).shape[0])
            fold(conv_to_matrix(cs, W), conv_bias_vector(cs, bias))
            c, d = cs.c_out, cs.d_out()
        elif l["kind"] == "avgpool":
            s = _lget(l, "s", 1)
            d_out = (d - l["k"]) // s + 1
            fold(pool_to_matrix(c, d, l["k"], s), np.zeros(c * d_out * d_out))
            d = d_out
        elif l["kind"] == "dense":
            fold(np.asarray(w[0], dtype=np.float64), np.asarray(w[1], dtype=np.float64))
        elif l["kind"] != "flatten":
            raise ShapeError("non-linear layer inside a fused run")
    if M is None:
        raise ShapeError("empty linear run")
    return M, b


def execute_program(model, weights, image, ctx, stages=None):
    """proj/src/netcompile.cpp:291-446.  weights as split_model_weights
    returns them.  Returns the logits."""
    stages = lower(model) if stages is None else stages
    layers, N = model["layers"], model["n_slots"]
    image = np.asarray(image, dtype=np.float64)
    shape = (model["in_c"], model["in_d"], False, 0)
    cts, maps, seeded = [], False, False
    for st in stages:
        ctx.begin_stage(st["label"])
        if not seeded and st["kind"] != "convpack":
            if _shape_size(shape) > N:
                raise CapacityError(f"input of {_shape_size(shape)} values exceeds n_slots")
            cts, seeded = [pack(image.ravel(), N, CIPHERTEXT)], True
        kind = st["kind"]
        if kind == "convpack":
            l = layers[st["layer_idx"][0]]
            cs = ConvShape(shape[1], shape[0], l["k"], _lget(l, "s", 1), l["out"])
            W, b = weights[st["layer_idx"][0]]
            cts = conv_packed_forward(conv_pack(image, cs, N), W, b, cs, ctx)
            maps, seeded = True, True
            shape = _apply_layer(shape, l, st["label"])
        elif kind == "merge":
            G = st["groups"]
            per, w = shape[0] // G, shape[1] * shape[1]
            cts = [merge_maps(cts[g * per:(g + 1) * per], w, ctx) for g in range(G)]
            maps = False
        elif kind == "square":
            cts = [square_layer(ct, ctx) for ct in cts]
        elif kind == "repackconv":
            l = layers[st["layer_idx"][0]]
            if l["k"] != 1:
                raise ShapeError(st["label"] + ": only 1x1 convolutions support the packed rotation lowering")
            w = shape[1] * shape[1]
            if maps:
                taps = cts
            else:
                G = len(cts)
                per = shape[0] // G
                taps = [rotate_left(cts[g], j * w, ctx) for g in range(G) for j in range(per)]
            cs = ConvShape(shape[1], shape[0], 1, 1, l["out"])
            W, b = weights[st["layer_idx"][0]]
            cts = conv_packed_forward(taps, W, b, cs, ctx)
            maps = True
            shape = _apply_layer(shape, l, st["label"])
        else:  # linear
            G = st["groups"]
            if len(cts) != G:
                raise ShapeError(f"{st['label']}: expected {G} input ciphertexts, have {len(cts)}")
            outs = []
            for g in range(G):
                M, bias = compose_group(model, weights, st["layer_idx"], g, G, shape)
                if st["policy"] == "hs":
                    out = hs_matvec(M, cts[g], ctx)
                elif st["policy"] == "lola-dense":
                    out = merge_maps(lola_dense_matvec(M, cts[g], ctx), 1, ctx)
                elif st["policy"] == "lola-stacked":
                    res, slot_of_row = lola_stacked_matvec(M, cts[g], ctx)
                    v = np.zeros(N)
                    v[:M.shape[0]] = res.slots[np.asarray(slot_of_row)]  # value-level de-interleave (free)
                    out = SlotVector(v, CIPHERTEXT)
                else:
                    raise ShapeError(st["label"] + ": ConvPack is not a matrix-vector kernel")
                out = add(out, pack(bias, N, PLAINTEXT), ctx)
                outs.append(out.masked_prefix(M.shape[0]))
            cts, maps = outs, False
            for r in st["layer_idx"]:
                shape = _apply_layer(shape, layers[r], st["label"])
    if len(cts) != 1:
        raise ShapeError("program must end in a single output ciphertext")
    return cts[0].slots[:_shape_size(shape)].copy()


def ref_forward_model(model, weights, image):
    """ref_forward (proj/src/netcompile.cpp:448-503) over a general layer
    list including SubConv groups"""
    t = np.asarray(image, dtype=np.float64)
    for l, w in zip(model["layers"], weights):
        kind = l["kind"]
        if kind == "conv":
            t = ref_conv(t, w[0], w[1], _lget(l, "s", 1))
        elif kind == "subconv":
            g = _lget(l, "groups", 1)
            per = t.shape[0] // g
            t = np.concatenate([ref_conv(t[i * per:(i + 1) * per], w[i][0], w[i][1], _lget(l, "s", 1))
                                for i in range(g)])
        elif kind == "avgpool":
            t = ref_avgpool(t, l["k"], _lget(l, "s", 1))
        elif kind == "square":
            t = ref_square(t)
        elif kind == "flatten":
            t = t.ravel()
        elif kind == "dense":
            t = ref_dense(np.ravel(t), w[0], w[1])
    return np.ravel(t)


def _L(kind, k=0, s=1, out=0, groups=1, policy=None, label=""):
    return dict(kind=kind, k=k, s=s, out=out, groups=groups, policy=policy, label=label)


def builtin_model(name):
    """proj/src/netcompile.cpp:567-635"""
    if name == "cryptonets-hs":
        return dict(name=name, in_c=1, in_d=29, n_slots=8192, layers=[
            _L("conv", 5, 2, 5, label="Conv1"), _L("square"), _L("avgpool", 2, 2),
            _L("conv", 5, 1, 50, label="Conv2"), _L("avgpool", 2, 2), _L("flatten"),
            _L("dense", out=100, label="Dense1"), _L("square"), _L("dense", out=10, label="Dense2")])
    if name == "me":
        return dict(name=name, in_c=1, in_d=30, n_slots=8192, layers=[
            _L("conv", 3, 1, 5, label="Conv1"), _L("square"), _L("avgpool", 3, 2),
            _L("conv", 3, 1, 50, label="Conv2"), _L("avgpool", 3, 2), _L("flatten"),
            _L("dense", out=32, label="Dense1"), _L("square"), _L("dense", out=10, label="Dense2")])
    if name == "ce":
        return dict(name=name, in_c=3, in_d=32, n_slots=16384, layers=[
            _L("conv", 3, 1, 18, label="Conv1"), _L("square"), _L("avgpool", 2, 2, label="Pool1"),
            _L("subconv", 3, 1, 15, 3, label="Conv2"), _L("conv", 1, 1, 64, policy="convpack", label="Conv3"),
            _L("square"), _L("avgpool", 2, 2, label="Pool2"), _L("conv", 3, 1, 64), _L("flatten"),
            _L("dense", out=256, label="Dense1"), _L("square"), _L("dense", out=10, label="Dense2")])
    return None


def model_json(model):
    """the model as a model file (proj/src/modelio.cpp:106-147 schema)"""
    import json
    layers = []
    for l in model["layers"]:
        d = {"kind": l["kind"]}
        if l["kind"] in ("conv", "subconv", "avgpool"):
            d["k"], d["s"] = l["k"], l.get("s") or 1
        if l["kind"] in ("conv", "subconv"):
            d["out_channels"] = l["out"]
        if l["kind"] == "dense":
            d["units"] = l["out"]
        if l["kind"] == "subconv":
            d["groups"] = l.get("groups") or 1
        if l.get("policy"):
            d["policy"] = l["policy"]
        if l.get("label"):
            d["label"] = l["label"]
        layers.append(d)
    return json.dumps({"name": model["name"], "input": [model["in_c"], model["in_d"], model["in_d"]],
                       "n_slots": model["n_slots"], "layers": layers})
