"""oracle/ckks_pipeline.py -- TEST INFRASTRUCTURE ONLY: the CPU-oracle versions of the layer compositions the GPU
path runs, built from oracle/ckks.py primitives and the slot-level
restatement of the reference (oracle/hesim_oracle.py).  Test
infrastructure only."""
from __future__ import annotations

import numpy as np

from oracle import hesim_oracle as HS


def hs_masks(ck, A, level, skip_zero=True):
    """extract_diagonals (proj/src/matvec.cpp:45-65) then mask'_i =
    rot_right(mask_i, i), encoded at scale q_{level-1} in the extended basis."""
    m, n = A.shape
    S = ck.S
    m_eff, masks = HS.extract_diagonals(A, S)
    folds = HS.hs_folds(m, n, S, m_eff)
    rots, enc = [], []
    for i in range(m_eff):
        if skip_zero and not masks[i].any():
            continue
        rots.append(i)
        enc.append(ck.encode(np.roll(masks[i], i), float(ck.primes[level - 1]), level, with_p=True))
    return m_eff, folds, rots, (np.concatenate(enc) if enc else np.zeros(0, dtype=np.uint64))


MAX_FOLD_GROUP = 5  # hoisted fold groups of at most 2^5 - 1 rotations (layers.cu fold_groups)


def fold_groups(folds):
    """the log-depth fold's `folds` doublings split into ceil(folds / 5)
    groups of near-equal size, larger first (layers.cu fold_groups)"""
    if folds <= 0:
        return []
    g = -(-folds // MAX_FOLD_GROUP)
    return [folds // g + (1 if i < folds % g else 0) for i in range(g)]


def fold_rotations(S, m_eff, folds, offset=0):
    """the log-depth fold s += rot_left(s, m_eff 2^t), t = folds-1 .. 0
    (proj/src/matvec.cpp:101-103) sums rot_left(s, m_eff u) over u <
    2^folds; a group of `folds` doublings starting at doubling `offset`
    sums rot_left(s, m_eff 2^offset u); as right rotations, ascending (0 first)"""
    step = m_eff << offset
    return sorted({(S - (step * u) % S) % S for u in range(1 << folds)})


def fold_sum(ck, u, l, m_eff, folds, key):
    """the fold as hoisted rotation sums: per group of a doublings one ModUp
    of u.c1, 2^a - 1 key-switch inner products on the rotated digits, one
    ModDown (the HS machinery with unit masks); groups applied in order of
    their offset -- the same slots as the serial folds, metered as the
    reference's `folds` rotations"""
    off = 0
    for a in fold_groups(folds):
        rots = fold_rotations(ck.S, m_eff, a, off)
        ones = np.ones(len(rots) * (l + 1) * ck.N, dtype=np.uint64)
        kl = [key(ck.galois_right(r)) for r in rots if r != 0]
        u = ck.hs_hoisted(u, l, np.array(rots, dtype=np.int64), ones, np.concatenate(kl))
        off += a
    return u


def hs_matvec(ck, v, level, A, skip_zero=True, keys=None):
    """Oracle HS layer: hoisted diagonal sum, rescale, log-depth fold
    (proj/src/matvec.cpp:82-105) as one hoisted rotation sum.  Returns ct at
    level-1."""
    m_eff, folds, rots, masks = hs_masks(ck, A, level, skip_zero)
    keys = keys if keys is not None else {}

    def key(g):
        if g not in keys:
            keys[g] = ck.galois_key(g)
        return keys[g]

    kl = [key(ck.galois_right(r)) for r in rots if r != 0]
    kbuf = np.concatenate(kl) if kl else np.zeros(1, dtype=np.uint64)
    u = ck.hs_hoisted(v, level, np.array(rots, dtype=np.int64), masks, kbuf)
    u = ck.rescale(u, level)
    return fold_sum(ck, u, level - 1, m_eff, folds, key)


def conv_layer(ck, taps, ntaps, level, weights, bias, w_used, tap_scale):
    """conv_packed_forward (proj/src/convlower.cpp:39-74) + rescale."""
    c_out = len(weights) // ntaps if np.ndim(weights) == 1 else np.asarray(weights).shape[0]
    w = np.asarray(weights, dtype=np.float64).reshape(c_out, ntaps)
    qlast = float(ck.primes[level - 1])
    bpts = np.concatenate([ck.encode(np.full(w_used, bias[co] if bias is not None else 0.0),
                                     tap_scale * qlast, level) for co in range(c_out)])
    maps = ck.conv_mac(taps, ntaps, level, w, c_out, qlast, bpts)
    per = 2 * level * ck.N
    return np.concatenate([ck.rescale(maps[co * per:(co + 1) * per], level) for co in range(c_out)])


def merge(ck, maps, nmaps, level, w, keys=None):
    """merge_maps (proj/src/convlower.cpp:145-160)."""
    keys = keys if keys is not None else {}
    kl = []
    for j in range(1, nmaps):
        g = ck.galois_right(j * w)
        if g not in keys:
            keys[g] = ck.galois_key(g)
        kl.append(keys[g])
    kbuf = np.concatenate(kl) if kl else np.zeros(1, dtype=np.uint64)
    return ck.merge(maps, nmaps, level, w, kbuf)


def square(ck, v, level, rlk):
    return ck.rescale(ck.square(v, level, rlk), level)


def conv_pack_taps(ck, cfg, image, nonce, tap_scale, merged=False):
    """Client side: conv_pack (proj/src/convlower.cpp:9-37) + encode + encrypt,
    nonces nonce*ntaps + t (same convention as hegpu_net_encrypt_image).
    merged: the stage driver's fused Conv1 + Flat1 -- each tap's window is
    packed at every map offset co * d_out^2 (hegpu_net_encrypt_image)."""
    shape = HS.ConvShape(cfg.in_d, cfg.in_c, cfg.k, cfg.s, cfg.c_out)
    taps = HS.conv_pack(image, shape, ck.S)
    L = ck.L
    ntaps = len(taps)
    w_used = shape.d_out() ** 2
    if not merged:
        return np.concatenate([ck.encrypt(ck.encode(t.slots[:w_used], tap_scale, L), L, nonce * ntaps + i)
                               for i, t in enumerate(taps)])
    # fused first layer: R taps per ciphertext, tap s's window replicated
    # over the c_out map blocks of region s % R (hegpu_net_encrypt_image)
    R = tap_regions(ck, cfg)
    F = cfg.c_out * w_used
    G = -(-ntaps // R)
    cts = []
    for g in range(G):
        used = min(R, ntaps - g * R)
        z = np.concatenate([np.tile(taps[g * R + r].slots[:w_used], cfg.c_out) for r in range(used)])
        cts.append(ck.encrypt(ck.encode(z, tap_scale, L), L, nonce * G + g))
    return np.concatenate(cts)


def tap_regions(ck, cfg):
    """taps packed per input ciphertext by the fused first layer"""
    d_out = (cfg.in_d - cfg.k) // cfg.s + 1
    return max(1, min(cfg.k * cfg.k * cfg.in_c, ck.S // (cfg.c_out * d_out * d_out)))


def merged_conv(ck, taps, ntaps, level, weights, bias, w_used, tap_scale, regions=1, keys=None):
    """the fused Conv1 + Flat1 of the stage driver on replicated taps:
    sum_s tap_s * P_s + bias_pt with P_s = W[co][s] on map block co (scale
    q_{level-1}) and the block bias at the product scale, then one rescale:
    the merged ciphertext (maps at offsets co * w_used) -- the same slots as
    conv_packed_forward + merge_maps (convlower.cpp:39-74, 145-160)"""
    W = np.asarray(weights, dtype=np.float64).reshape(-1, ntaps)
    c_out = W.shape[0]
    F = c_out * w_used
    qlast = float(ck.primes[level - 1])
    per = 2 * level * ck.N
    acc = None
    for s_ in range(ntaps):
        r, g = s_ % regions, s_ // regions
        p = ck.encode(np.concatenate([np.zeros(r * F), np.repeat(W[:, s_], w_used)]), qlast, level)
        term = ck.mul_pc(taps[g * per:(g + 1) * per], p, level)
        acc = term if acc is None else ck.add(acc, term, level)
    b = np.repeat(np.asarray(bias, dtype=np.float64) if bias is not None else np.zeros(c_out), w_used)
    acc = ck.add_pc(acc, ck.encode(b, tap_scale * qlast, level), level)
    x = ck.rescale(acc, level)
    if regions > 1:  # regions onto region 0: one hoisted rotation sum (unit masks)
        rots = sorted({(ck.S - (r * F) % ck.S) % ck.S for r in range(regions)})
        keys = keys if keys is not None else {}
        kl = []
        for rr in rots:
            if rr:
                gk = ck.galois_right(rr)
                if gk not in keys:
                    keys[gk] = ck.galois_key(gk)
                kl.append(keys[gk])
        x = ck.hs_hoisted(x, level - 1, np.array(rots, dtype=np.int64),
                          np.ones(len(rots) * level * ck.N, dtype=np.uint64), np.concatenate(kl))
    return x


class PreparedNet:
    """Server-side offline state for one model (keys, encoded HS masks,
    bias plaintexts) so that eval() times only the homomorphic evaluation."""

    def __init__(self, ck, cfg, weights, merged=False):
        """merged: Conv1 + Flat1 fused as the GPU stage driver runs them
        (replicated taps); False: the reference's per-map conv + merge
        (proj/src/netcompile.cpp:321-347) -- the CPU baseline's algorithm."""
        self.ck, self.cfg, self.merged = ck, cfg, merged
        self.tap_scale = 2.0 ** 40
        L = ck.L
        self.ntaps = cfg.k * cfg.k * cfg.in_c
        d_out = (cfg.in_d - cfg.k) // cfg.s + 1
        self.w_used = d_out * d_out
        self.conv_w = np.asarray(weights["conv_w"], dtype=np.float64).reshape(cfg.c_out, -1)
        self.conv_b = np.asarray(weights["conv_b"], dtype=np.float64)
        if not merged:
            qlast = float(ck.primes[L - 1])
            self.conv_bias = np.concatenate([
                ck.encode(np.full(self.w_used, self.conv_b[co]), self.tap_scale * qlast, L)
                for co in range(cfg.c_out)])
        keys = {}
        self.keys = keys

        def key(g):
            if g not in keys:
                keys[g] = ck.galois_key(g)
            return keys[g]

        l = L - 1
        if not merged:
            self.merge_keys = np.concatenate([key(ck.galois_right(j * self.w_used)) for j in range(1, cfg.c_out)]) \
                if cfg.c_out > 1 else np.zeros(1, dtype=np.uint64)
        self.rlk = ck.relin_key()
        scale = self.tap_scale
        self.layers = []
        for W, b in weights["dense"]:
            scale = scale * scale / float(ck.primes[l - 1])
            l -= 1
            m_eff, folds, rots, masks = hs_masks(ck, np.asarray(W), l, True)
            kl = [key(ck.galois_right(r)) for r in rots if r != 0]
            kbuf = np.concatenate(kl) if kl else np.zeros(1, dtype=np.uint64)
            fold, off = [], 0
            for a in fold_groups(folds):
                frots = fold_rotations(ck.S, m_eff, a, off)
                fkl = [key(ck.galois_right(r)) for r in frots if r != 0]
                fold.append((np.array(frots, dtype=np.int64), np.ones(len(frots) * l * ck.N, dtype=np.uint64),
                             np.concatenate(fkl)))
                off += a
            l -= 1
            bias = ck.encode(np.asarray(b), scale, l)
            self.layers.append((l + 1, np.array(rots, dtype=np.int64), masks, kbuf, fold, bias))
        self.out_scale = scale

    def eval(self, taps):
        ck, cfg = self.ck, self.cfg
        L = ck.L
        if self.merged:  # Conv1 + Flat1 fused on the region-packed replicated taps (the stage driver's form)
            x = merged_conv(ck, taps, self.ntaps, L, self.conv_w, self.conv_b, self.w_used, self.tap_scale,
                            tap_regions(ck, cfg), self.keys)
        else:  # the reference's per-map conv, rescale, merge
            maps = ck.conv_mac(taps, self.ntaps, L, self.conv_w, cfg.c_out, float(ck.primes[L - 1]), self.conv_bias)
            per = 2 * L * ck.N
            maps = np.concatenate([ck.rescale(maps[co * per:(co + 1) * per], L) for co in range(cfg.c_out)])
            x = ck.merge(maps, cfg.c_out, L - 1, self.w_used, self.merge_keys)
        l = L - 1
        for lv, rots, masks, kbuf, fold, bias in self.layers:
            x = ck.rescale(ck.square(x, l, self.rlk), l)
            l = lv
            u = ck.rescale(ck.hs_hoisted(x, l, rots, masks, kbuf), l)
            l -= 1
            for frots, fones, fkeys in fold:  # the folds as hoisted rotation sums
                u = ck.hs_hoisted(u, l, frots, fones, fkeys)
            x = ck.add_pc(u, bias, l)
        return x


def run_net(ck, cfg, weights, image, nonce=0, keys=None, merged=False):
    """Full oracle pipeline for one image (client encryption included);
    returns (output ct at the last level, output scale).  merged=False: the
    reference's first layer (conv_pack taps, per-map conv, merge), the GPU
    net's default; True: the fused, region-packed first layer."""
    prep = PreparedNet(ck, cfg, weights, merged=merged)
    taps = conv_pack_taps(ck, cfg, image, nonce, prep.tap_scale, merged=merged)
    return prep.eval(taps), prep.out_scale


def _key(ck, keys, g):
    if g not in keys:
        keys[g] = ck.galois_key(g)
    return keys[g]


def _rotate_and_sum(ck, u, l, delta, keys):
    """rotate_and_sum(v, delta, 1) (proj/src/matvec.cpp:67-80) at level l"""
    for t in range(HS._ceil_log2(delta) - 1, -1, -1):
        g = ck.galois_left(1 << t)
        u = ck.add(u, ck.rotate(u, l, g, _key(ck, keys, g)), l)
    return u


def lola_dense(ck, v, level, A, keys=None):
    """lola_dense_matvec (proj/src/matvec.cpp:107-123) on one ciphertext:
    per row, product with the packed row (scale q_{level-1}) + rescale,
    rotate_and_sum, then masked_prefix(1) as a mask multiply (scale
    q_{level-2}) + rescale.  Returns the m output ciphertexts at level-2."""
    keys = keys if keys is not None else {}
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    S = ck.S
    delta = HS.next_power_of_two(n)
    e0 = np.zeros(S)
    e0[0] = 1.0
    mask = ck.encode(e0, float(ck.primes[level - 2]), level - 1)
    outs = []
    for i in range(m):
        row = np.zeros(S)
        row[:n] = A[i]
        u = ck.rescale(ck.mul_pc(v, ck.encode(row, float(ck.primes[level - 1]), level), level), level)
        u = _rotate_and_sum(ck, u, level - 1, delta, keys)
        outs.append(ck.rescale(ck.mul_pc(u, mask, level - 1), level - 1))
    return np.concatenate(outs)


def lola_stacked(ck, v, level, A, keys=None):
    """lola_stacked_matvec (proj/src/matvec.cpp:125-166) on one ciphertext
    whose slots >= n are zero (the masked_prefix(n) of the input): stacked =
    v + sum_j rot_right(v, j delta); per batch the product with the stacked
    rows + rescale, rotate_and_sum, the segment starts kept by a mask
    multiply + rescale; res = batch_0 + sum_b rot_right(batch_b, b).
    Returns (ct at level-2, slot_of_row)."""
    keys = keys if keys is not None else {}
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    S = ck.S
    delta = HS.next_power_of_two(n)
    k = S // delta
    batches = -(-m // k)
    stacked = v
    for j in range(1, k):
        g = ck.galois_right(j * delta)
        stacked = ck.add(stacked, ck.rotate(v, level, g, _key(ck, keys, g)), level)
    res, slot_of_row = None, [0] * m
    l2 = level - 2
    for b in range(batches):
        rows, clean = np.zeros(S), np.zeros(S)
        for j in range(k):
            if b * k + j < m:
                rows[j * delta: j * delta + n] = A[b * k + j]
                clean[j * delta] = 1.0
                slot_of_row[b * k + j] = j * delta + b
        u = ck.rescale(ck.mul_pc(stacked, ck.encode(rows, float(ck.primes[level - 1]), level), level), level)
        u = _rotate_and_sum(ck, u, level - 1, delta, keys)
        u = ck.rescale(ck.mul_pc(u, ck.encode(clean, float(ck.primes[level - 2]), level - 1), level - 1), level - 1)
        if b == 0:
            res = u
        else:
            g = ck.galois_right(b)
            res = ck.add(res, ck.rotate(u, l2, g, _key(ck, keys, g)), l2)
    return res, slot_of_row


# ------------------------------------------------ general stage driver ---
def repack_conv(ck, taps, level, scale, W, bias, w_used):
    """conv_packed_forward (proj/src/convlower.cpp:39-74) on ciphertexts whose
    slots beyond w_used are NOT zero (the RepackConv stage's rotated group
    ciphertexts, netcompile.cpp:352-379): the reference's masked constant
    plaintexts pt(w[co,t] on slots < w) at scale q_{level-1}, products summed
    in tap order, the masked bias at the product scale, one rescale per map."""
    W = np.asarray(W, dtype=np.float64).reshape(np.asarray(W).shape[0], -1)
    c_out, ntaps = W.shape
    qlast = float(ck.primes[level - 1])
    outs = []
    for co in range(c_out):
        acc = None
        for t in range(ntaps):
            term = ck.mul_pc(taps[t], ck.encode(np.full(w_used, W[co, t]), qlast, level), level)
            acc = term if acc is None else ck.add(acc, term, level)
        acc = ck.add_pc(acc, ck.encode(np.full(w_used, bias[co]), scale * qlast, level), level)
        outs.append(ck.rescale(acc, level))
    return outs


def run_program(ck, model, weights, image, nonce=0, keys=None):
    """The reference's execute (proj/src/netcompile.cpp:291-446) over CKKS,
    stage for stage as hegpu_prog_run evaluates it (csrc/program.cpp):
    returns (output ct, level, scale, n_logits).  Levels: ConvPack,
    RepackConv, Square and Linear(HS) consume one prime, Linear(LoLa-dense)
    two; input scale 2^40 at the top level."""
    stages = HS.lower(model)
    layers, S = model["layers"], ck.S
    if model["n_slots"] != S:
        raise HS.ShapeError("model n_slots must equal the ring's slot count")
    keys = keys if keys is not None else {}
    image = np.asarray(image, dtype=np.float64)
    scale, l = 2.0 ** 40, ck.L
    shape = (model["in_c"], model["in_d"], False, 0)
    cts, maps, seeded, rlk = [], False, False, None
    for st in stages:
        kind = st["kind"]
        if not seeded and kind != "convpack":
            cts, seeded = [ck.encrypt(ck.encode(image.ravel(), scale, l), l, nonce)], True
        if kind == "convpack":
            ly = layers[st["layer_idx"][0]]
            cs = HS.ConvShape(shape[1], shape[0], ly["k"], ly.get("s") or 1, ly["out"])
            taps = HS.conv_pack(image, cs, S)
            w_used, ntaps = cs.d_out() ** 2, len(taps)
            enc = np.concatenate([ck.encrypt(ck.encode(t.slots[:w_used], scale, l), l, nonce * ntaps + i)
                                  for i, t in enumerate(taps)])
            W, b = weights[st["layer_idx"][0]]
            out = conv_layer(ck, enc, ntaps, l, np.asarray(W).reshape(ly["out"], -1), b, w_used, scale)
            l -= 1
            per = 2 * l * ck.N
            cts = [out[i * per:(i + 1) * per] for i in range(ly["out"])]
            maps, seeded = True, True
            shape = HS._apply_layer(shape, ly, st["label"])
        elif kind == "merge":
            G = st["groups"]
            per, w = shape[0] // G, shape[1] * shape[1]
            cts = [merge(ck, np.concatenate(cts[g * per:(g + 1) * per]), per, l, w, keys) for g in range(G)]
            maps = False
        elif kind == "square":
            rlk = rlk if rlk is not None else ck.relin_key()
            cts = [square(ck, v, l, rlk) for v in cts]
            scale = scale * scale / float(ck.primes[l - 1])
            l -= 1
        elif kind == "repackconv":
            ly = layers[st["layer_idx"][0]]
            w = shape[1] * shape[1]
            if maps:
                taps = cts
            else:
                G = len(cts)
                per = shape[0] // G
                taps = []
                for g in range(G):
                    for j in range(per):
                        if j == 0:
                            taps.append(cts[g])
                        else:
                            gl = ck.galois_left(j * w)
                            taps.append(ck.rotate(cts[g], l, gl, _key(ck, keys, gl)))
            W, b = weights[st["layer_idx"][0]]
            cts = repack_conv(ck, taps, l, scale, W, b, w)
            l -= 1
            maps = True
            shape = HS._apply_layer(shape, ly, st["label"])
        else:  # linear
            G = st["groups"]
            outs = []
            for g in range(G):
                M, bias = HS.compose_group(model, weights, st["layer_idx"], g, G, shape)
                if st["policy"] == "hs":
                    u, lo = hs_matvec(ck, cts[g], l, M, True, keys), l - 1
                elif st["policy"] == "lola-dense":
                    rows = lola_dense(ck, cts[g], l, M, keys)
                    u, lo = merge(ck, rows, M.shape[0], l - 2, 1, keys), l - 2
                else:
                    raise HS.ShapeError(st["label"] + ": policy outside the encrypted stage driver")
                outs.append(ck.add_pc(u, ck.encode(bias, scale, lo), lo))
            cts, maps, l = outs, False, lo
            for r in st["layer_idx"]:
                shape = HS._apply_layer(shape, layers[r], st["label"])
    if len(cts) != 1:
        raise HS.ShapeError("program must end in a single output ciphertext")
    return cts[0], l, scale, HS._shape_size(shape)
