"""oracle/ckks.py -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end of the plain-C CKKS checker (oracle/ckks_oracle.c).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product never does.  Parity status: limb level is
builder-authored ("parity unpinned", see ckks_oracle.h); slot semantics are
pinned against the reference through oracle/hesim_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libckks_oracle.so")
_lib = None

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def build() -> str:
    src = os.path.join(_HERE, "ckks_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def _cpu_fingerprint() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def use_native() -> str:
    """switch this process to the -march=native build, compiled on the
    machine that runs it (rebuilt when the host CPU model differs from the
    one it was built for) -- the CPU baseline's build.
    Must be called before the first lib()."""
    global _LIB_PATH
    src = os.path.join(_HERE, "ckks_oracle.c")
    path = os.path.join(_HERE, "libckks_oracle_native.so")
    stamp = path + ".cpu"
    fp = _cpu_fingerprint()
    have = open(stamp).read() if os.path.exists(stamp) else None
    if (not os.path.exists(path) or have != fp or os.path.getmtime(path) < os.path.getmtime(src)):
        subprocess.check_call(["make", "-s", "-C", _HERE, "native"])
        with open(stamp, "w") as f:
            f.write(fp)
    _LIB_PATH = path
    return path


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        vp, i, u, d = C.c_void_p, C.c_int, C.c_uint64, C.c_double
        sig = {
            "ock_create": (vp, [i, i, C.POINTER(C.c_int), i]),
            "ock_destroy": (None, [vp]),
            "ock_prime": (u, [vp, i]),
            "ock_psi": (u, [vp, i]),
            "ock_N": (i, [vp]),
            "ock_ntt": (None, [vp, i, u64p]),
            "ock_intt": (None, [vp, i, u64p]),
            "ock_automorph_ntt": (None, [vp, u, u64p, u64p, i]),
            "ock_automorph_coeff": (None, [vp, i, u, u64p, u64p]),
            "ock_galois_left": (u, [vp, C.c_int64]),
            "ock_galois_right": (u, [vp, C.c_int64]),
            "ock_encode": (None, [vp, f64p, i, d, i, i, u64p]),
            "ock_encode_coeffs": (None, [vp, f64p, i, i, u64p]),
            "ock_encode_fp": (None, [vp, f64p, i, d, f64p]),
            "ock_encode_direct": (None, [vp, f64p, i, d, f64p]),
            "ock_decode": (None, [vp, u64p, i, d, f64p]),
            "ock_secret": (None, [vp, u, u64p]),
            "ock_gen_galois_key": (None, [vp, u, u64p, u, u64p]),
            "ock_gen_relin_key": (None, [vp, u, u64p, u64p]),
            "ock_encrypt": (None, [vp, u, u, u64p, u64p, i, u64p]),
            "ock_decrypt": (None, [vp, u64p, u64p, i, u64p]),
            "ock_add": (None, [vp, u64p, u64p, i, u64p]),
            "ock_add_pc": (None, [vp, u64p, u64p, i, u64p]),
            "ock_mul_pc": (None, [vp, u64p, u64p, i, u64p]),
            "ock_rescale": (None, [vp, u64p, i, u64p]),
            "ock_rotate": (None, [vp, u64p, i, u, u64p, u64p]),
            "ock_square": (None, [vp, u64p, i, u64p, u64p]),
            "ock_conv_mac": (None, [vp, u64p, i, i, f64p, i, d, vp, u64p]),
            "ock_merge": (None, [vp, u64p, i, i, C.c_int64, u64p, u64p]),
            "ock_hs_hoisted": (None, [vp, u64p, i, i, i64p, u64p, u64p, u64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class Ckks:
    """One CKKS parameter set + secret key, mirroring the product's client."""

    def __init__(self, logN: int, qbits, pbits: int, seed: int = 1):
        self.L = len(qbits)
        arr = (C.c_int * self.L)(*qbits)
        self._c = lib().ock_create(logN, self.L, arr, pbits)
        if not self._c:
            raise ValueError("bad CKKS parameters")
        self.N = 1 << logN
        self.S = self.N // 2
        self.np = self.L + 1
        self.primes = [int(lib().ock_prime(self._c, i)) for i in range(self.np)]
        self.seed = seed
        self.s = np.zeros(self.np * self.N, dtype=np.uint64)
        lib().ock_secret(self._c, seed, self.s)
        self.key_words = self.L * 2 * self.np * self.N

    def __del__(self):
        try:
            if self._c:
                lib().ock_destroy(self._c)
        except Exception:
            pass

    # -- transforms ---------------------------------------------------------
    def ntt(self, a, pi):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().ock_ntt(self._c, pi, a)
        return a

    def intt(self, a, pi):
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        lib().ock_intt(self._c, pi, a)
        return a

    def galois_right(self, r):
        return int(lib().ock_galois_right(self._c, r))

    def galois_left(self, r):
        return int(lib().ock_galois_left(self._c, r))

    def automorph_ntt(self, a, g, nlimbs):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        out = np.empty_like(a)
        lib().ock_automorph_ntt(self._c, g, a, out, nlimbs)
        return out

    # -- client ---------------------------------------------------------------
    def encode(self, z, scale, level, with_p=False):
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.empty((level + (1 if with_p else 0)) * self.N, dtype=np.uint64)
        lib().ock_encode(self._c, z, len(z), scale, level, int(with_p), out)
        return out

    def encode_fp(self, z, scale):
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.empty(self.N, dtype=np.float64)
        lib().ock_encode_fp(self._c, z, len(z), scale, out)
        return out

    def encode_direct(self, z, scale):
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.empty(self.N, dtype=np.float64)
        lib().ock_encode_direct(self._c, z, len(z), scale, out)
        return out

    def decode(self, pt, level, scale):
        out = np.empty(self.S, dtype=np.float64)
        lib().ock_decode(self._c, np.ascontiguousarray(pt, dtype=np.uint64),
                         level, scale, out)
        return out

    def encrypt(self, pt, level, nonce):
        ct = np.empty(2 * level * self.N, dtype=np.uint64)
        lib().ock_encrypt(self._c, self.seed, nonce, self.s,
                          np.ascontiguousarray(pt, dtype=np.uint64), level, ct)
        return ct

    def decrypt(self, ct, level):
        pt = np.empty(level * self.N, dtype=np.uint64)
        lib().ock_decrypt(self._c, self.s, np.ascontiguousarray(ct), level, pt)
        return pt

    def decrypt_decode(self, ct, level, scale):
        return self.decode(self.decrypt(ct, level), level, scale)

    def galois_key(self, g):
        key = np.empty(self.key_words, dtype=np.uint64)
        lib().ock_gen_galois_key(self._c, self.seed, self.s, g, key)
        return key

    def relin_key(self):
        key = np.empty(self.key_words, dtype=np.uint64)
        lib().ock_gen_relin_key(self._c, self.seed, self.s, key)
        return key

    # -- evaluator ----------------------------------------------------------
    def add(self, a, b, l):
        out = np.empty_like(a)
        lib().ock_add(self._c, a, b, l, out)
        return out

    def add_pc(self, a, pt, l):
        out = np.empty_like(a)
        lib().ock_add_pc(self._c, a, np.ascontiguousarray(pt), l, out)
        return out

    def mul_pc(self, a, pt, l):
        out = np.empty_like(a)
        lib().ock_mul_pc(self._c, a, np.ascontiguousarray(pt), l, out)
        return out

    def rescale(self, a, l):
        out = np.empty(2 * (l - 1) * self.N, dtype=np.uint64)
        lib().ock_rescale(self._c, a, l, out)
        return out

    def rotate(self, a, l, g, key):
        out = np.empty_like(a)
        lib().ock_rotate(self._c, a, l, g, key, out)
        return out

    def square(self, a, l, rlk):
        out = np.empty_like(a)
        lib().ock_square(self._c, a, l, rlk, out)
        return out

    def conv_mac(self, taps, ntaps, l, weights, c_out, wscale, bias_pts=None):
        out = np.empty(c_out * 2 * l * self.N, dtype=np.uint64)
        w = np.ascontiguousarray(weights, dtype=np.float64).ravel()
        bp = None
        if bias_pts is not None:
            bias_pts = np.ascontiguousarray(bias_pts, dtype=np.uint64)
            bp = bias_pts.ctypes.data
        lib().ock_conv_mac(self._c, np.ascontiguousarray(taps), ntaps, l, w,
                           c_out, wscale, bp, out)
        return out

    def merge(self, maps, nmaps, l, w, keys):
        out = np.empty(2 * l * self.N, dtype=np.uint64)
        lib().ock_merge(self._c, np.ascontiguousarray(maps), nmaps, l, w,
                        np.ascontiguousarray(keys), out)
        return out

    def hs_hoisted(self, v, l, rots, masks_ext, keys):
        out = np.empty(2 * l * self.N, dtype=np.uint64)
        rots = np.ascontiguousarray(rots, dtype=np.int64)
        if keys is None or len(keys) == 0:
            keys = np.zeros(1, dtype=np.uint64)
        lib().ock_hs_hoisted(self._c, v, l, len(rots), rots,
                             np.ascontiguousarray(masks_ext),
                             np.ascontiguousarray(keys), out)
        return out
