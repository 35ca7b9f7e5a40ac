"""ctypes front end of libhegpu.so (include/hegpu.h) for tests and bench.py.

This is plumbing over the C-ABI, not a second implementation: every call
goes to the native library, and importing fails loudly if it is missing.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEGPU_LIB") or os.path.join(_HERE, "libhegpu.so")

OK, ERR_CAPACITY, ERR_SHAPE, ERR_LAYOUT, ERR_RANGE, ERR_IO, ERR_CUDA, ERR_NCCL, ERR_ARG, ERR_KEY = range(10)
CLIENT_ONLY = -1
MAX_Q = 15
TALLY_FIELDS = ("add_pc", "add_cc", "mul_pc", "mul_cc", "rot")


class HegpuError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[hegpu {code}] {msg}")
        self.code = code


class CapacityError(HegpuError):
    """hesim::CapacityError (proj/include/hesim/errors.hpp:9-12)"""


class ShapeError(HegpuError):
    """hesim::ShapeError"""


class LayoutError(HegpuError):
    """hesim::LayoutError"""


class RangeError(HegpuError, IndexError):
    """std::out_of_range (proj/src/slotvec.cpp:45-48)"""


class IoError(HegpuError):
    """hesim::IoError (model / weights / input files)"""


_ERR = {ERR_CAPACITY: CapacityError, ERR_SHAPE: ShapeError, ERR_LAYOUT: LayoutError, ERR_RANGE: RangeError,
        ERR_IO: IoError}


class Params(C.Structure):
    _fields_ = [("log_n", C.c_int), ("n_q", C.c_int), ("q_bits", C.c_int * MAX_Q),
                ("p_bits", C.c_int), ("seed", C.c_uint64)]


class NetSpec(C.Structure):
    _fields_ = [("in_c", C.c_int), ("in_d", C.c_int), ("k", C.c_int), ("stride", C.c_int),
                ("c_out", C.c_int), ("n_dense", C.c_int), ("dense_out", C.c_int * 4),
                ("first_layer", C.c_int)]


FIRST_LAYERS = {"reference": 0, "fused": 1}  # HEGPU_FIRST_LAYER_*


_lib = None
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2110_08321_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i, u, d, sz = C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_size_t
        pp = C.POINTER(C.c_void_p)
        sig = {
            "hegpu_ctx_create": (i, [C.POINTER(Params), i, pp]),
            "hegpu_ctx_destroy": (None, [vp]),
            "hegpu_last_error": (C.c_char_p, [vp]),
            "hegpu_ctx_info": (i, [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i), u64p]),
            "hegpu_sync": (i, [vp]),
            "hegpu_kernel_launches": (C.c_int64, [vp]),
            "hegpu_stream": (vp, [vp]),
            "hegpu_capture_begin": (i, [vp]),
            "hegpu_capture_end": (i, [vp, pp]),
            "hegpu_graph_launch": (i, [vp]),
            "hegpu_graph_destroy": (None, [vp]),
            "hegpu_kernel_timer": (i, [vp, C.c_char_p]),
            "hegpu_kernel_timer_read": (i, [vp, C.POINTER(d), C.POINTER(C.c_int64), C.POINTER(d)]),
            "hegpu_kernel_timer_read_ops": (i, [vp, C.POINTER(d), C.POINTER(C.c_int64), C.POINTER(d), C.POINTER(d)]),
            "hegpu_ct_export_device": (i, [vp, vp, sz]),
            "hegpu_begin_stage": (i, [vp, C.c_char_p]),
            "hegpu_num_stages": (i, [vp]),
            "hegpu_stage_tally": (i, [vp, i, C.c_char_p, i, i64p]),
            "hegpu_total_tally": (i, [vp, i64p]),
            "hegpu_reset_meter": (i, [vp]),
            "hegpu_ks_counters": (i, [vp, i64p]),
            "hegpu_encode": (i, [vp, f64p, i, d, i, i, u64p]),
            "hegpu_decode": (i, [vp, u64p, i, d, f64p]),
            "hegpu_encrypt": (i, [vp, u64p, i, u, u64p]),
            "hegpu_decrypt": (i, [vp, u64p, i, u64p]),
            "hegpu_gen_rotation_keys": (i, [vp, i64p, i]),
            "hegpu_gen_relin_key": (i, [vp]),
            "hegpu_export_rotation_key": (i, [vp, C.c_int64, u64p]),
            "hegpu_export_relin_key": (i, [vp, u64p]),
            "hegpu_ct_create": (i, [vp, i, i, pp]),
            "hegpu_ct_destroy": (None, [vp]),
            "hegpu_ct_upload": (i, [vp, vp, sz, d]),
            "hegpu_ct_download": (i, [vp, vp, sz]),
            "hegpu_ct_info": (i, [vp, C.POINTER(i), C.POINTER(i), C.POINTER(d)]),
            "hegpu_pt_create": (i, [vp, i, i, i, pp]),
            "hegpu_pt_destroy": (None, [vp]),
            "hegpu_pt_upload": (i, [vp, vp, sz, d]),
            "hegpu_pt_download": (i, [vp, vp, sz]),
            "hegpu_add": (i, [vp, vp, vp, vp]),
            "hegpu_add_plain": (i, [vp, vp, vp, vp]),
            "hegpu_mul_plain": (i, [vp, vp, vp, vp]),
            "hegpu_rescale": (i, [vp, vp, vp]),
            "hegpu_rotate_right": (i, [vp, vp, C.c_int64, vp]),
            "hegpu_rotate_left": (i, [vp, vp, C.c_int64, vp]),
            "hegpu_square": (i, [vp, vp, vp]),
            "hegpu_conv_packed_forward": (i, [vp, vp, i, f64p, i, vp, i, vp]),
            "hegpu_merge_maps": (i, [vp, vp, i, C.c_int64, vp]),
            "hegpu_conv_plan_create": (i, [vp, i, f64p, i, vp, i, i, d, pp]),
            "hegpu_conv_plan_destroy": (None, [vp]),
            "hegpu_conv_plan_run": (i, [vp, vp, vp, vp]),
            "hegpu_hs_plan_create": (i, [vp, f64p, i, i, i, i, pp]),
            "hegpu_hs_plan_destroy": (None, [vp]),
            "hegpu_hs_plan_rotations": (i, [vp, vp, i]),
            "hegpu_hs_plan_info": (i, [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i)]),
            "hegpu_hs_matvec": (i, [vp, vp, vp, vp]),
            "hegpu_lola_plan_create": (i, [vp, i, f64p, i, i, i, pp]),
            "hegpu_lola_plan_destroy": (None, [vp]),
            "hegpu_lola_plan_rotations": (i, [vp, vp, i]),
            "hegpu_lola_plan_info": (i, [vp] + [C.POINTER(i)] * 5),
            "hegpu_lola_slot_of_row": (C.c_int64, [vp, i]),
            "hegpu_lola_matvec": (i, [vp, vp, vp, vp]),
            "hegpu_hs_acc_words": (C.c_size_t, [vp, i]),
            "hegpu_hs_matvec_partial": (i, [vp, vp, vp, i, i, vp]),
            "hegpu_hs_matvec_finish": (i, [vp, vp, vp, vp, i, vp]),
            "hegpu_net_create": (i, [vp, C.POINTER(NetSpec), f64p, f64p, vp, vp, pp]),
            "hegpu_net_destroy": (None, [vp]),
            "hegpu_net_run": (i, [vp, vp, vp]),
            "hegpu_net_run_compact": (i, [vp, vp, i, vp]),
            "hegpu_model_parse": (i, [C.c_char_p, pp]),
            "hegpu_model_load": (i, [C.c_char_p, pp]),
            "hegpu_model_last_error": (C.c_char_p, [vp]),
            "hegpu_model_destroy": (None, [vp]),
            "hegpu_model_info": (i, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), C.POINTER(C.c_size_t)]),
            "hegpu_model_layer": (i, [vp, i] + [C.POINTER(C.c_int)] * 6),
            "hegpu_model_load_weights": (i, [vp, C.c_char_p, f64p, C.c_size_t]),
            "hegpu_model_save_weights": (i, [vp, C.c_char_p, f64p, C.c_size_t]),
            "hegpu_model_load_input": (i, [vp, C.c_char_p, f64p]),
            "hegpu_model_save_input": (i, [vp, C.c_char_p, f64p]),
            "hegpu_model_net_spec": (i, [vp, C.POINTER(NetSpec)]),
            "hegpu_model_compose": (i, [vp, f64p, C.c_size_t, i, vp, vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
            "hegpu_net_create_from_model": (i, [vp, vp, C.c_char_p, pp]),
            "hegpu_net_run_split": (i, [vp, vp, vp, i, i, i, REDUCE_FN, vp]),
            "hegpu_net_run_host": (i, [vp, vp, i, vp]),
            "hegpu_net_encrypt_image": (i, [vp, f64p, u, u64p]),
            "hegpu_net_decrypt_logits": (i, [vp, u64p, f64p]),
            "hegpu_net_output_scale": (d, [vp]),
            "hegpu_compact_bytes": (sz, [vp, i]),
            "hegpu_encrypt_compact": (i, [vp, u64p, i, u, vp]),
            "hegpu_ct_upload_compact": (i, [vp, vp, sz, d]),
            "hegpu_net_compact_image_bytes": (sz, [vp]),
            "hegpu_net_encrypt_image_compact": (i, [vp, f64p, u, vp]),
            "hegpu_net_run_host_compact": (i, [vp, vp, i, i, vp]),
            "hegpu_net_submit_host_compact": (i, [vp, vp, i, i, vp]),
            "hegpu_net_tap_cts": (i, [vp]),
            "hegpu_net_first_layer": (i, [vp]),
            "hegpu_net_wait": (i, [vp]),
            "hegpu_model_set_default_policy": (i, [vp, i]),
            "hegpu_model_set_n_slots": (i, [vp, i]),
            "hegpu_masked_conv_create": (i, [vp, i, f64p, i, vp, i, i, d, pp]),
            "hegpu_masked_conv_destroy": (None, [vp]),
            "hegpu_masked_conv_run": (i, [vp, vp, vp, vp]),
            "hegpu_ct_view": (i, [vp, i, i, pp]),
            "hegpu_ct_copy": (i, [vp, vp]),
            "hegpu_ct_gather": (i, [vp, i, vp, i, i, i]),
            "hegpu_ct_set_scale": (i, [vp, d]),
            "hegpu_prog_create": (i, [vp, vp, f64p, sz, pp]),
            "hegpu_prog_destroy": (None, [vp]),
            "hegpu_prog_info": (i, [vp] + [C.POINTER(i)] * 4),
            "hegpu_prog_stage": (i, [vp, i, C.c_char_p, i] + [C.POINTER(i)] * 3),
            "hegpu_model_lower": (i, [vp, i, vp, vp, vp, vp]),
            "hegpu_prog_encrypt_input": (i, [vp, f64p, u, u64p]),
            "hegpu_prog_run": (i, [vp, vp, vp]),
            "hegpu_prog_decrypt_logits": (i, [vp, u64p, f64p]),
            "hegpu_prog_output_scale": (d, [vp]),
            "hegpu_prog_last_error": (C.c_char_p, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


# int (*hegpu_reduce_fn)(void* dev_words, size_t words, void* user)
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_size_t, C.c_void_p)


class _DevWords:
    """zero-copy view of a library device buffer for torch (CUDA array interface)"""

    def __init__(self, ptr, words):
        self.__cuda_array_interface__ = {"shape": (words,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3, "strides": None}


def declared_symbols():
    """Every function include/hegpu.h declares (for the export test)."""
    import re
    root = os.path.dirname(_HERE)
    text = open(os.path.join(root, "include", "hegpu.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char|int64_t|double|size_t)\s*\*?\s*(hegpu_\w+)\(",
                                 text, re.M)))


def _ctx_alive(obj):
    """a handle tied to a context is destroyed only while that context lives
    (at interpreter shutdown the GC may finalize the context first: the
    context's teardown already released the device memory)"""
    ctx = getattr(obj, "ctx", None)
    return ctx is None or getattr(ctx, "h", None) is not None


class Context:
    def __init__(self, log_n, qbits, pbits, seed=1, device=0):
        p = Params()
        p.log_n = log_n
        p.n_q = len(qbits)
        for k, b in enumerate(qbits):
            p.q_bits[k] = b
        p.p_bits = pbits
        p.seed = seed
        h = C.c_void_p()
        rc = lib().hegpu_ctx_create(C.byref(p), device, C.byref(h))
        if rc:
            raise _ERR.get(rc, HegpuError)(rc, lib().hegpu_last_error(None).decode())
        self.h = h
        self.L = len(qbits)
        self.np = self.L + 1
        n, s, nq = C.c_int(), C.c_int(), C.c_int()
        primes = np.zeros(self.np, dtype=np.uint64)
        lib().hegpu_ctx_info(h, C.byref(n), C.byref(s), C.byref(nq), primes)
        self.N, self.S = n.value, s.value
        self.primes = [int(x) for x in primes]
        self.key_words = self.L * 2 * self.np * self.N

    def close(self):
        if getattr(self, "h", None):
            lib().hegpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc):
        if rc:
            raise _ERR.get(rc, HegpuError)(rc, lib().hegpu_last_error(self.h).decode())

    # -- client -----------------------------------------------------------
    def encode(self, z, scale, level, with_p=False):
        z = np.ascontiguousarray(z, dtype=np.float64)
        out = np.empty((level + int(with_p)) * self.N, dtype=np.uint64)
        self.check(lib().hegpu_encode(self.h, z, len(z), scale, level, int(with_p), out))
        return out

    def decode(self, pt, level, scale):
        out = np.empty(self.S, dtype=np.float64)
        self.check(lib().hegpu_decode(self.h, np.ascontiguousarray(pt, dtype=np.uint64), level, scale, out))
        return out

    def encrypt(self, pt, level, nonce):
        ct = np.empty(2 * level * self.N, dtype=np.uint64)
        self.check(lib().hegpu_encrypt(self.h, np.ascontiguousarray(pt, dtype=np.uint64), level, nonce, ct))
        return ct

    def compact_bytes(self, level):
        return int(lib().hegpu_compact_bytes(self.h, level))

    def encrypt_compact(self, pt, level, nonce):
        out = np.empty(self.compact_bytes(level), dtype=np.uint8)
        self.check(lib().hegpu_encrypt_compact(self.h, np.ascontiguousarray(pt, dtype=np.uint64), level, nonce,
                                               out.ctypes.data))
        return out

    def decrypt(self, ct, level):
        pt = np.empty(level * self.N, dtype=np.uint64)
        self.check(lib().hegpu_decrypt(self.h, np.ascontiguousarray(ct, dtype=np.uint64), level, pt))
        return pt

    def export_rotation_key(self, r):
        out = np.empty(self.key_words, dtype=np.uint64)
        self.check(lib().hegpu_export_rotation_key(self.h, r, out))
        return out

    def export_relin_key(self):
        out = np.empty(self.key_words, dtype=np.uint64)
        self.check(lib().hegpu_export_relin_key(self.h, out))
        return out

    def gen_rotation_keys(self, rights):
        r = np.ascontiguousarray(rights, dtype=np.int64)
        self.check(lib().hegpu_gen_rotation_keys(self.h, r, len(r)))

    def gen_relin_key(self):
        self.check(lib().hegpu_gen_relin_key(self.h))

    # -- device objects -------------------------------------------------------
    def ct(self, count, level, data=None, scale=1.0):
        return Ciphertext(self, count, level, data, scale)

    def pt(self, count, level, with_p=False, data=None, scale=1.0):
        return Plaintext(self, count, level, with_p, data, scale)

    # -- metering -------------------------------------------------------------
    def begin_stage(self, label):
        self.check(lib().hegpu_begin_stage(self.h, label.encode()))

    def stages(self):
        out = []
        buf = C.create_string_buffer(128)
        for i in range(lib().hegpu_num_stages(self.h)):
            t = np.zeros(5, dtype=np.int64)
            self.check(lib().hegpu_stage_tally(self.h, i, buf, 128, t))
            out.append((buf.value.decode(), tuple(int(x) for x in t)))
        return out

    def total(self):
        t = np.zeros(5, dtype=np.int64)
        self.check(lib().hegpu_total_tally(self.h, t))
        return tuple(int(x) for x in t)

    def reset_meter(self):
        self.check(lib().hegpu_reset_meter(self.h))

    KS_FIELDS = ("modups", "key_inner_products", "moddowns", "rescales")

    def ks_counters(self):
        """key-switch work actually executed since reset_meter (hegpu_ks_counters)"""
        t = np.zeros(4, dtype=np.int64)
        self.check(lib().hegpu_ks_counters(self.h, t))
        return dict(zip(self.KS_FIELDS, (int(x) for x in t)))

    def launches(self):
        return int(lib().hegpu_kernel_launches(self.h))

    def stream_ptr(self):
        return lib().hegpu_stream(self.h) or 0

    def capture(self, fn):
        """capture everything fn() enqueues into a CUDA graph; returns a
        replay callable (metering advances only during capture)"""
        self.check(lib().hegpu_capture_begin(self.h))
        try:
            fn()
        finally:
            g = C.c_void_p()
            self.check(lib().hegpu_capture_end(self.h, C.byref(g)))
        return Graph(self, g)

    def kernel_timer(self, name):
        """arm per-launch CUDA-event timing of one kernel (None disables)"""
        self.check(lib().hegpu_kernel_timer(self.h, name.encode() if name else None))

    def kernel_timer_read(self):
        """(total device ms, launches, algorithmic bytes) since arming"""
        ms, n, b = C.c_double(), C.c_int64(), C.c_double()
        self.check(lib().hegpu_kernel_timer_read(self.h, C.byref(ms), C.byref(n), C.byref(b)))
        return ms.value, n.value, b.value

    def kernel_timer_read_ops(self):
        """(total device ms, launches, algorithmic bytes, algorithmic modular
        multiplies) since arming"""
        ms, n, b, o = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        self.check(lib().hegpu_kernel_timer_read_ops(self.h, C.byref(ms), C.byref(n), C.byref(b), C.byref(o)))
        return ms.value, n.value, b.value, o.value

    def sync(self):
        self.check(lib().hegpu_sync(self.h))

    # -- evaluator ------------------------------------------------------------
    def add(self, a, b, out):
        self.check(lib().hegpu_add(self.h, a.h, b.h, out.h))
        return out

    def add_plain(self, a, p, out):
        self.check(lib().hegpu_add_plain(self.h, a.h, p.h, out.h))
        return out

    def mul_plain(self, a, p, out):
        self.check(lib().hegpu_mul_plain(self.h, a.h, p.h, out.h))
        return out

    def rescale(self, a, out):
        self.check(lib().hegpu_rescale(self.h, a.h, out.h))
        return out

    def rotate_right(self, a, r, out):
        self.check(lib().hegpu_rotate_right(self.h, a.h, r, out.h))
        return out

    def rotate_left(self, a, r, out):
        self.check(lib().hegpu_rotate_left(self.h, a.h, r, out.h))
        return out

    def square(self, a, out):
        self.check(lib().hegpu_square(self.h, a.h, out.h))
        return out

    def conv_packed_forward(self, taps, ntaps, weights, bias, w_used, out):
        w = np.ascontiguousarray(weights, dtype=np.float64).ravel()
        c_out = len(w) // ntaps
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        self.check(lib().hegpu_conv_packed_forward(self.h, taps.h, ntaps, w, c_out,
                                                   None if b is None else b.ctypes.data, w_used, out.h))
        return out

    def conv_plan(self, ntaps, weights, bias, w_used, level, tap_scale):
        return ConvPlan(self, ntaps, weights, bias, w_used, level, tap_scale)

    def conv_plan_run(self, plan, taps, out):
        self.check(lib().hegpu_conv_plan_run(self.h, plan.h, taps.h, out.h))
        return out

    def merge_maps(self, maps, c, w, out):
        self.check(lib().hegpu_merge_maps(self.h, maps.h, c, w, out.h))
        return out

    def hs_plan(self, A, level, skip_zero=True):
        return HsPlan(self, A, level, skip_zero)

    def hs_matvec(self, plan, v, out):
        self.check(lib().hegpu_hs_matvec(self.h, plan.h, v.h, out.h))
        return out

    def lola_plan(self, kind, A, level):
        """kind: "dense" (lola_dense_matvec) or "stacked" (lola_stacked_matvec)"""
        return LolaPlan(self, kind, A, level)

    def lola_matvec(self, plan, v, out):
        self.check(lib().hegpu_lola_matvec(self.h, plan.h, v.h, out.h))
        return out

    def hs_acc_words(self, plan, batch):
        return int(lib().hegpu_hs_acc_words(plan.h, batch))

    def hs_matvec_partial(self, plan, v, part, nparts, acc):
        """extended-basis partial accumulator of diagonal range `part` of
        `nparts` into `acc` (a CUDA int64 tensor of hs_acc_words words)"""
        self.check(lib().hegpu_hs_matvec_partial(self.h, plan.h, v.h, part, nparts, acc.data_ptr()))
        return acc

    def hs_matvec_finish(self, plan, v, acc, nparts, out):
        """ModDown + rescale + folds from the element-wise sum of nparts partials"""
        self.check(lib().hegpu_hs_matvec_finish(self.h, plan.h, v.h, acc.data_ptr(), nparts, out.h))
        return out


class Graph:
    def __init__(self, ctx, h):
        self.ctx, self.h = ctx, h

    def __call__(self):
        self.ctx.check(lib().hegpu_graph_launch(self.h))

    def __del__(self):
        try:
            if self.h and _ctx_alive(self):
                lib().hegpu_graph_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Ciphertext:
    def __init__(self, ctx, count, level, data=None, scale=1.0):
        self.ctx, self.count, self.level = ctx, count, level
        h = C.c_void_p()
        ctx.check(lib().hegpu_ct_create(ctx.h, count, level, C.byref(h)))
        self.h = h
        if data is not None:
            self.upload(data, scale)

    @property
    def words(self):
        return self.count * 2 * self.level * self.ctx.N

    def upload(self, data, scale=1.0):
        data = np.ascontiguousarray(data, dtype=np.uint64)
        self.ctx.check(lib().hegpu_ct_upload(self.h, data.ctypes.data, data.size, scale))

    def download(self):
        out = np.empty(self.words, dtype=np.uint64)
        self.ctx.check(lib().hegpu_ct_download(self.h, out.ctypes.data, out.size))
        return out

    def upload_compact(self, data, scale=1.0):
        data = np.ascontiguousarray(data, dtype=np.uint8)
        self.ctx.check(lib().hegpu_ct_upload_compact(self.h, data.ctypes.data, data.size, scale))

    def export_device(self, dev_ptr):
        self.ctx.check(lib().hegpu_ct_export_device(self.h, dev_ptr, self.words))

    @property
    def scale(self):
        s = C.c_double()
        lib().hegpu_ct_info(self.h, None, None, C.byref(s))
        return s.value

    def __del__(self):
        try:
            if self.h and _ctx_alive(self):
                lib().hegpu_ct_destroy(self.h)
                self.h = None
        except Exception:
            pass


class Plaintext:
    def __init__(self, ctx, count, level, with_p=False, data=None, scale=1.0):
        self.ctx, self.count, self.level, self.with_p = ctx, count, level, with_p
        h = C.c_void_p()
        ctx.check(lib().hegpu_pt_create(ctx.h, count, level, int(with_p), C.byref(h)))
        self.h = h
        if data is not None:
            self.upload(data, scale)

    @property
    def words(self):
        return self.count * (self.level + int(self.with_p)) * self.ctx.N

    def upload(self, data, scale=1.0):
        data = np.ascontiguousarray(data, dtype=np.uint64)
        self.ctx.check(lib().hegpu_pt_upload(self.h, data.ctypes.data, data.size, scale))

    def download(self):
        out = np.empty(self.words, dtype=np.uint64)
        self.ctx.check(lib().hegpu_pt_download(self.h, out.ctypes.data, out.size))
        return out

    def __del__(self):
        try:
            if self.h and _ctx_alive(self):
                lib().hegpu_pt_destroy(self.h)
                self.h = None
        except Exception:
            pass


class ConvPlan:
    def __init__(self, ctx, ntaps, weights, bias, w_used, level, tap_scale):
        w = np.ascontiguousarray(weights, dtype=np.float64).ravel()
        self.c_out = len(w) // ntaps
        self._b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        h = C.c_void_p()
        ctx.check(lib().hegpu_conv_plan_create(ctx.h, ntaps, w, self.c_out,
                                               None if self._b is None else self._b.ctypes.data,
                                               w_used, level, tap_scale, C.byref(h)))
        self.ctx, self.h = ctx, h

    def __del__(self):
        try:
            if self.h and _ctx_alive(self):
                lib().hegpu_conv_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass


class HsPlan:
    def __init__(self, ctx, A, level, skip_zero=True):
        A = np.ascontiguousarray(A, dtype=np.float64)
        self.ctx, self.m, self.n = ctx, A.shape[0], A.shape[1]
        h = C.c_void_p()
        ctx.check(lib().hegpu_hs_plan_create(ctx.h, A.ravel(), self.m, self.n, level, int(skip_zero),
                                             C.byref(h)))
        self.h = h
        me, fo, ke = C.c_int(), C.c_int(), C.c_int()
        lib().hegpu_hs_plan_info(h, C.byref(me), C.byref(fo), C.byref(ke))
        self.m_eff, self.folds, self.kept = me.value, fo.value, ke.value

    def rotations(self):
        n = lib().hegpu_hs_plan_rotations(self.h, None, 0)
        r = np.zeros(max(n, 1), dtype=np.int64)
        lib().hegpu_hs_plan_rotations(self.h, r.ctypes.data, n)
        return [int(x) for x in r[:n]]

    def __del__(self):
        try:
            if self.h and _ctx_alive(self):
                lib().hegpu_hs_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass


class LolaPlan:
    KINDS = {"dense": 0, "stacked": 1}

    def __init__(self, ctx, kind, A, level):
        A = np.ascontiguousarray(A, dtype=np.float64)
        self.ctx, self.kind, self.m, self.n, self.level = ctx, kind, A.shape[0], A.shape[1], level
        h = C.c_void_p()
        ctx.check(lib().hegpu_lola_plan_create(ctx.h, self.KINDS[kind], A.ravel(), self.m, self.n, level,
                                               C.byref(h)))
        self.h = h
        v = [C.c_int() for _ in range(5)]
        lib().hegpu_lola_plan_info(h, *[C.byref(x) for x in v])
        self.delta, self.k, self.batches, self.folds, self.per_input = (x.value for x in v)

    def rotations(self):
        n = lib().hegpu_lola_plan_rotations(self.h, None, 0)
        r = np.zeros(max(n, 1), dtype=np.int64)
        lib().hegpu_lola_plan_rotations(self.h, r.ctypes.data, n)
        return [int(x) for x in r[:n]]

    def slot_of_row(self):
        return [int(lib().hegpu_lola_slot_of_row(self.h, i)) for i in range(self.m)]

    def __del__(self):
        try:
            if self.h and _ctx_alive(self):
                lib().hegpu_lola_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass


LAYER_KINDS = ("conv", "subconv", "avgpool", "square", "flatten", "dense")
POLICIES = ("convpack", "hs", "lola-dense", "lola-stacked")


class _SpecCfg:
    """the NetConfig fields a Net needs, from a hegpu_net_spec"""

    def __init__(self, spec):
        self.in_c, self.in_d, self.k, self.s, self.c_out = spec.in_c, spec.in_d, spec.k, spec.stride, spec.c_out
        self.dense = tuple(spec.dense_out[i] for i in range(spec.n_dense))


class Model:
    """A model description (parse_model_json / resolve_model,
    proj/src/modelio.cpp:106-167) with its weights and input file formats."""

    def __init__(self, h):
        self.h = h
        ic, d, ns, nl, nw = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_size_t()
        self._check(lib().hegpu_model_info(h, C.byref(ic), C.byref(d), C.byref(ns), C.byref(nl), C.byref(nw)))
        self.in_c, self.in_d, self.n_slots, self.weight_floats = ic.value, d.value, ns.value, nw.value
        self.layers = []
        for k in range(nl.value):
            v = [C.c_int() for _ in range(6)]
            self._check(lib().hegpu_model_layer(h, k, *[C.byref(x) for x in v]))
            kind, kk, s, out, groups, pol = (x.value for x in v)
            self.layers.append({"kind": LAYER_KINDS[kind], "k": kk, "s": s, "out": out, "groups": groups,
                                "policy": POLICIES[pol] if pol >= 0 else None})

    @staticmethod
    def _status(rc, h=None):
        if rc:
            msg = lib().hegpu_model_last_error(h)
            raise _ERR.get(rc, HegpuError)(rc, msg.decode() if msg else "")

    def _check(self, rc):
        Model._status(rc, self.h)

    @classmethod
    def parse(cls, text):
        h = C.c_void_p()
        cls._status(lib().hegpu_model_parse(text.encode(), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, name_or_path):
        h = C.c_void_p()
        cls._status(lib().hegpu_model_load(str(name_or_path).encode(), C.byref(h)))
        return cls(h)

    def __del__(self):
        try:
            lib().hegpu_model_destroy(self.h)
        except Exception:
            pass

    def load_weights(self, path):
        out = np.empty(self.weight_floats, dtype=np.float64)
        self._check(lib().hegpu_model_load_weights(self.h, str(path).encode(), out, out.size))
        return out

    def save_weights(self, path, flat):
        flat = np.ascontiguousarray(flat, dtype=np.float64)
        self._check(lib().hegpu_model_save_weights(self.h, str(path).encode(), flat, flat.size))

    def load_input(self, path):
        out = np.empty(self.in_c * self.in_d * self.in_d, dtype=np.float64)
        self._check(lib().hegpu_model_load_input(self.h, str(path).encode(), out))
        return out.reshape(self.in_c, self.in_d, self.in_d)

    def save_input(self, path, x):
        x = np.ascontiguousarray(x, dtype=np.float64).ravel()
        self._check(lib().hegpu_model_save_input(self.h, str(path).encode(), x))

    def compose(self, weights, stage):
        """lower()'s composed affine map (M, b) of linear stage `stage`"""
        w = np.ascontiguousarray(weights, dtype=np.float64)
        r, c = C.c_int(), C.c_int()
        self._check(lib().hegpu_model_compose(self.h, w, w.size, stage, None, None, C.byref(r), C.byref(c)))
        M = np.empty((r.value, c.value))
        b = np.empty(r.value)
        self._check(lib().hegpu_model_compose(self.h, w, w.size, stage, M.ctypes.data, b.ctypes.data, None, None))
        return M, b

    def set_default_policy(self, policy):
        """ModelSpec::default_policy (netcompile.hpp:33-35): 'hs', 'lola-dense' or 'lola-stacked'"""
        self._check(lib().hegpu_model_set_default_policy(self.h, POLICIES.index(policy)))

    def set_n_slots(self, n_slots):
        self._check(lib().hegpu_model_set_n_slots(self.h, n_slots))
        self.n_slots = n_slots

    def lower(self):
        """lower() (proj/src/netcompile.cpp:106-213): the stage list as dicts
        {label, kind, groups, policy}"""
        cap = 64
        labels = (C.c_char * 64 * cap)()
        kinds, groups, pols = (C.c_int * cap)(), (C.c_int * cap)(), (C.c_int * cap)()
        n = lib().hegpu_model_lower(self.h, cap, labels, kinds, groups, pols)
        if n < 0:
            msg = lib().hegpu_prog_last_error(None)
            raise _ERR.get(-n, HegpuError)(-n, msg.decode() if msg else "")
        return [{"label": labels[k].value.decode(), "kind": STAGE_KINDS[kinds[k]], "groups": groups[k],
                 "policy": POLICIES[pols[k]]} for k in range(n)]

    def net_spec(self):
        spec = NetSpec()
        self._status(lib().hegpu_model_net_spec(self.h, C.byref(spec)), None)
        return spec


STAGE_KINDS = ("convpack", "merge", "square", "repackconv", "linear")


class Program:
    """The general stage driver (hegpu_prog, csrc/program.cpp): lower() +
    execute() (proj/src/netcompile.cpp:106-213, 291-446) with SubConv groups,
    grouped merges, RepackConv and the HS / LoLa-dense policies."""

    def __init__(self, ctx, model, weights):
        self.ctx, self.model = ctx, model
        w = np.ascontiguousarray(weights, dtype=np.float64)
        h = C.c_void_p()
        rc = lib().hegpu_prog_create(ctx.h, model.h, w, w.size, C.byref(h))
        if rc:
            msg = lib().hegpu_prog_last_error(None)
            raise _ERR.get(rc, HegpuError)(rc, msg.decode() if msg else "")
        self.h = h
        v = [C.c_int() for _ in range(4)]
        self._check(lib().hegpu_prog_info(h, *[C.byref(x) for x in v]))
        self.n_stages, self.input_cts, self.out_level, self.n_logits = (x.value for x in v)
        self.top = ctx.L
        self.stages = []
        for k in range(self.n_stages):
            buf = C.create_string_buffer(64)
            kind, groups, pol = C.c_int(), C.c_int(), C.c_int()
            self._check(lib().hegpu_prog_stage(h, k, buf, 64, C.byref(kind), C.byref(groups), C.byref(pol)))
            self.stages.append({"label": buf.value.decode(), "kind": STAGE_KINDS[kind.value],
                                "groups": groups.value, "policy": POLICIES[pol.value]})

    def _check(self, rc):
        if rc:
            msg = lib().hegpu_prog_last_error(self.h)
            raise _ERR.get(rc, HegpuError)(rc, msg.decode() if msg else "")

    @property
    def out_scale(self):
        return lib().hegpu_prog_output_scale(self.h)

    def encrypt_input(self, image, nonce):
        x = np.ascontiguousarray(image, dtype=np.float64).ravel()
        out = np.empty(self.input_cts * 2 * self.top * self.ctx.N, dtype=np.uint64)
        self._check(lib().hegpu_prog_encrypt_input(self.h, x, nonce, out))
        return out

    def run(self, input_ct, out_ct):
        self._check(lib().hegpu_prog_run(self.h, input_ct.h, out_ct.h))

    def decrypt_logits(self, out_ct_words):
        w = np.ascontiguousarray(out_ct_words, dtype=np.uint64)
        out = np.empty(self.n_logits, dtype=np.float64)
        self._check(lib().hegpu_prog_decrypt_logits(self.h, w, out))
        return out

    def __del__(self):
        try:
            if _ctx_alive(self) and getattr(self, "h", None):
                lib().hegpu_prog_destroy(self.h)
        except Exception:
            pass


SPLIT_FIRST_LAYER = -1  # hegpu_net_run_split: split Conv1 + Flat1 by output map


def split_first_and_dense(k):
    """hegpu_net_run_split layer code: the first layer and dense layer k"""
    return -2 - k


class Net:
    """Stage driver (execute, proj/src/netcompile.cpp:291-446) for the
    Conv -> (Square -> Dense)* family on a batch of images."""

    def __init__(self, ctx, cfg, weights, first_layer="reference"):
        """first_layer: "reference" (k^2 c_in conv_pack taps, per-map conv +
        rescale, merge_maps with c_out - 1 key switches; the reference's
        stages) or "fused" (region-packed replicated taps)"""
        self.ctx, self.cfg = ctx, cfg
        spec = NetSpec()
        spec.in_c, spec.in_d, spec.k, spec.stride, spec.c_out = cfg.in_c, cfg.in_d, cfg.k, cfg.s, cfg.c_out
        spec.first_layer = FIRST_LAYERS[first_layer]
        spec.n_dense = len(cfg.dense)
        for k, m in enumerate(cfg.dense):
            spec.dense_out[k] = m
        self._keep = [np.ascontiguousarray(W, dtype=np.float64) for W, _ in weights["dense"]]
        self._keepb = [np.ascontiguousarray(b, dtype=np.float64) for _, b in weights["dense"]]
        wp = (C.c_void_p * 4)(*[a.ctypes.data for a in self._keep])
        bp = (C.c_void_p * 4)(*[a.ctypes.data for a in self._keepb])
        cw = np.ascontiguousarray(weights["conv_w"], dtype=np.float64).ravel()
        cb = np.ascontiguousarray(weights["conv_b"], dtype=np.float64)
        h = C.c_void_p()
        ctx.check(lib().hegpu_net_create(ctx.h, C.byref(spec), cw, cb, C.cast(wp, C.c_void_p),
                                         C.cast(bp, C.c_void_p), C.byref(h)))
        self.h = h
        self._post_init()

    def _post_init(self):
        h, ctx = self.h, self.ctx
        self.tap_cts = int(lib().hegpu_net_tap_cts(h))  # tap ciphertexts per image
        self.ntaps = self.tap_cts  # (round-1 name)
        self.first_layer = {v: k for k, v in FIRST_LAYERS.items()}[int(lib().hegpu_net_first_layer(h))]
        self.top = ctx.L
        self.out_level = ctx.L - 1 - 2 * len(self.cfg.dense)
        self.tap_words = 2 * self.top * ctx.N
        self.out_words = 2 * self.out_level * ctx.N

    @classmethod
    def from_model(cls, ctx, model, weights_path):
        """hegpu_net_create_from_model: the model's conv / square / dense
        stack with its float32 weights file"""
        spec = model.net_spec()
        h = C.c_void_p()
        ctx.check(lib().hegpu_net_create_from_model(ctx.h, model.h, str(weights_path).encode(), C.byref(h)))
        self = cls.__new__(cls)
        self.ctx = ctx
        self.cfg = _SpecCfg(spec)
        self.h = h
        self._post_init()
        return self

    def encrypt_image(self, image, nonce):
        out = np.empty(self.ntaps * self.tap_words, dtype=np.uint64)
        self.ctx.check(lib().hegpu_net_encrypt_image(self.h, np.ascontiguousarray(image, dtype=np.float64).ravel(),
                                                     nonce, out))
        return out

    def run(self, taps_ct, out_ct):
        self.ctx.check(lib().hegpu_net_run(self.h, taps_ct.h, out_ct.h))
        return out_ct

    def run_split(self, taps_ct, out_ct, layer, part, nparts, reduce):
        """hegpu_net_run_split: dense layer `layer`'s HS over diagonal range
        `part` of `nparts` (layer = SPLIT_FIRST_LAYER: the conv + merge of
        output maps share `part`); reduce(t) receives the partial
        accumulator as a CUDA int64 tensor view and must sum it over all
        parts in place"""
        import torch

        def cb(ptr, words, _user):
            try:
                t = torch.as_tensor(_DevWords(ptr, words), device="cuda")
                reduce(t)
                torch.cuda.synchronize()
                return 0
            except Exception:  # reported as a failed reduction by the library
                return 1

        fn = REDUCE_FN(cb)
        self.ctx.check(lib().hegpu_net_run_split(self.h, taps_ct.h, out_ct.h, layer, part, nparts, fn, None))
        return out_ct

    def run_compact(self, dev_taps, batch, out_ct):
        """device-resident compact taps (a CUDA tensor / device pointer)"""
        ptr = dev_taps if isinstance(dev_taps, int) else dev_taps.data_ptr()
        self.ctx.check(lib().hegpu_net_run_compact(self.h, ptr, batch, out_ct.h))
        return out_ct

    def run_host(self, host_taps, batch, host_out):
        """host_taps / host_out: numpy or pinned torch buffers (.ctypes.data / data_ptr)."""
        pi = host_taps.ctypes.data if isinstance(host_taps, np.ndarray) else host_taps.data_ptr()
        po = host_out.ctypes.data if isinstance(host_out, np.ndarray) else host_out.data_ptr()
        self.ctx.check(lib().hegpu_net_run_host(self.h, pi, batch, po))

    @property
    def compact_image_bytes(self):
        return int(lib().hegpu_net_compact_image_bytes(self.h))

    def encrypt_image_compact(self, image, nonce):
        out = np.empty(self.compact_image_bytes, dtype=np.uint8)
        self.ctx.check(lib().hegpu_net_encrypt_image_compact(
            self.h, np.ascontiguousarray(image, dtype=np.float64).ravel(), nonce, out.ctypes.data))
        return out

    def run_host_compact(self, host_taps, batch, host_out, chunk=0):
        """compact taps (uint8, pinned or numpy) -> output wire cts; pipelined chunks"""
        pi = host_taps.ctypes.data if isinstance(host_taps, np.ndarray) else host_taps.data_ptr()
        po = host_out.ctypes.data if isinstance(host_out, np.ndarray) else host_out.data_ptr()
        self.ctx.check(lib().hegpu_net_run_host_compact(self.h, pi, batch, chunk, po))

    def submit_host_compact(self, host_taps, batch, host_out, chunk=0):
        """as run_host_compact without waiting (buffers must outlive wait())"""
        pi = host_taps.ctypes.data if isinstance(host_taps, np.ndarray) else host_taps.data_ptr()
        po = host_out.ctypes.data if isinstance(host_out, np.ndarray) else host_out.data_ptr()
        self.ctx.check(lib().hegpu_net_submit_host_compact(self.h, pi, batch, chunk, po))

    def wait(self):
        self.ctx.check(lib().hegpu_net_wait(self.h))

    def decrypt_logits(self, out_ct):
        m = self.cfg.dense[-1]
        out = np.empty(m, dtype=np.float64)
        self.ctx.check(lib().hegpu_net_decrypt_logits(self.h, np.ascontiguousarray(out_ct, dtype=np.uint64), out))
        return out

    def __del__(self):
        try:
            if self.h and _ctx_alive(self):
                lib().hegpu_net_destroy(self.h)
                self.h = None
        except Exception:
            pass
