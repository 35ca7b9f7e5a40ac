// modarith.cuh -- 64-bit RNS modular arithmetic for sm_100a.
//
// Primes are < 2^61 (an 8-way uint64 sum cannot overflow), so
// lazy values in [0, 4q) fit a word.  Three multipliers:
//   shoup_mul  constant operand with precomputed w' = floor(w 2^64 / q)
//              (NTT twiddles, N^{-1}, P^{-1}): 1 mul.hi + 2 mul.lo;
//   mont_mul   a * b * 2^-64 (keys, masks and plaintexts are stored in
//              Montgomery form, so mont_mul(x, y_mont) = x*y mod q);
//   mont_reduce128  one Montgomery reduction of a 128-bit accumulator, used
//              to fold a sum of products with a single reduction.
#pragma once
#include <cstdint>

namespace hegpu {

typedef unsigned long long u64d;

struct DevPrime {
  u64d q;
  u64d qneg_inv;  // -q^{-1} mod 2^64
  u64d r_mod;     // 2^64 mod q (to_mont of 1; reduce via mont_mul(x, r_mod))
  u64d r2_mod;    // 2^128 mod q
  u64d one_sh;    // floor(2^64 / q): Shoup companion of 1 (lazy x mod q)
};

#define HEGPU_MAX_PRIMES 16

struct PrimeTable {
  DevPrime p[HEGPU_MAX_PRIMES];
};

__device__ __forceinline__ u64d mulhi64(u64d a, u64d b) { return __umul64hi(a, b); }

__device__ __forceinline__ u64d add_mod_d(u64d a, u64d b, u64d q) {
  u64d s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ u64d sub_mod_d(u64d a, u64d b, u64d q) {
  return a >= b ? a - b : a + q - b;
}
__device__ __forceinline__ u64d shoup_mul_d(u64d a, u64d w, u64d wp, u64d q) {
  u64d h = mulhi64(a, wp);
  u64d r = a * w - h * q;
  return r >= q ? r - q : r;
}
// result in [0, 2q) (Harvey lazy form)
__device__ __forceinline__ u64d shoup_mul_lazy(u64d a, u64d w, u64d wp, u64d q) {
  u64d h = mulhi64(a, wp);
  return a * w - h * q;
}
__device__ __forceinline__ u64d mont_mul(u64d a, u64d b, u64d q, u64d qneg) {
  u64d lo = a * b, hi = mulhi64(a, b);
  u64d m = lo * qneg;
  u64d r = hi + mulhi64(m, q) + (lo != 0ull);
  return r >= q ? r - q : r;
}
// 128-bit accumulator (hi:lo) < q * 2^64  ->  (hi:lo) * 2^-64 mod q
__device__ __forceinline__ u64d mont_reduce128(u64d lo, u64d hi, u64d q, u64d qneg) {
  u64d m = lo * qneg;
  u64d r = hi + mulhi64(m, q) + (lo != 0ull);
  return r >= q ? r - q : r;
}
// 128-bit multiply-accumulate
__device__ __forceinline__ void mac128(u64d& lo, u64d& hi, u64d a, u64d b) {
  u64d pl = a * b, ph = mulhi64(a, b);
  lo += pl;
  hi += ph + (lo < pl);
}
// reduce any 64-bit value mod q: mont_mul(x, 2^64 mod q) = x mod q
__device__ __forceinline__ u64d reduce64(u64d x, const DevPrime& p) {
  return mont_mul(x, p.r_mod, p.q, p.qneg_inv);
}

// Shoup product with an approximate quotient: the high word of a * w' is
// formed from the three leading 32x32 partial products only (3 IMAD.WIDE
// instead of a full 64x64 high product), so the quotient is low by at most
// 2 and the result lies in [0, 4q) for any a < 2^64 (q < 2^61).
//
// The remainder a*w - h*q is formed as a*w + h*(2^64 - q) mod 2^64 from
// 32-bit partial products: the two low products accumulate in one 64-bit
// IMAD.WIDE chain and the four cross products go straight into the high
// word (6 multiply instructions, no separate 64-bit subtraction; the
// compiler's 64-bit a*w - h*q took ~11.5 SASS per call, ncu source view).
__device__ __forceinline__ u64d shoup_mul_lazy4(u64d a, u64d w, u64d wp, u64d q) {
  const uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32);
  const uint32_t p0 = (uint32_t)wp, p1 = (uint32_t)(wp >> 32);
  const u64d nq = 0ull - q;
  u64d r;
  asm("{\n\t.reg .u64 t1, t2, h;\n\t"
      ".reg .u32 h0, h1, rl, rh;\n\t"
      "mul.wide.u32 t1, %1, %3;\n\t"   // a1 * w0'
      "mul.wide.u32 t2, %2, %4;\n\t"   // a0 * w1'
      "shr.u64 t1, t1, 32;\n\t"
      "shr.u64 t2, t2, 32;\n\t"
      "add.u64 t1, t1, t2;\n\t"
      "mad.wide.u32 h, %1, %4, t1;\n\t"  // h ~ (a * w') >> 64
      "mov.b64 {h0, h1}, h;\n\t"
      "mul.wide.u32 t1, %2, %5;\n\t"     // a0 * w0
      "mad.wide.u32 t1, h0, %7, t1;\n\t" // + h0 * nq0
      "mov.b64 {rl, rh}, t1;\n\t"
      "mad.lo.u32 rh, %2, %6, rh;\n\t"   // + a0 * w1 << 32
      "mad.lo.u32 rh, %1, %5, rh;\n\t"   // + a1 * w0 << 32
      "mad.lo.u32 rh, h0, %8, rh;\n\t"   // + h0 * nq1 << 32
      "mad.lo.u32 rh, h1, %7, rh;\n\t"   // + h1 * nq0 << 32
      "mov.b64 %0, {rl, rh};\n\t"
      "}"
      : "=l"(r)
      : "r"(a1), "r"(a0), "r"(p0), "r"(p1), "r"((uint32_t)w), "r"((uint32_t)(w >> 32)), "r"((uint32_t)nq),
        "r"((uint32_t)(nq >> 32)));
  return r;
}

// a >= m ? a - m : a with the borrow of the 64-bit subtraction selecting
// through LOP3 (5 SASS instead of 2 compares + 2 selects + subtraction)
__device__ __forceinline__ u64d csub64(u64d a, u64d m) {
  u64d r;
  asm("{\n\t.reg .u32 a0, a1, m0, m1, d0, d1, b;\n\t"
      "mov.b64 {a0, a1}, %1;\n\t"
      "mov.b64 {m0, m1}, %2;\n\t"
      "sub.cc.u32 d0, a0, m0;\n\t"
      "subc.cc.u32 d1, a1, m1;\n\t"
      "subc.u32 b, 0, 0;\n\t"                // all ones iff a < m
      "lop3.b32 d0, a0, d0, b, 0xE4;\n\t"   // b ? a : a - m
      "lop3.b32 d1, a1, d1, b, 0xE4;\n\t"
      "mov.b64 %0, {d0, d1};\n\t"
      "}"
      : "=l"(r)
      : "l"(a), "l"(m));
  return r;
}

// lazy reduction of any x < 2^64 into [0, 4q): x - floor~(x / q) q
__device__ __forceinline__ u64d reduce_lazy4(u64d x, const DevPrime& p) {
  return shoup_mul_lazy4(x, 1ull, p.one_sh, p.q);
}

// ---- 31-bit split operands for multiply-accumulate ------------------------
// A residue x < 2^61 is stored "split" as x0 | x1 << 32 with x0 = x mod 2^31,
// x1 = x >> 31 (< 2^30).  A product of two split operands is four 32x32->64
// IMAD.WIDE partial products accumulated carry-free:
//   s0 += x0 y0 (< 2^62)   s1 += x0 y1 + x1 y0 (< 2^62)   s2 += x1 y1 (< 2^60)
// so up to 4 products fit before folding into a 192-bit total.
__device__ __forceinline__ u64d split31(u64d x) { return (x & 0x7FFFFFFFull) | ((x >> 31) << 32); }
__device__ __forceinline__ u64d unsplit31(u64d s) { return (s & 0xFFFFFFFFull) + ((s >> 32) << 31); }

// (top:hi:lo) * 2^-64 mod q: h = (top 2^64 + hi) mod q, then one Montgomery
// reduction of (h:lo).  top is 0 unless a sum of > 8 products of 61-bit
// operands carried past 2^128 (the rare path).
__device__ __forceinline__ u64d reduce192(u64d lo, u64d hi, uint32_t top, const DevPrime& pr) {
  u64d h;
  if (top) h = mont_mul(mont_reduce128(hi, (u64d)top, pr.q, pr.qneg_inv), pr.r2_mod, pr.q, pr.qneg_inv);
  else h = shoup_mul_d(hi, 1ull, pr.one_sh, pr.q);
  return mont_reduce128(lo, h, pr.q, pr.qneg_inv);
}

// 40-bit primes: operands split at 20 bits; every partial product is
// < 2^41, so hundreds of them sum carry-free in three 64-bit words and no
// fold is ever needed (AccC folds every 4 products).  Same integer total,
// same reduce192 -> bit-identical to AccC.
struct Acc20 {
  u64d s0, s1, s2;
  __device__ __forceinline__ void zero() { s0 = s1 = s2 = 0; }
  // x plain (< 2^40), ys in split31 form (< 2^40)
  __device__ __forceinline__ void mac(u64d x, u64d ys) {
    const uint32_t x0 = (uint32_t)x & 0xFFFFFu, x1 = (uint32_t)(x >> 20);
    const uint32_t yl = (uint32_t)ys, yh = (uint32_t)(ys >> 32);
    const uint32_t y0 = yl & 0xFFFFFu, y1 = (yl >> 20) | (yh << 11);
    s0 += (u64d)x0 * y0;
    s1 += (u64d)x0 * y1 + (u64d)x1 * y0;
    s2 += (u64d)x1 * y1;
  }
  // window words: staged plain (prep), multiplied by split31 operands (macw)
  __device__ __forceinline__ static u64d prep(u64d x) { return x; }
  __device__ __forceinline__ void macw(u64d x, u64d ys) { mac(x, ys); }
  __device__ __forceinline__ void fold() {}
  __device__ __forceinline__ u64d reduce(const DevPrime& pr) {
    const unsigned __int128 t = (unsigned __int128)s0 + ((unsigned __int128)s1 << 20) + ((unsigned __int128)s2 << 40);
    return reduce192((u64d)t, (u64d)(t >> 64), 0u, pr);
  }
};

struct Acc3 {  // s0 + s1 2^31 + s2 2^62 (partial), folded into lo:hi:top
  u64d s0, s1, s2, lo, hi;
  uint32_t top;
  __device__ __forceinline__ void zero() { s0 = s1 = s2 = lo = hi = 0; top = 0; }
  __device__ __forceinline__ void mad(u64d xs, u64d ys) {
    const uint32_t x0 = (uint32_t)xs, x1 = (uint32_t)(xs >> 32);
    const uint32_t y0 = (uint32_t)ys, y1 = (uint32_t)(ys >> 32);
    asm("mad.wide.u32 %0, %3, %5, %0;\n\t"
        "mad.wide.u32 %1, %3, %6, %1;\n\t"
        "mad.wide.u32 %1, %4, %5, %1;\n\t"
        "mad.wide.u32 %2, %4, %6, %2;\n\t"
        : "+l"(s0), "+l"(s1), "+l"(s2)
        : "r"(x0), "r"(x1), "r"(y0), "r"(y1));
  }
  __device__ __forceinline__ void fold() {
    // (an __int128 formulation measured 9% slower on the HS kernel)
    const u64d l1 = s1 << 31, h1 = s1 >> 33, l2 = s2 << 62, h2 = s2 >> 2;
    asm("add.cc.u64 %0, %0, %3;\n\t"
        "addc.cc.u64 %1, %1, 0;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        "add.cc.u64 %0, %0, %4;\n\t"
        "addc.cc.u64 %1, %1, %5;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        "add.cc.u64 %0, %0, %6;\n\t"
        "addc.cc.u64 %1, %1, %7;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        : "+l"(lo), "+l"(hi), "+r"(top)
        : "l"(s0), "l"(l1), "l"(h1), "l"(l2), "l"(h2));
    s0 = s1 = s2 = 0;
  }
  // (top:hi:lo) * 2^-64 mod q  (products of standard x Montgomery operands)
  __device__ __forceinline__ u64d reduce(const DevPrime& pr) {
    fold();
    return reduce192(lo, hi, top, pr);
  }
};

struct AccC {  // as Acc3; s0 + s1 2^31 + s2 2^62 kept as 32-bit halves
  // the PTX carry chains below (mad.lo.cc + madc.hi per product) become one
  // accumulating IMAD.WIDE.U32 per product, where Acc3's 64-bit mad.wide
  // chains are re-associated by ptxas into products plus IADD3 trees (14.3 ->
  // 10.6 SASS per MAC in the HS loop).  Costs registers: used by the HS and
  // conv kernels; the key-switch inner products keep Acc3 (profiles/r01_notes.md)
  uint32_t a0l, a0h, a1l, a1h, a2l, a2h;
  u64d lo, hi;
  uint32_t top;
  __device__ __forceinline__ void zero() {
    a0l = a0h = a1l = a1h = a2l = a2h = 0;
    lo = hi = 0;
    top = 0;
  }
  __device__ __forceinline__ void mad(u64d xs, u64d ys) {
    const uint32_t x0 = (uint32_t)xs, x1 = (uint32_t)(xs >> 32);
    const uint32_t y0 = (uint32_t)ys, y1 = (uint32_t)(ys >> 32);
    asm("mad.lo.cc.u32 %0, %6, %8, %0;\n\t"
        "madc.hi.u32 %1, %6, %8, %1;\n\t"
        "mad.lo.cc.u32 %2, %6, %9, %2;\n\t"
        "madc.hi.u32 %3, %6, %9, %3;\n\t"
        "mad.lo.cc.u32 %2, %7, %8, %2;\n\t"
        "madc.hi.u32 %3, %7, %8, %3;\n\t"
        "mad.lo.cc.u32 %4, %7, %9, %4;\n\t"
        "madc.hi.u32 %5, %7, %9, %5;\n\t"
        : "+r"(a0l), "+r"(a0h), "+r"(a1l), "+r"(a1h), "+r"(a2l), "+r"(a2h)
        : "r"(x0), "r"(x1), "r"(y0), "r"(y1));
  }
  __device__ __forceinline__ void mac(u64d x, u64d ys) { mad(split31(x), ys); }
  __device__ __forceinline__ static u64d prep(u64d x) { return split31(x); }
  __device__ __forceinline__ void macw(u64d xs, u64d ys) { mad(xs, ys); }
  __device__ __forceinline__ void fold() {
    // (an __int128 formulation measured 9% slower on the HS kernel)
    const u64d s0 = ((u64d)a0h << 32) | a0l, s1 = ((u64d)a1h << 32) | a1l, s2 = ((u64d)a2h << 32) | a2l;
    const u64d l1 = s1 << 31, h1 = s1 >> 33, l2 = s2 << 62, h2 = s2 >> 2;
    asm("add.cc.u64 %0, %0, %3;\n\t"
        "addc.cc.u64 %1, %1, 0;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        "add.cc.u64 %0, %0, %4;\n\t"
        "addc.cc.u64 %1, %1, %5;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        "add.cc.u64 %0, %0, %6;\n\t"
        "addc.cc.u64 %1, %1, %7;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        : "+l"(lo), "+l"(hi), "+r"(top)
        : "l"(s0), "l"(l1), "l"(h1), "l"(l2), "l"(h2));
    a0l = a0h = a1l = a1h = a2l = a2h = 0;
  }
  // (top:hi:lo) * 2^-64 mod q  (products of standard x Montgomery operands)
  __device__ __forceinline__ u64d reduce(const DevPrime& pr) {
    fold();
    return reduce192(lo, hi, top, pr);
  }
};

// Wide-limb accumulator: each partial sum (s0, s1, s2 as in Acc3) is kept in
// three 32-bit words and every product's carry is propagated at once
// (mad.lo.cc / madc.hi.cc / addc), so nothing is folded inside the loop
// (capacity 2^34 products); the 192-bit total is formed once in reduce().
struct AccW {
  uint32_t a[3], b[3], c[3];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < 3; ++i) a[i] = b[i] = c[i] = 0;
  }
  __device__ __forceinline__ void mad(u64d xs, u64d ys) {
    const uint32_t x0 = (uint32_t)xs, x1 = (uint32_t)(xs >> 32);
    const uint32_t y0 = (uint32_t)ys, y1 = (uint32_t)(ys >> 32);
    asm("mad.lo.cc.u32 %0, %9, %11, %0;\n\t"
        "madc.hi.cc.u32 %1, %9, %11, %1;\n\t"
        "addc.u32 %2, %2, 0;\n\t"
        "mad.lo.cc.u32 %3, %9, %12, %3;\n\t"
        "madc.hi.cc.u32 %4, %9, %12, %4;\n\t"
        "addc.u32 %5, %5, 0;\n\t"
        "mad.lo.cc.u32 %3, %10, %11, %3;\n\t"
        "madc.hi.cc.u32 %4, %10, %11, %4;\n\t"
        "addc.u32 %5, %5, 0;\n\t"
        "mad.lo.cc.u32 %6, %10, %12, %6;\n\t"
        "madc.hi.cc.u32 %7, %10, %12, %7;\n\t"
        "addc.u32 %8, %8, 0;\n\t"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(c[0]), "+r"(c[1]),
          "+r"(c[2])
        : "r"(x0), "r"(x1), "r"(y0), "r"(y1));
  }
  __device__ __forceinline__ static u64d prep(u64d x) { return split31(x); }
  __device__ __forceinline__ void macw(u64d xs, u64d ys) { mad(xs, ys); }
  __device__ __forceinline__ void fold() {}  // nothing to fold
  // s0 + s1 2^31 + s2 2^62 (each < 2^96) -> lo:hi:top, then as Acc3::reduce
  __device__ __forceinline__ u64d reduce(const DevPrime& pr) {
    u64d lo = 0, hi = 0;
    uint32_t top = 0;
    auto add_shifted = [&](const uint32_t (&v)[3], int sh) {
      const u64d v0 = ((u64d)v[1] << 32) | v[0], v1 = v[2];
      const u64d l = sh ? v0 << sh : v0;
      const u64d m = sh ? (v0 >> (64 - sh)) | (v1 << sh) : v1;
      const uint32_t t = sh ? (uint32_t)(v1 >> (64 - sh)) : 0u;
      asm("add.cc.u64 %0, %0, %3;\n\t"
          "addc.cc.u64 %1, %1, %4;\n\t"
          "addc.u32 %2, %2, %5;\n\t"
          : "+l"(lo), "+l"(hi), "+r"(top)
          : "l"(l), "l"(m), "r"(t));
    };
    add_shifted(a, 0);
    add_shifted(b, 31);
    add_shifted(c, 62);
    u64d x = mont_reduce128(hi, (u64d)top, pr.q, pr.qneg_inv);
    x = mont_mul(x, pr.r2_mod, pr.q, pr.qneg_inv);
    const u64d y = mont_reduce128(lo, 0ull, pr.q, pr.qneg_inv);
    return add_mod_d(x, y, pr.q);
  }
};

}  // namespace hegpu
