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

}  // namespace hegpu
