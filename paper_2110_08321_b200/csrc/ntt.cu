// ntt.cu -- batched negacyclic NTT / INTT over 64-bit primes (sm_100a).
//
// One CTA transforms one N-word limb (2^5 <= N <= 2^14) held in shared
// memory.  Each thread keeps R = 16 words in registers and runs up to 4
// radix-2 stages per pass on them (Cooley-Tukey forward with psi powers in
// bit-reversed order, Gentleman-Sande inverse), so an N = 8192 transform is
// 4 register passes with 3 shared-memory exchanges instead of 13
// stage-synchronous sweeps.  The pass schedule is resolved at compile time
// per log2 N.  Butterflies are Harvey-lazy (values in [0, 4q), Shoup twiddle
// products in [0, 2q)); primes < 2^61 keep 4q in a word.  Twiddles are
// (w, w') pairs read as one 16-byte load.
//
// Loads and stores are functors so every limb crosses HBM once per
// transform with the surrounding RNS step fused in:
//   forward : store scatters to the device SLOT ORDER (engine.hpp);
//             ModUp loads reduce a digit mod the target prime;
//             drop-limb (rescale / ModDown) loads lift the dropped residue
//             and the store finishes (x - X) * q_d^{-1} (+ add term);
//   inverse : key-switch loads apply the Galois shift and emit the shifted
//             own-prime limb for ModUp; stores multiply by N^{-1}.
#include <cooperative_groups.h>

#include "engine.hpp"

namespace hegpu {

namespace {

// registers per thread: R = 2^lr words.  R = 16 measured faster than R = 32
// on B200 (2 CTAs x 512 threads per SM for N = 2^13 beat 2 x 256 threads
// with 128 registers each; profiles/r01_notes.md)
#ifndef HEGPU_NTT_LR13
#define HEGPU_NTT_LR13 4
#endif
__host__ __device__ constexpr int lr_of(int logn) { return logn <= 13 ? HEGPU_NTT_LR13 : 4; }
constexpr int kMinLogN = 5, kMaxLogN = 15;
// N = 2^15 (FP64-only builds): one row is split over the two CTAs of a
// thread-block cluster, each transforming 2^14 words in its own shared
// memory.  Forward: both CTAs read the whole row, apply the first
// Cooley-Tukey stage while loading (CTA h keeps a + (-1)^h w b) and run the
// remaining 14 stages as an independent sub-transform whose twiddles are
// the full table's, indexed (2 + h) 2^s + i; its outputs are exactly slot
// positions [h S, (h + 1) S) (params.cpp: p < S <-> exponent = 1 mod 4 <->
// bit-reversed index < N / 2).  Inverse: 14 Gentleman-Sande stages per CTA,
// then the last stage pairs the two halves through distributed shared
// memory (cluster.map_shared_rank).
__host__ __device__ constexpr int sub_logn(int logn) { return logn > 14 ? 14 : logn; }
// HEGPU_NTT_PRIME_MAJOR=1 launches the rows prime-major (the prime index from
// the slow part of the launch index, so co-resident CTAs share one 64 KB
// twiddle table in L1).  Measured on cfg 2: no gain (3.134 vs 3.116 ms per
// step; the digit re-reads spread over the launch cost what the table hits
// save), so rows stay row-major (profiles/r02_notes.md).
#ifndef HEGPU_NTT_PRIME_MAJOR
#define HEGPU_NTT_PRIME_MAJOR 0
#endif
template <int LOGN>
struct RowCta {  // which row, which half of it, and the half's first position / index
  static constexpr int NT = 1 << sub_logn(LOGN);
  int r, h, base, rows;
  __device__ __forceinline__ RowCta() {
    if constexpr (LOGN > 14) {
      r = (int)(blockIdx.x >> 1);
      h = (int)(blockIdx.x & 1);
      rows = (int)(gridDim.x >> 1);
    } else {
      r = (int)blockIdx.x;
      h = 0;
      rows = (int)gridDim.x;
    }
    base = h * NT;
  }
  // split the launch index into (outer, fast) with `nfast` values of the fast
  // (prime) part: row-major outer * nfast + fast, or prime-major
  __device__ __forceinline__ int split(int nfast, int& fast) const {
#if HEGPU_NTT_PRIME_MAJOR
    const int nouter = rows / nfast;
    fast = r / nouter;
    return r - fast * nouter;
#else
    fast = r % nfast;
    return r / nfast;
#endif
  }
};

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }

__device__ __forceinline__ int shifted(int p, int s, int S) {
  const int h = p >= S ? S : 0;
  int j = p - h + s;
  if (j >= S) j -= S;
  return h + j;
}

__host__ __device__ constexpr int cmin(int a, int b) { return a < b ? a : b; }

struct TwArgs {
  const ulonglong2* tw;   // [np][2][N] (w, w') forward then inverse
  const u64d* ninv;       // [np][2]
  const uint32_t* slot_src;
  const double* twd;      // [np][2][N] w as doubles (FP64 butterflies)
  const double2* fpq;     // [np] (q, 1/q) for primes on the FP64 path, (0, 0) otherwise
};

// ------------------------------------------------------------------ forward
// Pass of RR stages starting at stage S0: thread element e = g * 2^RR + j sits
// at index hi * 2^(LOGN - S0) + j * 2^LOB + lo (LOB = LOGN - S0 - RR), where
// group grp = g * T + tid splits into (hi, lo).
template <int LOGN, int S0, int RR>
__device__ __forceinline__ int fwd_idx(int g, int j) {
  constexpr int T = (1 << LOGN) / (1 << lr_of(LOGN)), LOB = LOGN - S0 - RR;
  const int grp = g * T + (int)threadIdx.x;
  return ((grp >> LOB) << (LOGN - S0)) + (j << LOB) + (grp & ((1 << LOB) - 1));
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void fwd_pass(u64d (&x)[1 << lr_of(LOGN)], const ulonglong2* __restrict__ tw, u64d q) {
  constexpr int T = (1 << LOGN) / (1 << lr_of(LOGN)), G = (1 << lr_of(LOGN)) >> RR, J = 1 << RR, LOB = LOGN - S0 - RR;
  const u64d q4 = 4 * q;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int hi = (g * T + (int)threadIdx.x) >> LOB;
#pragma unroll
    for (int u = 0; u < RR; ++u) {
      const int half = J >> (u + 1);
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (j & half) continue;
        const ulonglong2 W = __ldg(tw + (1 << (S0 + u)) + (hi << u) + (j >> (RR - u)));
        // values in [0, 8q) (q < 2^60): one conditional subtraction per butterfly
        u64d a = x[g * J + j];
#ifdef HEGPU_CSUB_LOP3
        a = csub64(a, q4);
#else
        if (a >= q4) a -= q4;
#endif
        const u64d t = shoup_mul_lazy4(x[g * J + j + half], W.x, W.y, q);  // [0, 4q)
        x[g * J + j] = a + t;
        x[g * J + j + half] = a - t + q4;
      }
    }
  }
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void fwd_store(u64d* sm, const u64d (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) sm[pad(fwd_idx<LOGN, S0, RR>(g, j))] = x[g * (1 << RR) + j];
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void fwd_load(const u64d* sm, u64d (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) x[g * (1 << RR) + j] = sm[pad(fwd_idx<LOGN, S0, RR>(g, j))];
}

template <int LOGN, int S0>
__device__ __forceinline__ void fwd_passes(u64d (&x)[1 << lr_of(LOGN)], u64d* sm, const ulonglong2* tw, u64d q) {
  constexpr int RR = cmin(lr_of(LOGN), LOGN - S0);
  fwd_pass<LOGN, S0, RR>(x, tw, q);
  if constexpr (S0 + RR < LOGN) {
    constexpr int RN = cmin(lr_of(LOGN), LOGN - S0 - RR);
    fwd_store<LOGN, S0, RR>(sm, x);
    __syncthreads();
    fwd_load<LOGN, S0 + RR, RN>(sm, x);
    __syncthreads();
    fwd_passes<LOGN, S0 + RR>(x, sm, tw, q);
  } else {
    const u64d q2 = 2 * q, q4 = 4 * q;
#pragma unroll
    for (int e = 0; e < (1 << lr_of(LOGN)); ++e) {  // [0, 8q) -> [0, q)
      u64d v = x[e];
      if (v >= q4) v -= q4;
      if (v >= q2) v -= q2;
      if (v >= q) v -= q;
      x[e] = v;
    }
    fwd_store<LOGN, S0, RR>(sm, x);
    __syncthreads();
  }
}

// forward NTT of the row `ld` describes; result in smem (padded, canonical,
// bit-reversed index order), CTA synchronised on return
template <int LOGN, class Ld>
__device__ __forceinline__ void fwd_transform(u64d* sm, const Ld& ld, const ulonglong2* tw, u64d q) {
  constexpr int R0 = cmin(lr_of(LOGN), LOGN);
  u64d x[1 << lr_of(LOGN)];
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> R0); ++g)
#pragma unroll
    for (int j = 0; j < (1 << R0); ++j) x[g * (1 << R0) + j] = ld.load(fwd_idx<LOGN, 0, R0>(g, j));
  fwd_passes<LOGN, 0>(x, sm, tw, q);
}

// ------------------------------------------------------------------ inverse
// GS pass of RR stages starting at inverse stage S0 (distance 2^S0): element
// e = g * 2^RR + j sits at hi * 2^(S0 + RR) + j * 2^S0 + lo.
template <int LOGN, int S0, int RR>
__device__ __forceinline__ int inv_idx(int g, int j) {
  constexpr int T = (1 << LOGN) / (1 << lr_of(LOGN));
  const int grp = g * T + (int)threadIdx.x;
  return ((grp >> S0) << (S0 + RR)) + (j << S0) + (grp & ((1 << S0) - 1));
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void inv_pass(u64d (&x)[1 << lr_of(LOGN)], const ulonglong2* __restrict__ tw, u64d q) {
  constexpr int T = (1 << LOGN) / (1 << lr_of(LOGN)), G = (1 << lr_of(LOGN)) >> RR, J = 1 << RR;
  const u64d q4 = 4 * q;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int hi = (g * T + (int)threadIdx.x) >> S0;
#pragma unroll
    for (int u = 0; u < RR; ++u) {
      const int dist = 1 << u;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (j & dist) continue;
        const ulonglong2 W = __ldg(tw + (1 << (LOGN - S0 - u - 1)) + (hi << (RR - u - 1)) + (j >> (u + 1)));
        // values in [0, 4q): one conditional subtraction per butterfly
        const u64d a = x[g * J + j], b = x[g * J + j + dist];
        u64d s = a + b;
#ifdef HEGPU_CSUB_LOP3
        s = csub64(s, q4);
#else
        if (s >= q4) s -= q4;
#endif
        x[g * J + j] = s;
        x[g * J + j + dist] = shoup_mul_lazy4(a - b + q4, W.x, W.y, q);  // [0, 4q)
      }
    }
  }
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void inv_store(u64d* sm, const u64d (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) sm[pad(inv_idx<LOGN, S0, RR>(g, j))] = x[g * (1 << RR) + j];
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void inv_load(const u64d* sm, u64d (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) x[g * (1 << RR) + j] = sm[pad(inv_idx<LOGN, S0, RR>(g, j))];
}

template <int LOGN, int S0, class St>
__device__ __forceinline__ void inv_passes(u64d (&x)[1 << lr_of(LOGN)], u64d* sm, const ulonglong2* tw, u64d q, u64d nv,
                                           u64d nvp, St& st) {
  constexpr int RR = cmin(lr_of(LOGN), LOGN - S0);
  inv_pass<LOGN, S0, RR>(x, tw, q);
  if constexpr (S0 + RR < LOGN) {
    constexpr int RN = cmin(lr_of(LOGN), LOGN - S0 - RR);
    __syncthreads();
    inv_store<LOGN, S0, RR>(sm, x);
    __syncthreads();
    inv_load<LOGN, S0 + RR, RN>(sm, x);
    inv_passes<LOGN, S0 + RR>(x, sm, tw, q, nv, nvp, st);
  } else {
#pragma unroll
    for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
      for (int j = 0; j < (1 << RR); ++j)
        st.store(inv_idx<LOGN, S0, RR>(g, j), shoup_mul_d(x[g * (1 << RR) + j], nv, nvp, q));
  }
}

// inverse NTT: input already scattered into smem (bit-reversed index order,
// canonical) and synchronised; st.store(k, v) receives N^{-1} * INTT.
template <int LOGN, class St>
__device__ __forceinline__ void inv_transform(u64d* sm, St& st, const ulonglong2* tw, u64d q, u64d nv, u64d nvp) {
  constexpr int R0 = cmin(lr_of(LOGN), LOGN);
  u64d x[1 << lr_of(LOGN)];
  inv_load<LOGN, 0, R0>(sm, x);
  inv_passes<LOGN, 0>(x, sm, tw, q, nv, nvp, st);
}

// ------------------------------------------------- FP64 butterflies (§5.1)
// For primes q < 2^45 (the 40-bit limbs) the transform runs on the FP64
// pipe: residues are exact integers in doubles, and a product b*w mod q is
// formed exactly from the FMA two-product --
//   hi = fl(b w), lo = b w - hi (exact, one FMA),
//   k = rint(hi / q) (one FMA against the magic 1.5 * 2^52, one add),
//   t = (hi - k q) + lo (one FMA, exact since |hi - k q| < q; one add) --
// so |t| <= 0.52 q and t == b w (mod q) exactly.  Forward (CT) values grow
// by <= 0.52 q per stage from [0, 4q): after 14 stages |x| < 12 q < 2^49, no
// lazy reductions needed; inverse (GS) sums double per stage and are
// re-centred once per register pass.  Six FP64 instructions per product
// instead of ~20 integer instructions for the 64-bit Shoup multiply, and
// the integer pipes are left to address arithmetic.  Exact modular
// arithmetic, so the limbs equal the integer path's bit for bit.
#ifndef HEGPU_NTT_FP
#define HEGPU_NTT_FP 1
#endif
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: x + kMagic - kMagic = rint(x), |x| < 2^51
constexpr double kTwo52 = 4503599627370496.0;

__device__ __forceinline__ double u2d(u64d x) {  // exact for x < 2^52
  return __dadd_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)), -kTwo52);
}
__device__ __forceinline__ u64d d2u(double r) {  // r an integer in [0, 2^52)
  return (u64d)__double_as_longlong(__dadd_rn(r, kTwo52)) & 0xFFFFFFFFFFFFFull;
}
__device__ __forceinline__ double fp_mulmod(double b, double w, double2 fq) {
  const double hi = __dmul_rn(b, w);
  const double lo = __fma_rn(b, w, -hi);
  const double k = __dadd_rn(__fma_rn(hi, fq.y, kMagic), -kMagic);
  return __dadd_rn(__fma_rn(-k, fq.x, hi), lo);
}
__device__ __forceinline__ double fp_center(double v, double2 fq) {  // -> |v| <= q/2 + eps
  const double k = __dadd_rn(__fma_rn(v, fq.y, kMagic), -kMagic);
  return __fma_rn(-k, fq.x, v);
}
__device__ __forceinline__ u64d fp_canon(double v, double2 fq) {  // -> [0, q) as a word
  double r = fp_center(v, fq);
  if (r < 0.0) r = __dadd_rn(r, fq.x);
  return d2u(r);
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void fwd_pass_fp(double (&x)[1 << lr_of(LOGN)], const double* __restrict__ tw, double2 fq,
                                            const int pre = 1) {
  constexpr int T = (1 << LOGN) / (1 << lr_of(LOGN)), G = (1 << lr_of(LOGN)) >> RR, J = 1 << RR, LOB = LOGN - S0 - RR;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int hi = (g * T + (int)threadIdx.x) >> LOB;
#pragma unroll
    for (int u = 0; u < RR; ++u) {
      const int half = J >> (u + 1);
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (j & half) continue;
        const double W = __ldg(tw + (pre << (S0 + u)) + (hi << u) + (j >> (RR - u)));
        const double a = x[g * J + j];
        const double t = fp_mulmod(x[g * J + j + half], W, fq);
        x[g * J + j] = __dadd_rn(a, t);
        x[g * J + j + half] = __dadd_rn(a, -t);
      }
    }
  }
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void fwd_store_d(double* sm, const double (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) sm[pad(fwd_idx<LOGN, S0, RR>(g, j))] = x[g * (1 << RR) + j];
}
template <int LOGN, int S0, int RR>
__device__ __forceinline__ void fwd_load_d(const double* sm, double (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) x[g * (1 << RR) + j] = sm[pad(fwd_idx<LOGN, S0, RR>(g, j))];
}

template <int LOGN, int S0>
__device__ __forceinline__ void fwd_passes_fp(double (&x)[1 << lr_of(LOGN)], u64d* sm, const double* tw, double2 fq,
                                              const int pre = 1) {
  constexpr int RR = cmin(lr_of(LOGN), LOGN - S0);
  fwd_pass_fp<LOGN, S0, RR>(x, tw, fq, pre);
  if constexpr (S0 + RR < LOGN) {
    constexpr int RN = cmin(lr_of(LOGN), LOGN - S0 - RR);
    fwd_store_d<LOGN, S0, RR>(reinterpret_cast<double*>(sm), x);
    __syncthreads();
    fwd_load_d<LOGN, S0 + RR, RN>(reinterpret_cast<const double*>(sm), x);
    __syncthreads();
    fwd_passes_fp<LOGN, S0 + RR>(x, sm, tw, fq, pre);
  } else {
#pragma unroll
    for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
      for (int j = 0; j < (1 << RR); ++j) sm[pad(fwd_idx<LOGN, S0, RR>(g, j))] = fp_canon(x[g * (1 << RR) + j], fq);
    __syncthreads();
  }
}

template <int LOGN, class Ld>
__device__ __forceinline__ void fwd_transform_fp(u64d* sm, const Ld& ld, const double* tw, double2 fq) {
  constexpr int R0 = cmin(lr_of(LOGN), LOGN);
  double x[1 << lr_of(LOGN)];
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> R0); ++g)
#pragma unroll
    for (int j = 0; j < (1 << R0); ++j) x[g * (1 << R0) + j] = u2d(ld.load(fwd_idx<LOGN, 0, R0>(g, j)));
  fwd_passes_fp<LOGN, 0>(x, sm, tw, fq);
}

// N = 2^15: half h of the row.  `tw` is the full 2^15 table; values stay
// below 16 q < 2^49 over the 15 stages.
template <class Ld>
__device__ __forceinline__ void fwd_transform_fp_split(u64d* sm, const Ld& ld, const double* tw, double2 fq, int h) {
  constexpr int LS = 14, R = 1 << lr_of(LS), NH = 1 << LS;
  static_assert(lr_of(LS) <= LS, "one group per thread in the first pass");
  double x[R];
  const double w1 = __ldg(tw + 1);
#pragma unroll
  for (int e = 0; e < R; ++e) {
    const int k = fwd_idx<LS, 0, lr_of(LS)>(0, e);
    const double a = u2d(ld.load(k));
    const double t = fp_mulmod(u2d(ld.load(k + NH)), w1, fq);
    x[e] = __dadd_rn(a, h ? -t : t);
  }
  fwd_passes_fp<LS, 0>(x, sm, tw, fq, 2 + h);
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void inv_pass_fp(double (&x)[1 << lr_of(LOGN)], const double* __restrict__ tw, double2 fq,
                                            const int pre = 1) {
  constexpr int T = (1 << LOGN) / (1 << lr_of(LOGN)), G = (1 << lr_of(LOGN)) >> RR, J = 1 << RR;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int hi = (g * T + (int)threadIdx.x) >> S0;
#pragma unroll
    for (int u = 0; u < RR; ++u) {
      const int dist = 1 << u;
#pragma unroll
      for (int j = 0; j < J; ++j) {
        if (j & dist) continue;
        const double W = __ldg(tw + (pre << (LOGN - S0 - u - 1)) + (hi << (RR - u - 1)) + (j >> (u + 1)));
        const double a = x[g * J + j], b = x[g * J + j + dist];
        x[g * J + j] = __dadd_rn(a, b);
        x[g * J + j + dist] = fp_mulmod(__dadd_rn(a, -b), W, fq);
      }
    }
  }
  // sums grew by up to 2^RR: re-centre every value (|x| <= q/2 + eps)
#pragma unroll
  for (int e = 0; e < (1 << lr_of(LOGN)); ++e) x[e] = fp_center(x[e], fq);
}

template <int LOGN, int S0, int RR>
__device__ __forceinline__ void inv_store_d(double* sm, const double (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) sm[pad(inv_idx<LOGN, S0, RR>(g, j))] = x[g * (1 << RR) + j];
}
template <int LOGN, int S0, int RR>
__device__ __forceinline__ void inv_load_d(const double* sm, double (&x)[1 << lr_of(LOGN)]) {
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
    for (int j = 0; j < (1 << RR); ++j) x[g * (1 << RR) + j] = sm[pad(inv_idx<LOGN, S0, RR>(g, j))];
}

// SPLIT (N = 2^15): this CTA holds half h; after its 14 stages the last
// Gentleman-Sande stage pairs coefficient k of the two halves through
// distributed shared memory: out[k] = (a + b) / N, out[k + N/2] = (a - b) w / N.
template <int LOGN, int S0, bool SPLIT = false, class St>
__device__ __forceinline__ void inv_passes_fp(double (&x)[1 << lr_of(LOGN)], u64d* sm, const double* tw, double2 fq,
                                              double nv, St& st, const int pre = 1, const int h = 0) {
  constexpr int RR = cmin(lr_of(LOGN), LOGN - S0);
  inv_pass_fp<LOGN, S0, RR>(x, tw, fq, pre);
  if constexpr (S0 + RR < LOGN) {
    constexpr int RN = cmin(lr_of(LOGN), LOGN - S0 - RR);
    __syncthreads();
    inv_store_d<LOGN, S0, RR>(reinterpret_cast<double*>(sm), x);
    __syncthreads();
    inv_load_d<LOGN, S0 + RR, RN>(reinterpret_cast<const double*>(sm), x);
    inv_passes_fp<LOGN, S0 + RR, SPLIT>(x, sm, tw, fq, nv, st, pre, h);
  } else if constexpr (SPLIT) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int T = (1 << LOGN) / (1 << lr_of(LOGN)), R = 1 << lr_of(LOGN);
    double* xs = reinterpret_cast<double*>(sm);
    __syncthreads();  // every thread has loaded its last pass from sm
#pragma unroll
    for (int e = 0; e < R; ++e) xs[e * T + (int)threadIdx.x] = x[e];
    cl.sync();
    const double* other = cl.map_shared_rank(xs, (unsigned)(h ^ 1));
    const double wl = __ldg(tw + 1);
#pragma unroll
    for (int g = 0; g < (R >> RR); ++g)
#pragma unroll
      for (int j = 0; j < (1 << RR); ++j) {
        const int e = g * (1 << RR) + j;
        const double o = other[e * T + (int)threadIdx.x];
        const double v = h ? fp_mulmod(fp_mulmod(__dadd_rn(o, -x[e]), wl, fq), nv, fq)
                           : fp_mulmod(__dadd_rn(x[e], o), nv, fq);
        st.store(inv_idx<LOGN, S0, RR>(g, j) + h * (1 << LOGN), fp_canon(v, fq));
      }
    cl.sync();  // the partner has read this CTA's half
  } else {
#pragma unroll
    for (int g = 0; g < ((1 << lr_of(LOGN)) >> RR); ++g)
#pragma unroll
      for (int j = 0; j < (1 << RR); ++j)
        st.store(inv_idx<LOGN, S0, RR>(g, j), fp_canon(fp_mulmod(x[g * (1 << RR) + j], nv, fq), fq));
  }
}

// input: canonical words scattered into smem (bit-reversed order), synced
template <int LOGN, class St>
__device__ __forceinline__ void inv_transform_fp(u64d* sm, St& st, const double* tw, double2 fq, double nv) {
  constexpr int R0 = cmin(lr_of(LOGN), LOGN);
  double x[1 << lr_of(LOGN)];
#pragma unroll
  for (int g = 0; g < ((1 << lr_of(LOGN)) >> R0); ++g)
#pragma unroll
    for (int j = 0; j < (1 << R0); ++j) x[g * (1 << R0) + j] = u2d(sm[pad(inv_idx<LOGN, 0, R0>(g, j))]);
  inv_passes_fp<LOGN, 0>(x, sm, tw, fq, nv, st);
}

// N = 2^15: half h; input: this half's words scattered into smem (sub-index order), synced
template <class St>
__device__ __forceinline__ void inv_transform_fp_split(u64d* sm, St& st, const double* tw, double2 fq, double nv,
                                                       int h) {
  constexpr int LS = 14, R0 = lr_of(LS);
  double x[1 << lr_of(LS)];
#pragma unroll
  for (int j = 0; j < (1 << R0); ++j) x[j] = u2d(sm[pad(inv_idx<LS, 0, R0>(0, j))]);
  inv_passes_fp<LS, 0, true>(x, sm, tw, fq, nv, st, 2 + h, h);
}

// ------------------------------------------------------------ functors
struct LdPlain {
  const u64d* p;
  __device__ u64d load(int k) const { return p[k]; }
};
// NTT inputs may be lazy (< 8q), so digit lifts only reduce when the source
// prime exceeds the target prime, and then only into [0, 4q).
struct LdReduce {  // residue mod q_src (< q_src) into the target prime
  const u64d* p;
  DevPrime pr;
  bool need;  // q_src > q
  __device__ u64d load(int k) const {
    const u64d x = p[k];
    return need ? reduce_lazy4(x, pr) : x;
  }
};
struct LdLift {  // centered lift of a residue mod qd into q: (-qd/2, qd/2] -> [0, 4q]
  const u64d* p;
  DevPrime pr;
  u64d qd;
  bool need;  // qd / 2 >= q
  __device__ u64d load(int k) const {
    const u64d x = p[k];
    const bool neg = x > (qd >> 1);
    u64d y = neg ? qd - x : x;
    if (need) y = reduce_lazy4(y, pr);
    return neg ? 4 * pr.q - y : y;
  }
};
struct StPlain {
  u64d* p;
  __device__ void store(int k, u64d v) const { p[k] = v; }
};

__device__ __forceinline__ const ulonglong2* twf(const TwArgs& t, int pi, int N) {
  return t.tw + (size_t)pi * 2 * N;
}
__device__ __forceinline__ const ulonglong2* twi(const TwArgs& t, int pi, int N) {
  return t.tw + ((size_t)pi * 2 + 1) * N;
}

// forward / inverse transform of prime pi on the FP64 path when the prime
// allows it (q < 2^45), else on the integer path; same words either way
template <int LOGN, class Ld>
__device__ __forceinline__ void fwd_t(u64d* sm, const Ld& ld, const TwArgs& ta, int pi, u64d q, int h = 0) {
  constexpr int N = 1 << LOGN;
  if constexpr (LOGN > 14) {  // split over a CTA pair (FP64-only builds)
    fwd_transform_fp_split(sm, ld, ta.twd + (size_t)pi * 2 * N, ta.fpq[pi], h);
    return;
  }
#ifdef HEGPU_NTT_FPONLY  // every prime of the context is on the FP64 path (launcher checks)
  fwd_transform_fp<LOGN>(sm, ld, ta.twd + (size_t)pi * 2 * N, ta.fpq[pi]);
  return;
#endif
#if HEGPU_NTT_FP
  const double2 fq = ta.fpq[pi];
  if (fq.x != 0.0) {
    fwd_transform_fp<LOGN>(sm, ld, ta.twd + (size_t)pi * 2 * N, fq);
    return;
  }
#endif
  fwd_transform<LOGN>(sm, ld, twf(ta, pi, N), q);
}
template <int LOGN, class St>
__device__ __forceinline__ void inv_t(u64d* sm, St& st, const TwArgs& ta, int pi, u64d q, int h = 0) {
  constexpr int N = 1 << LOGN;
  if constexpr (LOGN > 14) {
    inv_transform_fp_split(sm, st, ta.twd + ((size_t)pi * 2 + 1) * N, ta.fpq[pi], u2d(ta.ninv[2 * pi]), h);
    return;
  }
#ifdef HEGPU_NTT_FPONLY
  inv_transform_fp<LOGN>(sm, st, ta.twd + ((size_t)pi * 2 + 1) * N, ta.fpq[pi], u2d(ta.ninv[2 * pi]));
  return;
#endif
#if HEGPU_NTT_FP
  const double2 fq = ta.fpq[pi];
  if (fq.x != 0.0) {
    inv_transform_fp<LOGN>(sm, st, ta.twd + ((size_t)pi * 2 + 1) * N, fq, u2d(ta.ninv[2 * pi]));
    return;
  }
#endif
  inv_transform<LOGN>(sm, st, twi(ta, pi, N), q, ta.ninv[2 * pi], ta.ninv[2 * pi + 1]);
}

// one pass over a row: R = 2^lr words per thread, compile-time trip count so
// the loads of all R iterations are issued together (measured: helps the
// drop-limb epilogue, costs spills in the other row kernels)
#define ROW_LOOP(P)                                         \
  _Pragma("unroll") for (int _e = 0; _e < (1 << lr_of(LOGN)); ++_e) \
    if (const int P = rc.base + _e * (RowCta<LOGN>::NT >> lr_of(LOGN)) + (int)threadIdx.x; true)

// the slot-order gathers / scatters around a transform (index load -> shared
// memory -> global).  HEGPU_NTT_UNROLL_IO=1 unrolls them fully (all R index
// loads in flight at once); measured on cfg 2: ModUp 0.567 -> 0.591 ms, the
// row INTTs 0.117 -> 0.109 ms, step 3.118 -> 3.138 ms -- not kept
// (profiles/r02_notes.md)
#ifndef HEGPU_NTT_UNROLL_IO
#define HEGPU_NTT_UNROLL_IO 0
#endif
#if HEGPU_NTT_UNROLL_IO
#define IO_LOOP(P) ROW_LOOP(P)
#else
#define IO_LOOP(P) for (int P = rc.base + threadIdx.x; P < rc.base + RowCta<LOGN>::NT; P += blockDim.x)
#endif

// two CTAs per SM for N <= 8192 (<= 64 registers per thread)
#ifndef HEGPU_NTT_MINB13
#define HEGPU_NTT_MINB13 2
#endif
#define NTT_BOUNDS __launch_bounds__((1 << sub_logn(LOGN)) / (1 << lr_of(LOGN)), (LOGN <= 13 ? HEGPU_NTT_MINB13 : 1))

// ------------------------------------------------------------ kernels
template <int LOGN>
__global__ void NTT_BOUNDS k_ntt_rows(TwArgs ta, PrimeTable pt, const u64d* __restrict__ src,
                                      u64d* __restrict__ dst, int nl, int p_limb, int p_index) {
  extern __shared__ u64d sm[];
  constexpr int N = 1 << LOGN, NT = RowCta<LOGN>::NT;
  const RowCta<LOGN> rc;
  int limb;
  const int r = rc.split(nl, limb) * nl + limb;
  const int pi = (limb == p_limb) ? p_index : limb;
  fwd_t<LOGN>(sm, LdPlain{src + (size_t)r * N}, ta, pi, pt.p[pi].q, rc.h);
  u64d* d = dst + (size_t)r * N;
  IO_LOOP(p) d[p] = sm[pad((int)__ldg(ta.slot_src + p) - rc.base)];
}

struct PMap {
  int8_t p[HEGPU_MAX_PRIMES];
};

template <int LOGN>
__global__ void NTT_BOUNDS k_intt_rows(TwArgs ta, PrimeTable pt, const u64d* __restrict__ src,
                                       u64d* __restrict__ dst, int n_inner, long so, long si, long dox, long di,
                                       PMap pm) {
  extern __shared__ u64d sm[];
  constexpr int NT = RowCta<LOGN>::NT;
  const RowCta<LOGN> rc;
  int i;
  const int o = rc.split(n_inner, i);
  const int pi = pm.p[i];
  const u64d* s = src + o * so + i * si;
  IO_LOOP(p) sm[pad((int)__ldg(ta.slot_src + p) - rc.base)] = s[p];
  __syncthreads();
  StPlain st{dst + o * dox + i * di};
  inv_t<LOGN>(sm, st, ta, pi, pt.p[pi].q, rc.h);
}

// KS input: digit j of (shifted) poly b -> coefficient row tmp[b][j]; also
// writes the shifted NTT-form limb into D[b][j][j] (ModUp's own-prime row).
template <int LOGN>
__global__ void NTT_BOUNDS k_ks_intt(TwArgs ta, PrimeTable pt, const u64d* __restrict__ src, long src_stride, int l,
                                     KeyRowMap km, int use_shift, u64d* __restrict__ tmp, u64d* __restrict__ D) {
  extern __shared__ u64d sm[];
  constexpr int N = 1 << LOGN, S = N >> 1, NT = RowCta<LOGN>::NT;
  const RowCta<LOGN> rc;
  int j;
  const int b = rc.split(l, j);
  const int s = use_shift ? km.shift[b % km.period] : 0;
  const u64d* in = src + (km.grp ? (b / km.grp) * km.grp_stride + (b % km.grp) * src_stride : b * src_stride) +
                   (size_t)j * N;
  u64d* own = D + (((size_t)b * l + j) * (l + 1) + j) * N;
  IO_LOOP(p) {
    const u64d v = in[s ? shifted(p, s, S) : p];
    own[p] = v;
    sm[pad((int)__ldg(ta.slot_src + p) - rc.base)] = v;
  }
  __syncthreads();
  StPlain st{tmp + ((size_t)b * l + j) * N};
  inv_t<LOGN>(sm, st, ta, j, pt.p[j].q, rc.h);
}

// ModUp: rows (b, j, t') with t = t' < j ? t' : t'+1 over the extended basis
// (t == l means P); NTT_t(tmp[b][j] mod q_t) -> D[b][j][t]
template <int LOGN>
__global__ void NTT_BOUNDS k_ks_modup(TwArgs ta, PrimeTable pt, const u64d* __restrict__ tmp, int l, int P_index,
                                      u64d* __restrict__ D) {
  extern __shared__ u64d sm[];
  constexpr int N = 1 << LOGN, NT = RowCta<LOGN>::NT;
  const RowCta<LOGN> rc;
  int tp;
  const int bj = rc.split(l, tp), j = bj % l, b = bj / l;
  const int t = tp < j ? tp : tp + 1;
  const int pi = t == l ? P_index : t;
  const DevPrime pr = pt.p[pi];
  // the FP64 path takes any word < 4q exactly: a digit of another prime
  // below 2^45 needs no reduction there (q_j < 2 q_t)
  const bool need = pt.p[j].q > pr.q && !(HEGPU_NTT_FP && ta.fpq[pi].x != 0.0 && pt.p[j].q < (1ull << 45));
  fwd_t<LOGN>(sm, LdReduce{tmp + ((size_t)b * l + j) * N, pr, need}, ta, pi, pr.q, rc.h);
  u64d* d = D + (((size_t)b * l + j) * (l + 1) + t) * N;
  IO_LOOP(p) d[p] = sm[pad((int)__ldg(ta.slot_src + p) - rc.base)];
}

__device__ __forceinline__ void cp_async16_g2s(u64d* dst, const u64d* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}

// shared words of the drop-limb kernel: the NTT buffer, then the source limb
// and the add term of the epilogue (prefetched during the transform)
// (N <= 2^13: the prefetch buffers fit next to the transform buffer)
#ifndef HEGPU_DROP_PRE
#define HEGPU_DROP_PRE 1
#endif
__host__ __device__ constexpr bool drop_prefetch(int N) { return HEGPU_DROP_PRE && N <= 8192; }
// without the shared-memory staging (two CTAs per SM): pull the epilogue's
// rows towards L2 while the transform runs
__device__ __forceinline__ void prefetch_row_l2(const u64d* row, int N) {
  for (int i = threadIdx.x * 16; i < N; i += blockDim.x * 16)
    asm volatile("prefetch.global.L2 [%0];\n" ::"l"(row + i));
}
__host__ __device__ constexpr size_t drop_smem_words(int N) {
  return ((size_t)(N + (N >> 4) + 1 + 1) & ~(size_t)1) + (drop_prefetch(N) ? 2 * (size_t)N : 0);
}

// drop-limb NTT: rows (b, p, t < nl).  The epilogue's operands (the source
// limb and the add term) are copied into shared memory with cp.async while
// the transform runs, so the epilogue does not wait on HBM.
template <int LOGN>
__global__ void NTT_BOUNDS k_drop_ntt(TwArgs ta, PrimeTable pt, const u64d* __restrict__ qinv, int np_all,
                                      DropArgs a, const u64d* __restrict__ tmpP, KeyRowMap km, int use_shift) {
  extern __shared__ u64d sm[];
  constexpr int N = 1 << LOGN, S = N >> 1;
  const RowCta<LOGN> rc;
  int t;
  const int bp = rc.split(a.nl, t), p = bp % 2, b = bp / 2;
  const DevPrime pr = pt.p[t];
  const u64d q = pr.q;
  const u64d qd = pt.p[a.pd].q;
  const u64d* in = a.src + b * a.src_b + p * a.src_p + (size_t)t * N;
  u64d* out = a.dst + b * a.dst_b + p * a.dst_p + (size_t)t * N;
  const bool add = (a.add_mask >> p) & 1;
  const u64d* ad = add ? a.add + b * a.add_b + p * a.add_p + (size_t)t * N : nullptr;
  constexpr bool kPre = drop_prefetch(N);
  const u64d* in_s = in;
  const u64d* ad_s = ad;
  if constexpr (kPre) {
    u64d* is = sm + (((size_t)N + (N >> 4) + 1 + 1) & ~(size_t)1);
    u64d* as = is + N;
    for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
      cp_async16_g2s(is + 2 * i, in + 2 * i);
      if (add) cp_async16_g2s(as + 2 * i, ad + 2 * i);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    in_s = is;
    ad_s = as;
  } else {
    prefetch_row_l2(in, N);
    if (add) prefetch_row_l2(ad, N);
  }
  fwd_t<LOGN>(sm, LdLift{tmpP + ((size_t)b * 2 + p) * N, pr, qd, (qd >> 1) >= q}, ta, t, q, rc.h);
  const u64d iv = qinv[((size_t)t * np_all + a.pd) * 2], ivp = qinv[((size_t)t * np_all + a.pd) * 2 + 1];
  const int sh = (use_shift && p == 0) ? km.shift[b % km.period] : 0;
  if constexpr (kPre) {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  ROW_LOOP(pos) {
    u64d v = shoup_mul_d(sub_mod_d(in_s[pos], sm[pad((int)__ldg(ta.slot_src + pos) - rc.base)], q), iv, ivp, q);
    if (add) v = add_mod_d(v, ad_s[sh ? shifted(pos, sh, S) : pos], q);
    out[pos] = v;
  }
}

// ------------------------------------------- fused ModDown + rescale (§4.8)
// The ModDown of an extended-basis accumulator (limbs q_0..q_{l-1}, P) is
// directly followed by a rescale that drops q_{l-1}.  Two successive drops
// cost INTT(P) + l NTTs, then INTT(q_{l-1}) + (l-1) NTTs per polynomial;
// fused they cost INTT(P) + INTT(q_{l-1}) + (l-1) NTTs, with limbs equal to
// the two-step result residue for residue:
//   x = INTT_P(acc_P)                        (ModDown's dropped residue)
//   z = INTT_qd(acc_qd P^-1 + add_qd)         (qd = q_{l-1})
//   y = z - lift_P(x) P^-1  mod qd           (= INTT of the ModDown's limb qd,
//                                             by linearity of the INTT)
//   out_t = (acc_t P^-1 + add_t - NTT_t(lift_P(x) P^-1 + lift_qd(y))) qd^-1
// Step 1 (k_md_intt): rows (b, p, {P, qd}) -> xz[b][p][{x, z}][N].
template <int LOGN>
__global__ void NTT_BOUNDS k_md_intt(TwArgs ta, PrimeTable pt, const u64d* __restrict__ qinv, int np_all, DropArgs a,
                                     u64d* __restrict__ xz) {
  extern __shared__ u64d sm[];
  constexpr int N = 1 << LOGN, NT = RowCta<LOGN>::NT;
  const RowCta<LOGN> rc;
  int which;
  const int bp = rc.split(2, which), p = bp & 1, b = bp >> 1;
  const int lq = a.src_limbs - 2;          // limb (and prime index) of q_{l-1}
  const int pi = which ? lq : a.pd;        // a.pd: prime index of P
  const u64d* row = a.src + b * a.src_b + p * a.src_p + (size_t)(which ? lq : a.src_limbs - 1) * N;
  if (which) {
    const u64d q = pt.p[lq].q;
    const u64d iv = qinv[((size_t)lq * np_all + a.pd) * 2], ivp = qinv[((size_t)lq * np_all + a.pd) * 2 + 1];
    const bool add = (a.add_mask >> p) & 1;
    const u64d* ad = add ? a.add + b * a.add_b + p * a.add_p + (size_t)lq * N : nullptr;
    IO_LOOP(i) {
      u64d v = shoup_mul_d(row[i], iv, ivp, q);
      if (add) v = add_mod_d(v, ad[i], q);
      sm[pad((int)__ldg(ta.slot_src + i) - rc.base)] = v;
    }
  } else {
    IO_LOOP(i) sm[pad((int)__ldg(ta.slot_src + i) - rc.base)] = row[i];
  }
  __syncthreads();
  StPlain st{xz + ((size_t)bp * 2 + which) * N};
  inv_t<LOGN>(sm, st, ta, pi, pt.p[pi].q, rc.h);
}

// centered lift of a residue mod m (< m) times a constant c (Shoup pair), mod q
__device__ __forceinline__ u64d lift_mul(u64d v, u64d m, u64d c, u64d cp, u64d q) {
  const bool neg = v > (m >> 1);
  const u64d r = shoup_mul_d(neg ? m - v : v, c, cp, q);  // Shoup: any word input, result in [0, q)
  return (neg && r) ? q - r : r;
}

// Step 2: rows (b, p, t < nl = l - 1): u = lift_P(x) P^-1 + lift_qd(y) mod
// q_t, NTT, out_t = (acc_t P^-1 + add_t - NTT(u)) qd^-1; the epilogue's
// operands are prefetched into shared memory during the transform
struct LdMd {
  const u64d* x;
  const u64d* z;
  u64d P, qd, q;
  u64d pv, pvp;    // P^-1 mod q_t
  u64d pqv, pqvp;  // P^-1 mod qd
  u64d one_sh;     // floor(2^64 / q_t)
  __device__ u64d load(int k) const {
    const u64d xv = x[k];
    const u64d y = sub_mod_d(z[k], lift_mul(xv, P, pqv, pqvp, qd), qd);
    return add_mod_d(lift_mul(xv, P, pv, pvp, q), lift_mul(y, qd, 1ull, one_sh, q), q);
  }
};

template <int LOGN>
__global__ void NTT_BOUNDS k_md_ntt(TwArgs ta, PrimeTable pt, const u64d* __restrict__ qinv, int np_all, DropArgs a,
                                    const u64d* __restrict__ xz) {
  extern __shared__ u64d sm[];
  constexpr int N = 1 << LOGN;
  const RowCta<LOGN> rc;
  int t;
  const int bp = rc.split(a.nl, t), p = bp % 2, b = bp / 2;
  const int lq = a.src_limbs - 2;
  const DevPrime pr = pt.p[t];
  const u64d q = pr.q;
  const u64d* in = a.src + b * a.src_b + p * a.src_p + (size_t)t * N;
  u64d* out = a.dst + b * a.dst_b + p * a.dst_p + (size_t)t * N;
  const bool add = (a.add_mask >> p) & 1;
  const u64d* ad = add ? a.add + b * a.add_b + p * a.add_p + (size_t)t * N : nullptr;
  constexpr bool kPre = drop_prefetch(N);
  const u64d* in_s = in;
  const u64d* ad_s = ad;
  if constexpr (kPre) {
    u64d* is = sm + (((size_t)N + (N >> 4) + 1 + 1) & ~(size_t)1);
    u64d* as = is + N;
    for (int i = threadIdx.x; i < N / 2; i += blockDim.x) {
      cp_async16_g2s(is + 2 * i, in + 2 * i);
      if (add) cp_async16_g2s(as + 2 * i, ad + 2 * i);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    in_s = is;
    ad_s = as;
  } else {
    prefetch_row_l2(in, N);
    if (add) prefetch_row_l2(ad, N);
  }
  const u64d pv = qinv[((size_t)t * np_all + a.pd) * 2], pvp = qinv[((size_t)t * np_all + a.pd) * 2 + 1];
  const u64d qv = qinv[((size_t)t * np_all + lq) * 2], qvp = qinv[((size_t)t * np_all + lq) * 2 + 1];
  const u64d* X = xz + (size_t)bp * 2 * N;
  LdMd ld{X, X + N, pt.p[a.pd].q, pt.p[lq].q, q, pv, pvp,
          qinv[((size_t)lq * np_all + a.pd) * 2], qinv[((size_t)lq * np_all + a.pd) * 2 + 1], pr.one_sh};
  fwd_t<LOGN>(sm, ld, ta, t, q, rc.h);
  if constexpr (kPre) {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
  }
  ROW_LOOP(pos) {
    u64d v = shoup_mul_d(in_s[pos], pv, pvp, q);
    if (add) v = add_mod_d(v, ad_s[pos], q);
    out[pos] = shoup_mul_d(sub_mod_d(v, sm[pad((int)__ldg(ta.slot_src + pos) - rc.base)], q), qv, qvp, q);
  }
}

// wire (bit-reversed) <-> slot order, optional Montgomery conversion
__global__ void k_wire_to_slot(const u64d* __restrict__ src, u64d* __restrict__ dst,
                               const uint32_t* __restrict__ slot_src, PrimeTable pt, int N, int to_mont, int nl,
                               int p_limb, int p_index) {
  const size_t r = blockIdx.y;
  const int limb = (int)(r % nl);
  const DevPrime pr = pt.p[limb == p_limb ? p_index : limb];
  const u64d* s = src + r * N;
  u64d* d = dst + r * N;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    u64d v = s[__ldg(slot_src + p)];
    d[p] = to_mont ? mont_mul(v, pr.r2_mod, pr.q, pr.qneg_inv) : v;
  }
}

__global__ void k_slot_to_wire(const u64d* __restrict__ src, u64d* __restrict__ dst,
                               const uint32_t* __restrict__ slot_src, PrimeTable pt, int N, int from_mont, int nl,
                               int p_limb, int p_index) {
  const size_t r = blockIdx.y;
  const int limb = (int)(r % nl);
  const DevPrime pr = pt.p[limb == p_limb ? p_index : limb];
  const u64d* s = src + r * N;
  u64d* d = dst + r * N;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    u64d v = s[p];
    d[__ldg(slot_src + p)] = from_mont ? mont_mul(v, 1ull, pr.q, pr.qneg_inv) : v;
  }
}

TwArgs tw_args(Context& c) {
  return TwArgs{(const ulonglong2*)c.d_tw, c.ninv_tab(), c.d_slot_src, c.d_twd, (const double2*)c.d_fpq};
}

size_t ntt_smem(int N) { return (size_t)(N + (N >> 4) + 1) * 8; }

template <typename K>
void prep_kernel(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

// <<<grid, threads>>> for N <= 2^14; N = 2^15 launches two CTAs per row as
// a thread-block cluster (the inverse kernels exchange halves through DSMEM)
template <typename... KA, typename... A>
void launch_rows(void (*kernel)(KA...), int lg, int grid, size_t smb, cudaStream_t st, A&&... args) {
  const int threads = (1 << sub_logn(lg)) >> lr_of(lg);
  if (lg <= 14) {
    kernel<<<grid, threads, smb, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2u * (unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smb;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, kernel, KA(args)...));
}

// N = 2^15 exists in the 16-word FP64-only builds only (every prime < 2^45)
#if defined(HEGPU_NTT_FPONLY) && HEGPU_NTT_LR13 == 4
#define NTT_GO15(KERNEL, GRID, ...) NTT_GO(15, KERNEL, GRID, __VA_ARGS__)
#else
#define NTT_GO15(KERNEL, GRID, ...) \
  fail(HEGPU_ERR_ARG, "N = 2^15 runs on the FP64 NTT only: every prime of the chain must be below 2^45")
#endif

// one launch per op, dispatched on log2 N
#define NTT_DISPATCH(logn, KERNEL, GRID, ...)                                                       \
  do {                                                                                              \
    switch (logn) {                                                                                 \
      case 5: NTT_GO(5, KERNEL, GRID, __VA_ARGS__); break;                                          \
      case 6: NTT_GO(6, KERNEL, GRID, __VA_ARGS__); break;                                          \
      case 7: NTT_GO(7, KERNEL, GRID, __VA_ARGS__); break;                                          \
      case 8: NTT_GO(8, KERNEL, GRID, __VA_ARGS__); break;                                          \
      case 9: NTT_GO(9, KERNEL, GRID, __VA_ARGS__); break;                                          \
      case 10: NTT_GO(10, KERNEL, GRID, __VA_ARGS__); break;                                        \
      case 11: NTT_GO(11, KERNEL, GRID, __VA_ARGS__); break;                                        \
      case 12: NTT_GO(12, KERNEL, GRID, __VA_ARGS__); break;                                        \
      case 13: NTT_GO(13, KERNEL, GRID, __VA_ARGS__); break;                                        \
      case 14: NTT_GO(14, KERNEL, GRID, __VA_ARGS__); break;                                        \
      case 15: NTT_GO15(KERNEL, GRID, __VA_ARGS__); break;                                          \
      default: fail(HEGPU_ERR_ARG, "NTT: log2 N must be in [5, 15] on the device");                \
    }                                                                                               \
  } while (0)

#define NTT_GO(LG, KERNEL, GRID, ...)                                                               \
  do {                                                                                              \
    static PerDeviceOnce prepared;                                                                  \
    const size_t smb = ntt_smem(1 << sub_logn(LG));                                                 \
    if (prepared.first()) prep_kernel(KERNEL<LG>, smb);                                             \
    LAUNCH_BO(c, #KERNEL, _ntt_bytes, (double)(GRID) * (LG << (LG - 1)),                           \
              launch_rows(KERNEL<LG>, LG, (GRID), smb, c.stream, __VA_ARGS__));                     \
  } while (0)

}  // namespace

// ntt_r8.cu re-includes this file with 8 words per thread for N <= 2^13
// (1024-thread CTAs, no register spills): measured faster for the row
// INTTs and the drop-limb NTTs, slower for ModUp (profiles/r01_notes.md),
// so those two entry points dispatch to the _r8 build.
#if defined(HEGPU_NTT_SUFFIX)
#define NTT_PUB_CAT_(x, s) x##s
#define NTT_PUB_CAT(x, s) NTT_PUB_CAT_(x, s)
#define NTT_PUB(x) NTT_PUB_CAT(x, HEGPU_NTT_SUFFIX)
#elif defined(HEGPU_NTT_R8_VARIANT)
#define NTT_PUB(x) x##_r8
#else
#define NTT_PUB(x) x##_r16
#endif

#ifndef HEGPU_NTT_R8_VARIANT
// HEGPU_NTT_FP=0 keeps every prime on the integer butterflies (A/B switch)
bool ntt_fp_enabled() {
  const char* e = getenv("HEGPU_NTT_FP");
  return !(e && e[0] == '0');
}
// HEGPU_NTT_R8=1: every N <= 2^13 entry point on the 8-words-per-thread build
static bool ntt_all_r8() {
  const char* e = getenv("HEGPU_NTT_R8");
  return e && e[0] == '1';
}

void upload_twiddles(Context& c) {
  const Params& P = *c.P;
  const int np = P.np(), N = P.n;
  if (P.log_n < kMinLogN || P.log_n > kMaxLogN) fail(HEGPU_ERR_ARG, "device NTT supports 2^5 <= N <= 2^15");
  std::vector<u64> tw((size_t)np * 2 * N * 2);
  for (int i = 0; i < np; ++i) {
    const Prime& pr = P.primes[i];
    for (int k = 0; k < N; ++k) {
      tw[(((size_t)i * 2 + 0) * N + k) * 2 + 0] = pr.w[k];
      tw[(((size_t)i * 2 + 0) * N + k) * 2 + 1] = pr.wp[k];
      tw[(((size_t)i * 2 + 1) * N + k) * 2 + 0] = pr.iw[k];
      tw[(((size_t)i * 2 + 1) * N + k) * 2 + 1] = pr.iwp[k];
    }
  }
  CK(cudaMalloc((void**)&c.d_tw, tw.size() * 8));
  CK(cudaMemcpy(c.d_tw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice));
  // FP64 butterflies (§5.1) for primes below 2^45: w as exact doubles, (q, 1/q)
  std::vector<double> twd((size_t)np * 2 * N), fpq((size_t)np * 2, 0.0);
  for (int i = 0; i < np; ++i) {
    const Prime& pr = P.primes[i];
    if (pr.q >= (1ull << 45) || !ntt_fp_enabled()) continue;
    fpq[2 * i] = (double)pr.q;
    fpq[2 * i + 1] = 1.0 / (double)pr.q;
    for (int k = 0; k < N; ++k) {
      twd[((size_t)i * 2 + 0) * N + k] = (double)pr.w[k];
      twd[((size_t)i * 2 + 1) * N + k] = (double)pr.iw[k];
    }
  }
  CK(cudaMalloc((void**)&c.d_twd, twd.size() * 8));
  CK(cudaMemcpy(c.d_twd, twd.data(), twd.size() * 8, cudaMemcpyHostToDevice));
  c.fp_all = true;
  for (int i = 0; i < np; ++i) c.fp_all = c.fp_all && fpq[2 * i] != 0.0;
  if (P.log_n > 14 && !c.fp_all)
    fail(HEGPU_ERR_ARG, "N = 2^15 runs on the FP64 NTT only: every prime of the chain must be below 2^45");
  CK(cudaMalloc((void**)&c.d_fpq, fpq.size() * 8));
  CK(cudaMemcpy(c.d_fpq, fpq.data(), fpq.size() * 8, cudaMemcpyHostToDevice));
}

#endif  // !HEGPU_NTT_R8_VARIANT

#ifndef HEGPU_NTT_ONLY_DROP
void NTT_PUB(launch_ntt_rows)(Context& c, const u64d* src, u64d* dst, int rows, int nl, int p_limb) {
  if (rows <= 0) return;
  if (nl <= 0 || rows % nl) fail(HEGPU_ERR_ARG, "ntt_rows: the row count must be a multiple of the limb count");
  const double _ntt_bytes = 16.0 * c.N() * rows;  // read + write one limb per row
  NTT_DISPATCH(c.P->log_n, k_ntt_rows, rows, tw_args(c), c.primes, src, dst, nl, p_limb, c.L());
}
#endif

void NTT_PUB(launch_intt_rows)(Context& c, const u64d* src, u64d* dst, int n_outer, int n_inner, long so, long si,
                               long dox, long di, const int* prime_of_inner) {
  if (n_outer * n_inner <= 0) return;
  if (n_inner > HEGPU_MAX_PRIMES) fail(HEGPU_ERR_ARG, "intt_rows: too many limbs");
  PMap pm{};
  for (int i = 0; i < n_inner; ++i) pm.p[i] = (int8_t)prime_of_inner[i];
  const double _ntt_bytes = 16.0 * c.N() * n_outer * n_inner;
  NTT_DISPATCH(c.P->log_n, k_intt_rows, n_outer * n_inner, tw_args(c), c.primes, src, dst, n_inner, so, si, dox,
               di, pm);
}

#ifndef HEGPU_NTT_R8_VARIANT
void launch_wire_to_slot(Context& c, const u64d* src, u64d* dst, size_t rows, int to_mont, int nl, int p_limb) {
  if (!rows) return;
  dim3 grid((c.N() + 255) / 256 < 8 ? (c.N() + 255) / 256 : 8, (unsigned)rows);
  LAUNCH(c, "k_wire_to_slot",
         k_wire_to_slot<<<grid, 256, 0, c.stream>>>(src, dst, c.d_slot_src, c.primes, c.N(), to_mont, nl, p_limb,
                                                    c.L()));
}

void launch_slot_to_wire(Context& c, const u64d* src, u64d* dst, size_t rows, int from_mont, int nl, int p_limb) {
  if (!rows) return;
  dim3 grid((c.N() + 255) / 256 < 8 ? (c.N() + 255) / 256 : 8, (unsigned)rows);
  LAUNCH(c, "k_slot_to_wire",
         k_slot_to_wire<<<grid, 256, 0, c.stream>>>(src, dst, c.d_slot_src, c.primes, c.N(), from_mont, nl, p_limb,
                                                    c.L()));
}

#endif  // !HEGPU_NTT_R8_VARIANT

#ifndef HEGPU_NTT_ONLY_DROP
void NTT_PUB(ks_modup)(Context& c, const u64d* src, long src_stride, int B, int l, const KeyRowMap* shifts,
                       u64d* tmp, u64d* D) {
  KeyRowMap dummy{};
  dummy.period = 1;
  double _ntt_bytes = 24.0 * c.N() * B * l;  // read digit, write coefficients + own-prime copy
  NTT_DISPATCH(c.P->log_n, k_ks_intt, B * l, tw_args(c), c.primes, src, src_stride, l, shifts ? *shifts : dummy,
               shifts != nullptr, tmp, D);
  _ntt_bytes = 16.0 * c.N() * B * l * l;
  if (B * l * l > 0) NTT_DISPATCH(c.P->log_n, k_ks_modup, B * l * l, tw_args(c), c.primes, tmp, l, c.L(), D);
}
#endif

void NTT_PUB(drop_last_limb)(Context& c, int B, const DropArgs& a, u64d* tmpP) {
  const int N = c.N();
  if (a.fuse_rescale) {
    // ModDown by P and rescale by q_{l-1} in one pass (§4.8): a.nl = l - 1
    KeyRowMap dummy{};
    dummy.period = 1;
    if (a.shifts) fail(HEGPU_ERR_ARG, "fused ModDown + rescale: no shifted add term");
    u64d* xz = c.alloc((size_t)B * 2 * 2 * N);
    double _ntt_bytes = 8.0 * N * B * 2 * (2.0 + 1.0 + (a.add_mask ? 1.0 : 0.0) + 2.0);
    NTT_DISPATCH(c.P->log_n, k_md_intt, B * 4, tw_args(c), c.primes, c.qinv_tab(), c.P->np(), a, xz);
    if (a.nl > 0) {
      // read x, z, acc_t (+ add_t), write out_t
      _ntt_bytes = (32.0 + (a.add_mask ? 8.0 : 0.0)) * N * B * 2 * a.nl;
#undef NTT_GO
#define NTT_GO(LG, KERNEL, GRID, ...)                                                               \
  do {                                                                                              \
    static PerDeviceOnce prepared;                                                                  \
    const size_t smb = drop_smem_words(1 << sub_logn(LG)) * 8;                                      \
    if (prepared.first()) prep_kernel(KERNEL<LG>, smb);                                             \
    LAUNCH_BO(c, #KERNEL, _ntt_bytes, (double)(GRID) * (LG << (LG - 1)),                           \
              launch_rows(KERNEL<LG>, LG, (GRID), smb, c.stream, __VA_ARGS__));                     \
  } while (0)
      NTT_DISPATCH(c.P->log_n, k_md_ntt, B * 2 * a.nl, tw_args(c), c.primes, c.qinv_tab(), c.P->np(), a, xz);
#undef NTT_GO
#define NTT_GO(LG, KERNEL, GRID, ...)                                                               \
  do {                                                                                              \
    static PerDeviceOnce prepared;                                                                  \
    const size_t smb = ntt_smem(1 << sub_logn(LG));                                                 \
    if (prepared.first()) prep_kernel(KERNEL<LG>, smb);                                             \
    LAUNCH_BO(c, #KERNEL, _ntt_bytes, (double)(GRID) * (LG << (LG - 1)),                           \
              launch_rows(KERNEL<LG>, LG, (GRID), smb, c.stream, __VA_ARGS__));                     \
  } while (0)
    }
    c.free(xz);
    (void)dummy;
    return;
  }
  const int pmap[2] = {a.pd, a.pd};
  NTT_PUB(launch_intt_rows)(c, a.src + (size_t)(a.src_limbs - 1) * N, tmpP, B, 2, a.src_b, a.src_p, 2L * N, N, pmap);
  if (a.nl <= 0) return;
  KeyRowMap dummy{};
  dummy.period = 1;
  // read lifted residue + source limb (+ add term), write the output limb
  const double _ntt_bytes = (24.0 + (a.add ? 8.0 : 0.0)) * N * B * 2 * a.nl;
#undef NTT_GO
#define NTT_GO(LG, KERNEL, GRID, ...)                                                               \
  do {                                                                                              \
    static PerDeviceOnce prepared;                                                                  \
    const size_t smb = drop_smem_words(1 << sub_logn(LG)) * 8;                                      \
    if (prepared.first()) prep_kernel(KERNEL<LG>, smb);                                             \
    LAUNCH_BO(c, #KERNEL, _ntt_bytes, (double)(GRID) * (LG << (LG - 1)),                           \
              launch_rows(KERNEL<LG>, LG, (GRID), smb, c.stream, __VA_ARGS__));                     \
  } while (0)
  NTT_DISPATCH(c.P->log_n, k_drop_ntt, B * 2 * a.nl, tw_args(c), c.primes, c.qinv_tab(), c.P->np(), a, tmpP,
               a.shifts ? *a.shifts : dummy, a.shifts != nullptr);
#undef NTT_GO
#define NTT_GO(LG, KERNEL, GRID, ...)                                                               \
  do {                                                                                              \
    static PerDeviceOnce prepared;                                                                  \
    const size_t smb = ntt_smem(1 << sub_logn(LG));                                                 \
    if (prepared.first()) prep_kernel(KERNEL<LG>, smb);                                             \
    LAUNCH_BO(c, #KERNEL, _ntt_bytes, (double)(GRID) * (LG << (LG - 1)),                           \
              launch_rows(KERNEL<LG>, LG, (GRID), smb, c.stream, __VA_ARGS__));                     \
  } while (0)
}

#ifndef HEGPU_NTT_R8_VARIANT
// Per-entry-point choice of the build (thread granularity, FP64-only):
// when every prime of the context is below 2^45 the FP64-only builds run
// (ntt_fp16.cu: 16 words per thread, ntt_fp8.cu: 8 words per thread at two
// 1024-thread CTAs per SM), with no integer-butterfly code in the kernels;
// otherwise the dual-path builds (ntt.cu: 16, ntt_r8.cu: 8 words per thread).
// HEGPU_NTT_FPV=<ntt><intt><modup><md> digits (1 = 16 words, 0 = 8 words)
// overrides the FP64-only choice for A/B measurements.  Measured (cfg 2,
// profiles/r02_notes.md): the 16-word FP64-only build is fastest for the row
// transforms and ModUp; the drop-limb kernels (rescale / ModDown, and the
// fused ModDown + rescale) run the 16-word build WITHOUT the shared-memory
// staging of their epilogue operands (ntt_fp16n.cu): 69 KB per CTA keeps two
// CTAs per SM, where the staged kernels (200 KB) ran one.
static bool fpv16(int entry, bool dflt) {
  const char* e = getenv("HEGPU_NTT_FPV");
  if (!e || (int)strlen(e) <= entry) return dflt;
  return e[entry] == '1';
}
void launch_ntt_rows(Context& c, const u64d* src, u64d* dst, int rows, int nl, int p_limb) {
  if (c.fp_all && c.P->log_n <= 13 && !fpv16(0, true)) launch_ntt_rows_fp8(c, src, dst, rows, nl, p_limb);
  else if (c.fp_all) launch_ntt_rows_fp16(c, src, dst, rows, nl, p_limb);
  else if (ntt_all_r8()) launch_ntt_rows_r8(c, src, dst, rows, nl, p_limb);
  else launch_ntt_rows_r16(c, src, dst, rows, nl, p_limb);
}
void launch_intt_rows(Context& c, const u64d* src, u64d* dst, int n_outer, int n_inner, long so, long si, long dox,
                      long di, const int* prime_of_inner) {
  if (c.fp_all && c.P->log_n <= 13 && !fpv16(1, true))
    launch_intt_rows_fp8(c, src, dst, n_outer, n_inner, so, si, dox, di, prime_of_inner);
  else if (c.fp_all) launch_intt_rows_fp16(c, src, dst, n_outer, n_inner, so, si, dox, di, prime_of_inner);
  else launch_intt_rows_r8(c, src, dst, n_outer, n_inner, so, si, dox, di, prime_of_inner);
}
void ks_modup(Context& c, const u64d* src, long src_stride, int B, int l, const KeyRowMap* shifts, u64d* tmp,
              u64d* D) {
  c.ks[KS_MODUP] += B;
  if (c.fp_all && c.P->log_n <= 13 && !fpv16(2, true)) ks_modup_fp8(c, src, src_stride, B, l, shifts, tmp, D);
  else if (c.fp_all) ks_modup_fp16(c, src, src_stride, B, l, shifts, tmp, D);
  else if (ntt_all_r8()) ks_modup_r8(c, src, src_stride, B, l, shifts, tmp, D);
  else ks_modup_r16(c, src, src_stride, B, l, shifts, tmp, D);
}
// HEGPU_DROP_V=<md><plain>: 0 = r8 dual-path, 1 = fp16 (smem-staged epilogue), 2 = fp16n (no staging;
// default: two CTAs per SM beat the staged epilogue, cfg 2 drop 0.46 -> 0.40 ms, md_ntt 0.23 -> 0.21 ms)
static int dropv(int entry, int dflt) {
  const char* e = getenv("HEGPU_DROP_V");
  if (!e || (int)strlen(e) <= entry) return dflt;
  return e[entry] - '0';
}
void drop_last_limb(Context& c, int B, const DropArgs& a, u64d* tmpP) {
  c.ks[a.pd == c.L() ? KS_MODDOWN : KS_RESCALE] += B;
  if (a.fuse_rescale) c.ks[KS_RESCALE] += B;
  if (c.fp_all) {
    const int v = dropv(a.fuse_rescale ? 0 : 1, 2);
    if (v == 2) return drop_last_limb_fp16n(c, B, a, tmpP);
    if (v == 1) {
      if (a.fuse_rescale && c.P->log_n <= 13 && !fpv16(3, true)) return drop_last_limb_fp8(c, B, a, tmpP);
      return drop_last_limb_fp16(c, B, a, tmpP);
    }
  }
  drop_last_limb_r8(c, B, a, tmpP);
}
#endif

}  // namespace hegpu
