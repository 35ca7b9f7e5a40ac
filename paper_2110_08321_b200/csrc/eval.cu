#include <type_traits>
// eval.cu -- pointwise RNS kernels, the key-switch inner product, the
// conv-pack MAC, the Halevi-Shoup diagonal accumulation, and the evaluator
// compositions (rescale, Galois rotation, square + relinearise).
//
// Reference semantics: add / mul (proj/src/slotvec.cpp:97-109), rotate_right
// / rotate_left (:42-66), square_layer (proj/src/convlower.cpp:141-143),
// conv_packed_forward (:39-74), hs_matvec (proj/src/matvec.cpp:82-105).  The
// CKKS math (hybrid key switch, alpha = 1, one special prime) is fixed in
// DESIGN.md §3 and restated by oracle/ckks_oracle.c.
#include <algorithm>
#include <cstdlib>

#include "engine.hpp"

namespace hegpu {

namespace {

constexpr int kTpb = 256;

__device__ __forceinline__ int shifted_pos(int p, int s, int S) {
  const int h = p >= S ? S : 0;
  int j = p - h + s;
  if (j >= S) j -= S;
  return h + j;
}

// 192-bit multiply-accumulate (lo, hi, top) += a * b
__device__ __forceinline__ void mad192(u64d& lo, u64d& hi, uint32_t& top, u64d a, u64d b) {
  asm("mad.lo.cc.u64 %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u64 %1, %3, %4, %1;\n\t"
      "addc.u32 %2, %2, 0;\n\t"
      : "+l"(lo), "+l"(hi), "+r"(top)
      : "l"(a), "l"(b));
}
// (top:hi:lo) * 2^-64 mod q  (the sum of products of standard x Montgomery)
__device__ __forceinline__ u64d red192(u64d lo, u64d hi, uint32_t top, const DevPrime& pr) {
  u64d x = mont_reduce128(hi, (u64d)top, pr.q, pr.qneg_inv);  // (top:hi) R^-1
  x = mont_mul(x, pr.r2_mod, pr.q, pr.qneg_inv);              // (top:hi) mod q
  const u64d y = mont_reduce128(lo, 0ull, pr.q, pr.qneg_inv); // lo R^-1
  return add_mod_d(x, y, pr.q);
}

// elementwise over [count][2][l][N]
__global__ void k_add(PrimeTable pt, const u64d* __restrict__ a, const u64d* __restrict__ b,
                      u64d* __restrict__ out, size_t total, int l, int N) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int limb = (int)((i / N) % l);
    out[i] = add_mod_d(a[i], b[i], pt.p[limb].q);
  }
}

// add a (Montgomery) plaintext to poly 0; copy poly 1
__global__ void k_add_plain(PrimeTable pt, const u64d* __restrict__ a, const u64d* __restrict__ p,
                            long p_stride, u64d* __restrict__ out, size_t total, int l, int N) {
  const size_t per = (size_t)2 * l * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / per, r = i % per;
    const int poly = (int)(r / ((size_t)l * N));
    const size_t lk = r % ((size_t)l * N);
    if (poly == 0) {
      const DevPrime pr = pt.p[lk / N];
      const u64d pv = mont_mul(p[b * p_stride + lk], 1ull, pr.q, pr.qneg_inv);
      out[i] = add_mod_d(a[i], pv, pr.q);
    } else {
      out[i] = a[i];
    }
  }
}

__global__ void k_mul_plain(PrimeTable pt, const u64d* __restrict__ a, const u64d* __restrict__ p,
                            long p_stride, u64d* __restrict__ out, size_t total, int l, int N) {
  const size_t per = (size_t)2 * l * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / per, r = i % per;
    const size_t lk = r % ((size_t)l * N);
    const DevPrime pr = pt.p[lk / N];
    out[i] = mont_mul(a[i], p[b * p_stride + lk], pr.q, pr.qneg_inv);
  }
}

// (c0, c1)^2 -> d01 = [c0^2, 2 c0 c1], d2 = c1^2
__global__ void k_tensor_square(PrimeTable pt, const u64d* __restrict__ a, u64d* __restrict__ d01,
                                u64d* __restrict__ d2, size_t total /* count*l*N */, int l, int N) {
  const size_t ln = (size_t)l * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t b = i / ln, r = i % ln;
    const DevPrime pr = pt.p[r / N];
    const u64d c0 = a[b * 2 * ln + r], c1 = a[b * 2 * ln + ln + r];
    const u64d c0m = mont_mul(c0, pr.r2_mod, pr.q, pr.qneg_inv);
    const u64d c1m = mont_mul(c1, pr.r2_mod, pr.q, pr.qneg_inv);
    const u64d x01 = mont_mul(c0m, c1, pr.q, pr.qneg_inv);
    d01[b * 2 * ln + r] = mont_mul(c0m, c0, pr.q, pr.qneg_inv);
    d01[b * 2 * ln + ln + r] = add_mod_d(x01, x01, pr.q);
    d2[b * ln + r] = mont_mul(c1m, c1, pr.q, pr.qneg_inv);
  }
}

// key-switch inner product: acc[b][p][t] = sum_j D[b][j][t] * key_b[j][p][pi(t)].
// Rows sharing a key (b = (u*KT + bb) * period + jkey) are tiled KT per
// thread so every key word is loaded once for KT ciphertexts.
// rows per thread / accumulator of the key-switch inner products: measured
// on cfg2 (profiles/r01_notes.md) KT=1 with the carry-chain AccC 0.735 ms,
// KT=1 Acc3 0.789, KT=2 Acc3 0.797, KT=4 Acc3 1.07, KT=4 AccC 1.48, KT=8 1.84
#ifndef HEGPU_KS_KT
#define HEGPU_KS_KT 1
#endif
#ifndef HEGPU_KS_ACC
#define HEGPU_KS_ACC AccC
#endif
__device__ __forceinline__ void cp_async8(u64d* dst, const u64d* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int kKsKT = HEGPU_KS_KT;
#ifndef HEGPU_KS_STAGE
#define HEGPU_KS_STAGE 0  // 1: KT = 1 stages the key and digit words with cp.async (measured 0.757 vs 0.735 ms)
#endif
__global__ void __launch_bounds__(kTpb) k_ks_inner(PrimeTable pt, const u64d* __restrict__ D, int B, int l, int L,
                                                   int N, KeyRowMap km, u64d* __restrict__ acc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  const int jkey = blockIdx.z % km.period, u = blockIdx.z / km.period;
  if (k >= N) return;
  const int pi = t == l ? L : t;
  const DevPrime pr = pt.p[pi];
  const u64d* key = km.key[jkey] + (size_t)pi * N + k;  // split-31 Montgomery words
  const size_t kp = (size_t)(L + 1) * N;                // one key poly over all primes
  int rows[kKsKT];
  HEGPU_KS_ACC a0[kKsKT], a1[kKsKT];
#pragma unroll
  for (int bb = 0; bb < kKsKT; ++bb) {
    rows[bb] = (u * kKsKT + bb) * km.period + jkey;
    a0[bb].zero();
    a1[bb].zero();
  }
#if HEGPU_KS_STAGE
  if constexpr (kKsKT == 1) {
    // all 3l words of this thread in flight at once, into its own smem slots
    extern __shared__ u64d stg[];
    u64d* my = stg + threadIdx.x;
    const int row = rows[0];
    if (row < B) {
      for (int j = 0; j < l; ++j) {
        cp_async8(my + (3 * j) * blockDim.x, key + (size_t)j * 2 * kp);
        cp_async8(my + (3 * j + 1) * blockDim.x, key + (size_t)j * 2 * kp + kp);
        cp_async8(my + (3 * j + 2) * blockDim.x, D + (((size_t)row * l + j) * (l + 1) + t) * N + k);
      }
      cp_async_wait_all();
      for (int j = 0; j < l; ++j) {
        const u64d d = split31(my[(3 * j + 2) * blockDim.x]);
        a0[0].mad(d, my[(3 * j) * blockDim.x]);
        a1[0].mad(d, my[(3 * j + 1) * blockDim.x]);
        if ((j & 3) == 3) a0[0].fold(), a1[0].fold();
      }
      u64d* o = acc + ((size_t)row * 2 * (l + 1) + t) * N + k;
      o[0] = a0[0].reduce(pr);
      o[(size_t)(l + 1) * N] = a1[0].reduce(pr);
    }
    return;
  }
#endif
  for (int j = 0; j < l; ++j) {
    const u64d k0 = __ldg(key + (size_t)j * 2 * kp), k1 = __ldg(key + (size_t)j * 2 * kp + kp);
#pragma unroll
    for (int bb = 0; bb < kKsKT; ++bb) {
      if (rows[bb] >= B) break;
      const u64d d = split31(D[(((size_t)rows[bb] * l + j) * (l + 1) + t) * N + k]);
      a0[bb].mad(d, k0);
      a1[bb].mad(d, k1);
    }
    if ((j & 3) == 3) {
#pragma unroll
      for (int bb = 0; bb < kKsKT; ++bb) a0[bb].fold(), a1[bb].fold();
    }
  }
#pragma unroll
  for (int bb = 0; bb < kKsKT; ++bb) {
    if (rows[bb] >= B) break;
    u64d* o = acc + ((size_t)rows[bb] * 2 * (l + 1) + t) * N + k;
    o[0] = a0[bb].reduce(pr);
    o[(size_t)(l + 1) * N] = a1[bb].reduce(pr);
  }
}

// the same with the digit count a template parameter: every load of the
// thread (LV digit words, 2 LV key words) is issued before the first
// multiply-accumulate and all addressing is compile-time strided (the
// runtime-l loop above executed ~680 SASS per output pair at l = 5)
template <int LV>
__global__ void __launch_bounds__(kTpb) k_ks_inner_t(PrimeTable pt, const u64d* __restrict__ D, int B, int L, int N,
                                                     KeyRowMap km, u64d* __restrict__ acc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y;
  const int jkey = blockIdx.z % km.period, row = (blockIdx.z / km.period) * km.period + jkey;
  if (k >= N || row >= B) return;
  const int pi = t == LV ? L : t;
  const DevPrime pr = pt.p[pi];
  const u64d* key = km.key[jkey] + (size_t)pi * N + k;  // split-31 Montgomery words
  const size_t kp = (size_t)(L + 1) * N;
  const u64d* d = D + ((size_t)row * LV * (LV + 1) + t) * N + k;
  u64d dv[LV], k0[LV], k1[LV];
#pragma unroll
  for (int j = 0; j < LV; ++j) {
    dv[j] = d[(size_t)j * (LV + 1) * N];
    k0[j] = __ldg(key + (size_t)j * 2 * kp);
    k1[j] = __ldg(key + (size_t)j * 2 * kp + kp);
  }
  HEGPU_KS_ACC a0, a1;
  a0.zero();
  a1.zero();
#pragma unroll
  for (int j = 0; j < LV; ++j) {
    const u64d x = split31(dv[j]);
    a0.mad(x, k0[j]);
    a1.mad(x, k1[j]);
    if ((j & 3) == 3 && j + 1 < LV) a0.fold(), a1.fold();
  }
  u64d* o = acc + ((size_t)row * 2 * (LV + 1) + t) * N + k;
  o[0] = a0.reduce(pr);
  o[(size_t)(LV + 1) * N] = a1.reduce(pr);
}

// merged first layer: out[b][p][t][k] = sum_s tap_s[b][p][t][k] * P_s[t][k]
// (+ the block bias on part 0), one thread per output word, taps streamed
// from HBM once (each weight word is shared by all images through L1/L2)
template <class Acc>
__device__ __forceinline__ u64d conv_pt_mac(const u64d* __restrict__ x, const u64d* __restrict__ w, int G,
                                            size_t ct, size_t wstride, const DevPrime& pr) {
  Acc a;
  a.zero();
  int g = 0;
  for (; g + 4 <= G; g += 4) {
    u64d xv[4], wv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      xv[u] = x[(size_t)(g + u) * ct];
      wv[u] = __ldg(w + (size_t)(g + u) * wstride);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) a.mac(xv[u], wv[u]);
    a.fold();
  }
  for (; g < G; ++g) a.mac(x[(size_t)g * ct], __ldg(w + (size_t)g * wstride));
  return a.reduce(pr);
}

__global__ void __launch_bounds__(kTpb) k_conv_pt(PrimeTable pt, const u64d* __restrict__ taps, int G, int l,
                                                  int N, const u64d* __restrict__ pw,
                                                  const u64d* __restrict__ pbias, u64d* __restrict__ out) {
  // tap ciphertext g carries R taps in disjoint slot regions; pw row g is the
  // sum of their block plaintexts (ConvLayer::make_merged), so one product
  // per tap ciphertext; 40-bit limbs accumulate fold-free (Acc20)
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % l, p = blockIdx.y / l, b = blockIdx.z;
  if (k >= N) return;
  const DevPrime pr = pt.p[t];
  const size_t ct = (size_t)2 * l * N;
  const u64d* x = taps + (size_t)b * G * ct + (size_t)p * l * N + (size_t)t * N + k;
  const u64d* w = pw + (size_t)t * N + k;
  u64d v = pr.q >> 40 ? conv_pt_mac<AccC>(x, w, G, ct, (size_t)l * N, pr)
                      : conv_pt_mac<Acc20>(x, w, G, ct, (size_t)l * N, pr);
  if (p == 0) v = add_mod_d(v, __ldg(pbias + (size_t)t * N + k), pr.q);
  out[(size_t)b * ct + (size_t)p * l * N + (size_t)t * N + k] = v;
}

// masked-constant conv (the RepackConv stage, proj/src/netcompile.cpp:352-379):
//   out[co][b][p][t][k] = sum_s tap[s][b][p][t][k] * P[co][s][t][k] (+ bias[co] on part 0)
// taps tap-major [s][b], outputs map-major [co][b]; one thread per output word
__global__ void __launch_bounds__(kTpb) k_conv_masked(PrimeTable pt, const u64d* __restrict__ taps, int B, int G,
                                                      int l, int N, const u64d* __restrict__ pw,
                                                      const u64d* __restrict__ pbias, u64d* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % l, p = blockIdx.y / l, b = blockIdx.z % B, co = blockIdx.z / B;
  if (k >= N) return;
  const DevPrime pr = pt.p[t];
  const size_t ct = (size_t)2 * l * N;
  const u64d* x = taps + (size_t)b * ct + (size_t)p * l * N + (size_t)t * N + k;
  const u64d* w = pw + (size_t)co * G * l * N + (size_t)t * N + k;
  u64d v = pr.q >> 40 ? conv_pt_mac<AccC>(x, w, G, (size_t)B * ct, (size_t)l * N, pr)
                      : conv_pt_mac<Acc20>(x, w, G, (size_t)B * ct, (size_t)l * N, pr);
  if (p == 0) v = add_mod_d(v, __ldg(pbias + ((size_t)co * l + t) * N + k), pr.q);
  out[((size_t)co * B + b) * ct + (size_t)p * l * N + (size_t)t * N + k] = v;
}

// merge inner product, summed over the G rotated maps of each image:
//   acc[img][p][t] = sum_j sum_d D[img*G + j][d][t] * key_j[d][p][pi(t)]
__global__ void __launch_bounds__(kTpb) k_ks_inner_sum(PrimeTable pt, const u64d* __restrict__ D, int nimg, int G,
                                                       int l, int L, int N, KeyRowMap km,
                                                       u64d* __restrict__ acc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y, i0 = blockIdx.z * kKsKT;
  if (k >= N) return;
  const int pi = t == l ? L : t;
  const DevPrime pr = pt.p[pi];
  const size_t kp = (size_t)(L + 1) * N;
  HEGPU_KS_ACC a0[kKsKT], a1[kKsKT];
#pragma unroll
  for (int bb = 0; bb < kKsKT; ++bb) a0[bb].zero(), a1[bb].zero();
  int cnt = 0;
  for (int j = 0; j < G; ++j) {
    const u64d* key = km.key[j] + (size_t)pi * N + k;
    for (int d = 0; d < l; ++d) {
      const u64d k0 = __ldg(key + (size_t)d * 2 * kp), k1 = __ldg(key + (size_t)d * 2 * kp + kp);
#pragma unroll
      for (int bb = 0; bb < kKsKT; ++bb) {
        const int img = i0 + bb;
        if (img >= nimg) break;
        const u64d x = split31(D[((((size_t)img * G + j) * l + d) * (l + 1) + t) * N + k]);
        a0[bb].mad(x, k0);
        a1[bb].mad(x, k1);
      }
      if ((++cnt & 3) == 0) {
#pragma unroll
        for (int bb = 0; bb < kKsKT; ++bb) a0[bb].fold(), a1[bb].fold();
      }
    }
  }
#pragma unroll
  for (int bb = 0; bb < kKsKT; ++bb) {
    const int img = i0 + bb;
    if (img >= nimg) break;
    u64d* o = acc + ((size_t)img * 2 * (l + 1) + t) * N + k;
    o[0] = a0[bb].reduce(pr);
    o[(size_t)(l + 1) * N] = a1[bb].reduce(pr);
  }
}

// the merge inner sum with the digit count a template parameter (loads of
// one rotation issued together, compile-time strides)
template <int LV>
__global__ void __launch_bounds__(kTpb) k_ks_inner_sum_t(PrimeTable pt, const u64d* __restrict__ D, int nimg, int G,
                                                         int L, int N, KeyRowMap km, u64d* __restrict__ acc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y, img = blockIdx.z;
  if (k >= N || img >= nimg) return;
  const int pi = t == LV ? L : t;
  const DevPrime pr = pt.p[pi];
  const size_t kp = (size_t)(L + 1) * N;
  HEGPU_KS_ACC a0, a1;
  a0.zero();
  a1.zero();
  int cnt = 0;
  for (int j = 0; j < G; ++j) {
    const u64d* key = km.key[j] + (size_t)pi * N + k;
    const u64d* d = D + (((size_t)img * G + j) * LV * (LV + 1) + t) * N + k;
    u64d dv[LV], k0[LV], k1[LV];
#pragma unroll
    for (int q = 0; q < LV; ++q) {
      dv[q] = d[(size_t)q * (LV + 1) * N];
      k0[q] = __ldg(key + (size_t)q * 2 * kp);
      k1[q] = __ldg(key + (size_t)q * 2 * kp + kp);
    }
#pragma unroll
    for (int q = 0; q < LV; ++q) {
      const u64d x = split31(dv[q]);
      a0.mad(x, k0[q]);
      a1.mad(x, k1[q]);
      if (++cnt == 4) a0.fold(), a1.fold(), cnt = 0;
    }
  }
  u64d* o = acc + ((size_t)img * 2 * (LV + 1) + t) * N + k;
  o[0] = a0.reduce(pr);
  o[(size_t)(LV + 1) * N] = a1.reduce(pr);
}

// merge Q-basis part: C0 = map_0.c0 + sum_j sigma_j(map_j.c0), C1 = map_0.c1
__global__ void k_merge_c(PrimeTable pt, const u64d* __restrict__ maps, int nimg, int c, int l, int N,
                          KeyRowMap km, u64d* __restrict__ C) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % l, p = blockIdx.y / l, img = blockIdx.z;
  if (k >= N) return;
  const int S = N >> 1;
  const u64d q = pt.p[t].q;
  const size_t st = (size_t)2 * l * N;
  const u64d* m = maps + (size_t)img * c * st + (size_t)p * l * N + (size_t)t * N;
  u64d v = m[k];
  if (p == 0)
    for (int j = 1; j < c; ++j) v = add_mod_d(v, m[(size_t)j * st + shifted_pos(k, km.shift[j - 1], S)], q);
  C[(size_t)img * st + (size_t)p * l * N + (size_t)t * N + k] = v;
}

// the Q-basis part of one rank's share of a merge (maps lo..lo+M-1 of an
// image, map j rotated by its own offset; kc.shift[j] = 0 for global map 0):
// poly 0 = sum_j sigma_j(c0_j), poly 1 = c1 of global map 0 if this share has it
__global__ void k_merge_c_part(PrimeTable pt, const u64d* __restrict__ maps, int nimg, int M, int has0, int l, int N,
                               KeyRowMap kc, u64d* __restrict__ C) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % l, p = blockIdx.y / l, img = blockIdx.z;
  if (k >= N) return;
  const int S = N >> 1;
  const u64d q = pt.p[t].q;
  const size_t st = (size_t)2 * l * N;
  const u64d* m = maps + (size_t)img * M * st + (size_t)p * l * N + (size_t)t * N;
  u64d v = 0;
  if (p == 0) {
    for (int j = 0; j < M; ++j) v = add_mod_d(v, m[(size_t)j * st + shifted_pos(k, kc.shift[j], S)], q);
  } else if (has0) {
    v = m[k];
  }
  C[(size_t)img * st + (size_t)p * l * N + (size_t)t * N + k] = v;
}

#ifndef HEGPU_CONV_CO
#define HEGPU_CONV_CO 8
#endif

// tap source of the conv MAC: tap s of this thread's (image, poly, limb,
// position) in a full device ciphertext batch
struct TapsFull {
  const u64d* taps;
  __device__ const u64d* addr(int s, int b, int ntaps, int poly, int t, int l, int k, int N) const {
    const size_t ct_words = (size_t)2 * l * N;
    return taps + ((size_t)b * ntaps + s) * ct_words + (size_t)poly * l * N + (size_t)t * N + k;
  }
  __device__ u64d operator()(int s, int b, int ntaps, int poly, int t, int l, int k, int N) const {
    return __ldg(addr(s, b, ntaps, poly, t, l, k, N));
  }
};

#ifndef HEGPU_CONV_STAGE
#define HEGPU_CONV_STAGE 32  // taps per cp.async batch staged per thread in shared memory (0: direct loads)
#endif

// conv-pack MAC (convlower.cpp:39-74): CO output maps per thread, taps
// streamed 4 at a time so each thread keeps independent loads in flight.
template <int CO, class Taps>
__global__ void __launch_bounds__(kTpb) k_conv_mac(PrimeTable pt, Taps taps, int ntaps, int l, int N,
                                                   const u64d* __restrict__ w, int c_out,
                                                   const u64d* __restrict__ bias, u64d* __restrict__ out) {
  extern __shared__ u64d ws[];  // [CO][ntaps] split-31 Montgomery scalars of this (t, group)
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % l, poly = blockIdx.y / l;
  const int groups = (c_out + CO - 1) / CO;
  const int b = blockIdx.z / groups, cg = blockIdx.z % groups;
  const int nco = c_out - cg * CO < CO ? c_out - cg * CO : CO;
  for (int e = threadIdx.x; e < CO * ntaps; e += blockDim.x) {
    const int c = e / ntaps, s = e % ntaps;
    ws[e] = c < nco ? __ldg(w + ((size_t)(cg * CO + c) * ntaps + s) * l + t) : 0ull;
  }
  __syncthreads();
  if (k >= N) return;
  const DevPrime pr = pt.p[t];
  const size_t ct_words = (size_t)2 * l * N;
  auto tap = [&](int s) -> u64d { return taps(s, b, ntaps, poly, t, l, k, N); };
  AccC acc[CO];
#pragma unroll
  for (int c = 0; c < CO; ++c) acc[c].zero();
  int s = 0;
#if HEGPU_CONV_STAGE
  // every tap word of this thread is fetched with cp.async into its own
  // shared-memory slots (no register cost, all loads in flight at once)
  u64d* stg = ws + CO * ntaps + threadIdx.x;
  for (int s0 = 0; s0 < ntaps; s0 += HEGPU_CONV_STAGE) {
    const int s1 = min(ntaps, s0 + HEGPU_CONV_STAGE);
    for (int q = s0; q < s1; ++q)
      cp_async8(stg + (q - s0) * blockDim.x, taps.addr(q, b, ntaps, poly, t, l, k, N));
    cp_async_wait_all();
    for (s = s0; s + 4 <= s1; s += 4) {
      u64d x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = split31(stg[(s + u - s0) * blockDim.x]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int c = 0; c < CO; ++c) acc[c].mad(x[u], ws[c * ntaps + s + u]);
#pragma unroll
      for (int c = 0; c < CO; ++c) acc[c].fold();
    }
    for (; s < s1; ++s) {
      const u64d x = split31(stg[(s - s0) * blockDim.x]);
#pragma unroll
      for (int c = 0; c < CO; ++c) acc[c].mad(x, ws[c * ntaps + s]);
#pragma unroll
      for (int c = 0; c < CO; ++c) acc[c].fold();
    }
  }
  s = ntaps;
#endif
  // 4 taps in flight per thread; fold every 4 products
  for (; s + 4 <= ntaps; s += 4) {
    u64d x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = split31(tap(s + u));
    // tap-major: the CO accumulators advance in turn (independent chains)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < CO; ++c) acc[c].mad(x[u], ws[c * ntaps + s + u]);
#pragma unroll
    for (int c = 0; c < CO; ++c) acc[c].fold();
  }
  for (; s < ntaps; ++s) {
    const u64d x = split31(tap(s));
#pragma unroll
    for (int c = 0; c < CO; ++c) acc[c].mad(x, ws[c * ntaps + s]);
  }
#pragma unroll
  for (int c = 0; c < CO; ++c) {
    if (c >= nco) break;
    const int co = cg * CO + c;
    u64d v = acc[c].reduce(pr);
    if (poly == 0 && bias)
      v = add_mod_d(v, mont_mul(bias[((size_t)co * l + t) * N + k], 1ull, pr.q, pr.qneg_inv), pr.q);
    out[((size_t)b * c_out + co) * ct_words + (size_t)poly * l * N + (size_t)t * N + k] = v;
  }
}

// ---------------------------------------------------------------------------
// Halevi-Shoup diagonal accumulation over the hoisted ModUp digits D of v.c1
// (DESIGN.md §4.3).  Diagonal i rotates right by r_i; its Galois key is
// pre-multiplied by the (pre-rotated) mask, so per output word and image the
// work is a pure 192-bit multiply-accumulate:
//   acc[p][t]  += sum_j D_j[k - r_i] * (key_i[j][p][t] * m_i[t])[k]   (r_i > 0)
//   cacc[0][t] += c0[k - r_i] * m_i[t][k]                              (t < l)
//   r_i == 0   : cacc[p][t] += c_p[k] * m_0[t][k]
// The diagonals of a chunk have r in [r_lo, r_hi] (< KB + CW positions), so
// the CTA stages the D / c0 window of its k-block in shared memory once and
// every diagonal of the chunk reads it from there.
constexpr int kHsKB = 128;  // output positions per CTA
constexpr int kHsCW = 128;  // max r span of a chunk
#ifndef HEGPU_HS_BT
#define HEGPU_HS_BT 4
#endif
#ifndef HEGPU_HS_MINB
#define HEGPU_HS_MINB 4
#endif
#ifndef HEGPU_HS_ACC
#define HEGPU_HS_ACC AccC  // accumulator of the HS kernel (AccW: no in-loop folds)
#endif
#ifndef HEGPU_HS_PD1
#define HEGPU_HS_PD1 4  // cp.async prefetch depth (diagonals) at 1 image per thread (measured 4 > 8 > 16 > 0)
#endif
#ifndef HEGPU_HS_PD2
#define HEGPU_HS_PD2 8  // ... at 2 images per thread (measured 8 = 16 > 4 > 0)
#endif
constexpr int kHsBTMax = HEGPU_HS_BT;  // images per thread (smaller batches use 2 or 1)

// PD > 0 (small batches, where the fused keys stream from HBM once per use):
// each thread keeps the fused-key words of the next PD - 1 diagonals in
// flight with cp.async into its own shared-memory ring slots
template <int LV, int kHsBT, int PD, class Acc>
__device__ __forceinline__ void hs_diag_body(PrimeTable& pt, const u64d* __restrict__ v,
                                             const u64d* __restrict__ D, int B, int L, int N,
                                             const HsDiagTable& tab, u64d* __restrict__ acc,
                                             u64d* __restrict__ cacc, int gsplit, size_t part_acc,
                                             size_t part_cacc) {
  extern __shared__ u64d win[];  // [BT][LV + 1][kHsW], Acc::prep words (split-31, or plain for Acc20)
  constexpr int kW = kHsKB + kHsCW;  // window row stride (compile-time -> immediate LDS offsets)
  const int S = N >> 1;
  // blockIdx.x = image tile * gsplit + diagonal group: with few images the
  // diagonal chunks are split over gsplit CTAs writing partial sums
  const int g = blockIdx.x % gsplit;
  const int kb = blockIdx.y, t = blockIdx.z >> 1, p = blockIdx.z & 1, b0 = (blockIdx.x / gsplit) * kHsBT;
  acc += (size_t)g * part_acc;
  cacc += (size_t)g * part_cacc;
  const int ch_lo = (int)((long)tab.nchunk * g / gsplit), ch_hi = (int)((long)tab.nchunk * (g + 1) / gsplit);
  const int k0 = kb * kHsKB, k = k0 + threadIdx.x;
  const int half = k0 >= S ? S : 0;
  const int pi = t == LV ? L : t;
  const DevPrime pr = pt.p[pi];
  const bool has_c = t < LV;
  const bool do_c0 = has_c && p == 0;
  const int nrow = do_c0 ? LV + 1 : LV;  // D digits (+ c0)
  const int ln = LV * N, kp = (LV + 1) * N;

  Acc a[kHsBT], c[kHsBT];
#pragma unroll
  for (int bb = 0; bb < kHsBT; ++bb) a[bb].zero(), c[bb].zero();

  const u64d* mrow = tab.masks + (size_t)t * N + k;
  for (int ch = ch_lo; ch < ch_hi; ++ch) {
    const int i0 = __ldg(tab.chunk + ch), i1 = __ldg(tab.chunk + ch + 1);
    const int r_lo = __ldg(tab.r + i0), r_hi = __ldg(tab.r + i1 - 1);
    const int W = kHsKB + r_hi - r_lo;
    // stage window positions k0 - r_hi + w (mod S, inside this half), split
    __syncthreads();
    for (int row = 0; row < kHsBT * nrow; ++row) {
      const int bb = row / nrow, rr = row % nrow, b = b0 + bb;
      const u64d* src = b >= B ? nullptr
                        : rr < LV ? D + (((size_t)b * LV + rr) * (LV + 1) + t) * N
                                  : v + (size_t)b * 2 * ln + (size_t)t * N;
      u64d* dst = win + (bb * (LV + 1) + rr) * kW;
      for (int w = threadIdx.x; w < W; w += kHsKB) {
        int pos = k0 - half - r_hi + w;
        if (pos < 0) pos += S;
        dst[w] = src ? Acc::prep(src[half + pos]) : 0ull;
      }
    }
    __syncthreads();
    const u64d* wb = win + threadIdx.x + r_hi;
    // software pipeline: the fused-key words and mask of diagonal i + 1 are
    // in flight while diagonal i is accumulated (addresses are arithmetic:
    // no load feeds another load's address)
    const u64d* fkb = tab.fk + p * kp + t * N + k;
    u64d* ring = win + kHsBT * (LV + 1) * kW + threadIdx.x;  // [PD][LV + 1][KB]
    auto issue = [&](int i) {
      u64d* slot = ring + (i % (PD > 0 ? PD : 1)) * (LV + 1) * kHsKB;
      if (i >= tab.first_keyed) {
        const u64d* fk = fkb + (size_t)(i - tab.first_keyed) * tab.fk_words;
#pragma unroll
        for (int j = 0; j < LV; ++j) cp_async8(slot + j * kHsKB, fk + j * 2 * kp);
      }
      if (do_c0) cp_async8(slot + LV * kHsKB, mrow + (size_t)i * kp);
    };
    if constexpr (PD > 0) {
#pragma unroll
      for (int d = 0; d < PD - 1; ++d) {
        if (i0 + d < i1) issue(i0 + d);
        cp_async_commit();
      }
    }
    u64d kn[LV], mn = 0;
    int rn = __ldg(tab.r + i0);
    if constexpr (PD == 0) {
      const u64d* fk = fkb + (size_t)(i0 - tab.first_keyed) * tab.fk_words;
#pragma unroll
      for (int j = 0; j < LV; ++j) kn[j] = i0 >= tab.first_keyed ? __ldg(fk + j * 2 * kp) : 0ull;
      if (do_c0) mn = __ldg(mrow + (size_t)i0 * kp);
    }
    for (int i = i0; i < i1; ++i) {
      u64d kv[LV];
      u64d m;
      int r;
      if constexpr (PD > 0) {
        if (i + PD - 1 < i1) issue(i + PD - 1);
        cp_async_commit();
        cp_async_wait<(PD > 0 ? PD - 1 : 0)>();
        const u64d* slot = ring + (i % (PD > 0 ? PD : 1)) * (LV + 1) * kHsKB;
#pragma unroll
        for (int j = 0; j < LV; ++j) kv[j] = slot[j * kHsKB];
        m = do_c0 ? slot[LV * kHsKB] : 0ull;
        r = __ldg(tab.r + i);
      } else {
      r = rn;
#pragma unroll
      for (int j = 0; j < LV; ++j) kv[j] = kn[j];
      m = mn;
      if (i + 1 < i1) {
        rn = __ldg(tab.r + i + 1);
        const u64d* fk = fkb + (size_t)(i + 1 - tab.first_keyed) * tab.fk_words;
#pragma unroll
        for (int j = 0; j < LV; ++j) kn[j] = __ldg(fk + j * 2 * kp);  // i + 1 >= 1 >= first_keyed
        if (do_c0) mn = __ldg(mrow + (size_t)(i + 1) * kp);
      }
      }
      const u64d* wp = wb - r;  // + (bb * (LV + 1) + row) * kW, compile-time below
      if (do_c0) {
#pragma unroll
        for (int bb = 0; bb < kHsBT; ++bb) c[bb].macw(wp[(bb * (LV + 1) + LV) * kW], m);
      }
      if (r != 0) {
        // digit-major: the BT accumulators advance in turn (independent
        // chains; image-major measured 6% slower)
#pragma unroll
        for (int j = 0; j < LV; ++j) {
#pragma unroll
          for (int bb = 0; bb < kHsBT; ++bb) {
            a[bb].macw(wp[(bb * (LV + 1) + j) * kW], kv[j]);
            if ((j & 3) == 3) a[bb].fold();
          }
        }
        if (LV & 3) {
#pragma unroll
          for (int bb = 0; bb < kHsBT; ++bb) a[bb].fold();
        }
      }
      if (do_c0 && ((i - i0) & 3) == 3) {
#pragma unroll
        for (int bb = 0; bb < kHsBT; ++bb) c[bb].fold();
      }
    }
#pragma unroll
    for (int bb = 0; bb < kHsBT; ++bb) c[bb].fold();
  }
  // r == 0 diagonal (if kept) is the only contributor to the c1 part
  u64d m0 = 0;
  const bool c1_term = has_c && p == 1 && g == 0 && tab.own_c1 && tab.ndiag > 0 && __ldg(tab.r) == 0;
  if (c1_term) m0 = unsplit31(__ldg(tab.masks + (size_t)t * N + k));
#pragma unroll
  for (int bb = 0; bb < kHsBT; ++bb) {
    const int b = b0 + bb;
    if (b >= B) break;
    acc[(size_t)b * 2 * kp + (size_t)p * kp + (size_t)t * N + k] = a[bb].reduce(pr);
    if (has_c) {
      u64d* cb = cacc + (size_t)b * 2 * ln + (size_t)p * ln + (size_t)t * N + k;
      if (p == 0) *cb = c[bb].reduce(pr);
      else *cb = c1_term ? mont_mul(v[(size_t)b * 2 * ln + ln + (size_t)t * N + k], m0, pr.q, pr.qneg_inv) : 0ull;
    }
  }
}

template <int LV, int kHsBT, int PD>
__global__ void __launch_bounds__(kHsKB, HEGPU_HS_MINB) k_hs_diag(PrimeTable pt, const u64d* __restrict__ v,
                                                   const u64d* __restrict__ D, int B, int L, int N,
                                                   HsDiagTable tab, u64d* __restrict__ acc,
                                                   u64d* __restrict__ cacc, int gsplit, size_t part_acc,
                                                   size_t part_cacc) {
  // limbs of 40-bit primes accumulate fold-free in Acc20 (CTA-uniform)
  const int t = blockIdx.z >> 1;
  if (pt.p[t == LV ? L : t].q >> 40)
    hs_diag_body<LV, kHsBT, PD, HEGPU_HS_ACC>(pt, v, D, B, L, N, tab, acc, cacc, gsplit, part_acc, part_cacc);
  else
    hs_diag_body<LV, kHsBT, PD, Acc20>(pt, v, D, B, L, N, tab, acc, cacc, gsplit, part_acc, part_cacc);
}

// narrow diagonal bands (a few rotations, e.g. the 10-row output layer):
// one thread per (image, limb, position) for both key parts, every operand
// read straight from L1/L2 (consecutive positions -> coalesced; a warp of 32
// positions x 8 images per CTA shares each fused-key word), no window
// staging -- the windowed kernel exposed its staging latency at 16 warps/SM
template <int LV, int IPT, bool UNIT, class Acc>
__device__ __forceinline__ void hs_narrow_body(const DevPrime& pr, const u64d* __restrict__ v,
                                               const u64d* __restrict__ D, int B, int N, const HsDiagTable& tab,
                                               u64d* __restrict__ acc, u64d* __restrict__ cacc, int k, int b0, int t) {
  const int S = N >> 1, half = k >= S ? S : 0, kh = k - half;
  const bool has_c = t < LV;
  const size_t kp = (size_t)(LV + 1) * N, ln = (size_t)LV * N;
  const u64d* Db[IPT];
  const u64d* c0[IPT];
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int b = b0 + q < B ? b0 + q : B - 1;  // (extra lanes recompute the last image, not stored)
    Db[q] = D + ((size_t)b * LV * (LV + 1) + t) * N + half;
    c0[q] = v + (size_t)b * 2 * ln + (size_t)t * N + half;
  }
  Acc a0[IPT], a1[IPT], cc[IPT];
  u64d cs[IPT];
#pragma unroll
  for (int q = 0; q < IPT; ++q) a0[q].zero(), a1[q].zero(), cc[q].zero(), cs[q] = 0;
  int na = 0, nc = 0;
  const int i0 = __ldg(tab.chunk), i1 = __ldg(tab.chunk + tab.nchunk);  // absolute diagonal range
  for (int i = i0; i < i1; ++i) {
    const int r = __ldg(tab.r + i), pos = (kh - r) & (S - 1);
    if (r != 0) {
      const u64d* fk = tab.fk + (size_t)(i - tab.first_keyed) * tab.fk_words + (size_t)t * N + k;
      u64d k0[LV], k1[LV], d[IPT][LV];
#pragma unroll
      for (int j = 0; j < LV; ++j) {
        k0[j] = __ldg(fk + (size_t)(j * 2) * kp);
        k1[j] = __ldg(fk + (size_t)(j * 2 + 1) * kp);
#pragma unroll
        for (int q = 0; q < IPT; ++q) d[q][j] = Db[q][(size_t)j * kp + pos];
      }
#pragma unroll
      for (int j = 0; j < LV; ++j) {
#pragma unroll
        for (int q = 0; q < IPT; ++q) {
          a0[q].mac(d[q][j], k0[j]);
          a1[q].mac(d[q][j], k1[j]);
        }
        if (std::is_same<Acc, AccC>::value && ++na == 4) {
#pragma unroll
          for (int q = 0; q < IPT; ++q) a0[q].fold(), a1[q].fold();
          na = 0;
        }
      }
    }
    if (has_c) {
      if constexpr (UNIT) {
#pragma unroll
        for (int q = 0; q < IPT; ++q) cs[q] = add_mod_d(cs[q], c0[q][pos], pr.q);
      } else {
        const u64d m = __ldg(tab.masks + ((size_t)i * (LV + 1) + t) * N + k);
#pragma unroll
        for (int q = 0; q < IPT; ++q) cc[q].mac(c0[q][pos], m);
        if (std::is_same<Acc, AccC>::value && ++nc == 4) {
#pragma unroll
          for (int q = 0; q < IPT; ++q) cc[q].fold();
          nc = 0;
        }
      }
    }
  }
  const bool c1_term = has_c && tab.own_c1 && tab.ndiag > 0 && __ldg(tab.r) == 0;
  const u64d m0 = c1_term && !UNIT ? unsplit31(__ldg(tab.masks + (size_t)t * N + k)) : 0ull;
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int b = b0 + q;
    if (b >= B) break;
    u64d* o = acc + (size_t)b * 2 * kp + (size_t)t * N + k;
    o[0] = a0[q].reduce(pr);
    o[kp] = a1[q].reduce(pr);
    if (has_c) {
      u64d* cb = cacc + (size_t)b * 2 * ln + (size_t)t * N + k;
      cb[0] = UNIT ? cs[q] : cc[q].reduce(pr);
      const u64d c1 = v[(size_t)b * 2 * ln + ln + (size_t)t * N + k];
      cb[ln] = !c1_term ? 0ull : UNIT ? c1 : mont_mul(c1, m0, pr.q, pr.qneg_inv);
    }
  }
}

template <int LV, int IPT, bool UNIT, int NC>
#ifndef HEGPU_NARROW_WARPS
#define HEGPU_NARROW_WARPS 4  // image warps per CTA (measured 1: 0.459, 2: 0.451, 4: 0.454, 8: 0.490, 16: 0.621 ms)
#endif
__global__ void __launch_bounds__(32 * HEGPU_NARROW_WARPS) k_hs_narrow(PrimeTable pt, const u64d* __restrict__ v,
                                                   const u64d* __restrict__ D, int B, int L, int n_rt, HsDiagTable tab,
                                                   u64d* __restrict__ acc, u64d* __restrict__ cacc) {
  // IPT images per thread share every fused-key word (register reuse);
  // UNIT: all masks are 1 (the fold's rotation sum) -> the c0 part is a sum;
  // limbs of a 40-bit prime accumulate fold-free in Acc20 (CTA-uniform branch);
  // NC: compile-time ring degree (0 = runtime) -> per-digit offsets fold
  // into the loads' immediates
  const int N = NC ? NC : n_rt;
  const int k = blockIdx.x * 32 + (threadIdx.x & 31), b0 = (blockIdx.y * HEGPU_NARROW_WARPS + (threadIdx.x >> 5)) * IPT;
  const int t = blockIdx.z;
  if (k >= N || b0 >= B) return;
  const int pi = t == LV ? L : t;
  const DevPrime pr = pt.p[pi];
  if (pr.q >> 40) hs_narrow_body<LV, IPT, UNIT, AccC>(pr, v, D, B, N, tab, acc, cacc, k, b0, t);
  else hs_narrow_body<LV, IPT, UNIT, Acc20>(pr, v, D, B, N, tab, acc, cacc, k, b0, t);
}

// fused key: fk[j][p][t] = key[j][p][pi(t)] * m[t]   (t over the ext basis);
// key, mask and result are split-31 Montgomery words
__global__ void k_fuse_key(PrimeTable pt, const u64d* __restrict__ key, const u64d* __restrict__ m, int l, int L,
                           int N, u64d* __restrict__ fk) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % (l + 1), jp = blockIdx.y / (l + 1);  // jp = j * 2 + p
  if (k >= N) return;
  const int pi = t == l ? L : t;
  const DevPrime pr = pt.p[pi];
  const u64d kv = unsplit31(key[((size_t)jp * (L + 1) + pi) * N + k]);
  const u64d mv = unsplit31(m[(size_t)t * N + k]);
  fk[((size_t)jp * (l + 1) + t) * N + k] = split31(mont_mul(kv, mv, pr.q, pr.qneg_inv));
}

// out[i] = sum_g part[g][i] mod q(limb of i); rows of nl limbs, limb p_limb -> P
__global__ void k_sum_parts(PrimeTable pt, const u64d* __restrict__ part, u64d* __restrict__ out, size_t n,
                            int gs, int nl, int p_limb, int L, int N) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int limb = (int)((i / N) % nl);
    const u64d q = pt.p[limb == p_limb ? L : limb].q;
    u64d s = part[i];
    for (int g = 1; g < gs; ++g) s = add_mod_d(s, part[(size_t)g * n + i], q);
    out[i] = s;
  }
}

// exact x mod q per word; rows of nl limbs, limb p_limb -> P
__global__ void k_reduce_rows(PrimeTable pt, u64d* __restrict__ p, size_t n, int nl, int p_limb, int L, int N) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const int limb = (int)((i / N) % nl);
    const DevPrime pr = pt.p[limb == p_limb ? L : limb];
    u64d v = reduce_lazy4(p[i], pr);
    if (v >= 2 * pr.q) v -= 2 * pr.q;
    if (v >= pr.q) v -= pr.q;
    p[i] = v;
  }
}

// in-place split-31 re-packing of Montgomery multiplier tables
__global__ void k_split31(u64d* __restrict__ p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = split31(p[i]);
}

unsigned grid_for(size_t total) {
  size_t g = (total + kTpb - 1) / kTpb;
  return (unsigned)(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

template <int LV, int kHsBT, int PD>
void launch_hs_lvbt(Context& c, const u64d* v, int B, const u64d* D, const HsDiagTable& t, u64d* acc, u64d* cacc) {
  const int N = c.N(), S = N / 2;
  if (S < kHsKB) fail(HEGPU_ERR_ARG, "hs_matvec on the device needs N >= 256");
  dim3 grid((B + kHsBT - 1) / kHsBT, N / kHsKB, 2 * (LV + 1));
  const size_t sm = ((size_t)kHsBT * (LV + 1) * (kHsKB + kHsCW) + (size_t)PD * (LV + 1) * kHsKB) * 8;
  static size_t done_dev[64] = {0}; size_t& done = done_dev[current_device() & 63];
  if (sm > 48 * 1024 && sm > done) {
    CK(cudaFuncSetAttribute(k_hs_diag<LV, kHsBT, PD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    done = sm;
  }
  // fused keys + masks (c-part limbs) once; v, D read once; acc, cacc written once
  const double NB = 8.0 * N;
  const double bytes = NB * (t.keyed * LV * 2.0 * (LV + 1) + t.ndiag * LV + B * (LV * (LV + 1.0) + 2.0 * LV) +
                             B * (2.0 * (LV + 1) + 2.0 * LV));
  // multiply-accumulates: keyed diagonals x digits x ext limbs x 2, plus c0 x mask
  const double ops = (double)N * B * (t.keyed * LV * (LV + 1) * 2.0 + t.ndiag * LV);
  // small batches: split the diagonal chunks over more CTAs (partial sums)
  const int base = (int)(grid.x * grid.y * grid.z), target = 148 * 32;
  int gsplit = 1;
  if (base < target && t.nchunk > 1) gsplit = std::min(t.nchunk, (target + base - 1) / base);
  if (gsplit == 1) {
    LAUNCH_BO(c, "k_hs_diag", bytes, ops,
             k_hs_diag<LV, kHsBT, PD><<<grid, kHsKB, sm, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc, 1, 0, 0));
    return;
  }
  const size_t acc_w = (size_t)B * 2 * (LV + 1) * N, cacc_w = (size_t)B * 2 * LV * N;
  u64d* pa = c.alloc(gsplit * acc_w);
  u64d* pc = c.alloc(gsplit * cacc_w);
  grid.x *= gsplit;
  LAUNCH_BO(c, "k_hs_diag", bytes, ops,
           k_hs_diag<LV, kHsBT, PD><<<grid, kHsKB, sm, c.stream>>>(c.primes, v, D, B, c.L(), N, t, pa, pc, gsplit, acc_w,
                                                         cacc_w));
  LAUNCH_B(c, "k_sum_parts", 8.0 * (gsplit + 1) * acc_w,
           k_sum_parts<<<grid_for(acc_w), kTpb, 0, c.stream>>>(c.primes, pa, acc, acc_w, gsplit, LV + 1, LV, c.L(), N));
  LAUNCH_B(c, "k_sum_parts", 8.0 * (gsplit + 1) * cacc_w,
           k_sum_parts<<<grid_for(cacc_w), kTpb, 0, c.stream>>>(c.primes, pc, cacc, cacc_w, gsplit, LV, -1, c.L(), N));
  c.free(pa);
  c.free(pc);
}

// images per thread: 4 for batches >= 4 (fused keys reused 4x), else the
// batch itself (B = 1 would otherwise compute 3 zero images per thread)
template <int LV>
void launch_hs_lv(Context& c, const u64d* v, int B, const u64d* D, const HsDiagTable& t, u64d* acc, u64d* cacc) {
  if (B >= kHsBTMax) launch_hs_lvbt<LV, kHsBTMax, 0>(c, v, B, D, t, acc, cacc);
  else if (B >= 2) launch_hs_lvbt<LV, 2, HEGPU_HS_PD2>(c, v, B, D, t, acc, cacc);
  else launch_hs_lvbt<LV, 1, HEGPU_HS_PD1>(c, v, B, D, t, acc, cacc);
}

}  // namespace

int hs_chunk_span() { return kHsCW; }

void launch_add(Context& c, const u64d* a, const u64d* b, u64d* out, int count, int l) {
  const size_t total = (size_t)count * 2 * l * c.N();
  LAUNCH_B(c, "k_add", 24.0 * total, k_add<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, b, out, total, l, c.N()));
}

void launch_add_plain(Context& c, const u64d* a, const u64d* p, long p_stride, u64d* out, int count, int l) {
  const size_t total = (size_t)count * 2 * l * c.N();
  LAUNCH_B(c, "k_add_plain", 16.0 * total + 4.0 * total / count,
         k_add_plain<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, p, p_stride, out, total, l, c.N()));
}

void launch_mul_plain(Context& c, const u64d* a, const u64d* p, long p_stride, u64d* out, int count, int l) {
  const size_t total = (size_t)count * 2 * l * c.N();
  LAUNCH_B(c, "k_mul_plain", 16.0 * total + 4.0 * total / count,
         k_mul_plain<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, p, p_stride, out, total, l, c.N()));
}

void launch_tensor_square(Context& c, const u64d* a, u64d* d01, u64d* d2, int count, int l) {
  const size_t total = (size_t)count * l * c.N();
  LAUNCH_B(c, "k_tensor_square", 40.0 * total,
         k_tensor_square<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, d01, d2, total, l, c.N()));
}

void ks_inner(Context& c, const u64d* D, int B, int l, const KeyRowMap& keys, u64d* acc) {
  c.ks[KS_INNER] += B;
  const int per = keys.period, rows_per_key = (B + per - 1) / per;
  const int tiles = (rows_per_key + kKsKT - 1) / kKsKT;
  dim3 grid((c.N() + kTpb - 1) / kTpb, l + 1, per * tiles);
  double kb = 0;  // distinct keys read once each
  for (int i = 0; i < per && i < B; ++i) kb += 8.0 * l * 2 * (l + 1) * c.N();
  const size_t sm = (HEGPU_KS_STAGE && kKsKT == 1) ? (size_t)3 * l * kTpb * 8 : 0;
  static size_t done_dev[64] = {0}; size_t& done = done_dev[current_device() & 63];
  if (sm > 48 * 1024 && sm > done) {
    CK(cudaFuncSetAttribute(k_ks_inner, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    done = sm;
  }
  const double kbytes = 8.0 * B * (l + 2) * (l + 1) * c.N() + kb, kops = 2.0 * B * l * (l + 1) * c.N();
  if (kKsKT == 1 && !HEGPU_KS_STAGE && l <= 8) {
#define KSI_GO(LV) \
  case LV: \
    LAUNCH_BO(c, "k_ks_inner", kbytes, kops, \
              k_ks_inner_t<LV><<<grid, kTpb, 0, c.stream>>>(c.primes, D, B, c.L(), c.N(), keys, acc)); \
    break;
    switch (l) { KSI_GO(1) KSI_GO(2) KSI_GO(3) KSI_GO(4) KSI_GO(5) KSI_GO(6) KSI_GO(7) KSI_GO(8) }
#undef KSI_GO
    return;
  }
  LAUNCH_BO(c, "k_ks_inner", kbytes, kops,
           k_ks_inner<<<grid, kTpb, sm, c.stream>>>(c.primes, D, B, l, c.L(), c.N(), keys, acc));
}

template <class Taps>
void launch_conv_mac_t(Context& c, const Taps& taps, double tap_bytes, int B, int ntaps, int l, const u64d* w,
                       int c_out, const u64d* bias, u64d* out) {
  // taps read once, maps written once, bias plaintexts read once
  const double bytes = tap_bytes + 8.0 * c.N() * l * (2.0 * B * c_out + c_out);
  const int co = c_out < HEGPU_CONV_CO ? c_out : HEGPU_CONV_CO;  // output maps per thread
  dim3 grid((c.N() + kTpb - 1) / kTpb, 2 * l, B * ((c_out + co - 1) / co));
  const size_t sm = (size_t)co * ntaps * 8 + (size_t)HEGPU_CONV_STAGE * kTpb * 8;
  if (sm > 200 * 1024) fail(HEGPU_ERR_CAPACITY, "conv_packed_forward: too many taps");
#define CONV_GO(CO)                                                                                        \
  case CO: {                                                                                               \
    static size_t done_dev[64] = {0}; size_t& done = done_dev[current_device() & 63];                                                                                \
    if (sm > 48 * 1024 && sm > done) {                                                                     \
      CK(cudaFuncSetAttribute(k_conv_mac<CO, Taps>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
      done = sm;                                                                                           \
    }                                                                                                      \
    LAUNCH_BO(c, "k_conv_mac", bytes, 2.0 * c.N() * l * B * ntaps * c_out,                                 \
             k_conv_mac<CO, Taps><<<grid, kTpb, sm, c.stream>>>(c.primes, taps, ntaps, l, c.N(), w, c_out, bias, out)); \
    break;                                                                                                 \
  }
  switch (co) {
    CONV_GO(1) CONV_GO(2) CONV_GO(3) CONV_GO(4) CONV_GO(5) CONV_GO(6) CONV_GO(7) CONV_GO(8)
    default: fail(HEGPU_ERR_ARG, "conv: bad c_out");
  }
#undef CONV_GO
}

void launch_conv_pt(Context& c, const u64d* taps, int B, int ntaps, int regions, int l, const u64d* pw,
                    const u64d* pbias, u64d* out) {
  const int N = c.N(), G = (ntaps + regions - 1) / regions;
  dim3 grid((N + kTpb - 1) / kTpb, 2 * l, B);
  // tap ciphertexts once, per-ciphertext weights + bias once, outputs once
  const double bytes = 8.0 * N * l * (2.0 * B * G + G + 1 + 2.0 * B);
  LAUNCH_BO(c, "k_conv_mac", bytes, 2.0 * N * l * B * G,
            k_conv_pt<<<grid, kTpb, 0, c.stream>>>(c.primes, taps, G, l, N, pw, pbias, out));
}

void launch_conv_masked(Context& c, const u64d* taps, int B, int ntaps, int c_out, int l, const u64d* pw,
                        const u64d* pbias, u64d* out) {
  const int N = c.N();
  if ((size_t)B * c_out > 65535) fail(HEGPU_ERR_ARG, "conv_masked: batch * maps exceeds the grid");
  dim3 grid((N + kTpb - 1) / kTpb, 2 * l, B * c_out);
  // per output word: the taps and the map's plaintexts once, the output once
  const double bytes = 8.0 * N * l * (2.0 * B * ntaps * c_out + (double)ntaps * c_out + c_out + 2.0 * B * c_out);
  LAUNCH_BO(c, "k_conv_mac", bytes, 2.0 * N * l * B * ntaps * c_out,
            k_conv_masked<<<grid, kTpb, 0, c.stream>>>(c.primes, taps, B, ntaps, l, N, pw, pbias, out));
}

void launch_conv_mac(Context& c, const u64d* taps, int B, int ntaps, int l, const u64d* w, int c_out,
                     const u64d* bias, u64d* out) {
  launch_conv_mac_t(c, TapsFull{taps}, 8.0 * c.N() * l * 2.0 * B * ntaps, B, ntaps, l, w, c_out, bias, out);
}

void launch_reduce_rows(Context& c, u64d* p, size_t words, int nl, int p_limb) {
  if (!words) return;
  LAUNCH_B(c, "k_reduce_rows", 16.0 * words,
           k_reduce_rows<<<grid_for(words), kTpb, 0, c.stream>>>(c.primes, p, words, nl, p_limb, c.L(), c.N()));
}

void launch_split31(Context& c, u64d* p, size_t words) {
  if (!words) return;
  LAUNCH_B(c, "k_split31", 16.0 * words, k_split31<<<grid_for(words), kTpb, 0, c.stream>>>(p, words));
}

void launch_fuse_key(Context& c, const u64d* key, const u64d* mask, int l, u64d* fk) {
  dim3 grid((c.N() + kTpb - 1) / kTpb, 2 * l * (l + 1));
  LAUNCH(c, "k_fuse_key", k_fuse_key<<<grid, kTpb, 0, c.stream>>>(c.primes, key, mask, l, c.L(), c.N(), fk));
}

void launch_hs_diag(Context& c, const u64d* v, int B, int l, const u64d* D, const HsDiagTable& t, u64d* acc,
                    u64d* cacc) {
  static const int narrow_max = [] {
    const char* e = getenv("HEGPU_HS_NARROW");
    return e ? atoi(e) : 32;
  }();
  if (t.ndiag <= narrow_max && l <= 8) {
    const int N = c.N();
    constexpr int IPT = 1;
    constexpr int NW = HEGPU_NARROW_WARPS;
    dim3 grid((N + 31) / 32, (B + NW * IPT - 1) / (NW * IPT), l + 1);
    const double NB = 8.0 * N;
    const double bytes = NB * (t.keyed * l * 2.0 * (l + 1) + t.ndiag * l + B * (l * (l + 1.0) + 2.0 * l) +
                               B * (2.0 * (l + 1) + 2.0 * l));
    const double ops = (double)N * B * (t.keyed * l * (l + 1) * 2.0 + t.ndiag * l);
#define NARROW_GO(LV)                                                                                        \
  case LV:                                                                                                   \
    if (t.unit_masks)                                                                                        \
      LAUNCH_BO(c, "k_hs_diag", bytes, ops,                                                                  \
                (N == 8192 ? k_hs_narrow<LV, IPT, true, 8192><<<grid, 32 * NW, 0, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc) \
                 : N == 16384 ? k_hs_narrow<LV, IPT, true, 16384><<<grid, 32 * NW, 0, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc) \
                           : k_hs_narrow<LV, IPT, true, 0><<<grid, 32 * NW, 0, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc))); \
    else                                                                                                     \
      LAUNCH_BO(c, "k_hs_diag", bytes, ops,                                                                  \
                (N == 8192 ? k_hs_narrow<LV, IPT, false, 8192><<<grid, 32 * NW, 0, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc) \
                 : N == 16384 ? k_hs_narrow<LV, IPT, false, 16384><<<grid, 32 * NW, 0, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc) \
                           : k_hs_narrow<LV, IPT, false, 0><<<grid, 32 * NW, 0, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc))); \
    return;
    switch (l) { NARROW_GO(1) NARROW_GO(2) NARROW_GO(3) NARROW_GO(4) NARROW_GO(5) NARROW_GO(6) NARROW_GO(7) NARROW_GO(8) }
#undef NARROW_GO
  }
  switch (l) {
    case 1: launch_hs_lv<1>(c, v, B, D, t, acc, cacc); break;
    case 2: launch_hs_lv<2>(c, v, B, D, t, acc, cacc); break;
    case 3: launch_hs_lv<3>(c, v, B, D, t, acc, cacc); break;
    case 4: launch_hs_lv<4>(c, v, B, D, t, acc, cacc); break;
    case 5: launch_hs_lv<5>(c, v, B, D, t, acc, cacc); break;
    case 6: launch_hs_lv<6>(c, v, B, D, t, acc, cacc); break;
    case 7: launch_hs_lv<7>(c, v, B, D, t, acc, cacc); break;
    case 8: launch_hs_lv<8>(c, v, B, D, t, acc, cacc); break;
    default: fail(HEGPU_ERR_ARG, "hs_matvec: level above 8 not supported");
  }
}

// ---------------------------------------------------------------- compositions
void eval_rescale(Context& c, const CtBatch& a, CtBatch& out) {
  const int l = a.level, N = c.N(), B = a.count;
  u64d* tmpP = c.alloc((size_t)B * 2 * N);
  DropArgs d{};
  d.src = a.d; d.src_b = (long)a.stride(); d.src_p = (long)l * N; d.src_limbs = l;
  d.dst = out.d; d.dst_b = (long)out.stride(); d.dst_p = (long)(l - 1) * N;
  d.pd = l - 1; d.nl = l - 1;
  d.add = nullptr; d.add_mask = 0; d.shifts = nullptr;
  drop_last_limb(c, B, d, tmpP);
  c.free(tmpP);
}

void eval_rotate(Context& c, const u64d* a, long a_stride, int B, int l, const KeyRowMap& km, u64d* out,
                 long out_stride) {
  const int N = c.N();
  u64d* tmp = c.alloc((size_t)B * l * N);
  u64d* D = c.alloc((size_t)B * l * (l + 1) * N);
  u64d* acc = c.alloc((size_t)B * 2 * (l + 1) * N);
  u64d* tmpP = c.alloc((size_t)B * 2 * N);
  ks_modup(c, a + (size_t)l * N, a_stride, B, l, &km, tmp, D);
  ks_inner(c, D, B, l, km, acc);
  DropArgs d{};
  d.src = acc; d.src_b = 2L * (l + 1) * N; d.src_p = (long)(l + 1) * N; d.src_limbs = l + 1;
  d.dst = out; d.dst_b = out_stride; d.dst_p = (long)l * N;
  d.pd = c.L(); d.nl = l;
  d.add = a; d.add_b = a_stride; d.add_p = 0; d.add_mask = 1; d.shifts = &km;
  drop_last_limb(c, B, d, tmpP);
  c.free(tmp); c.free(D); c.free(acc); c.free(tmpP);
}

// acc[b] = sum_g <ModUp digits D[b][g], key_g> over G rotated inputs per image
static void ks_inner_sum(Context& c, const u64d* D, int B, int G, int l, const KeyRowMap& km, u64d* acc) {
  const int N = c.N();
  c.ks[KS_INNER] += (int64_t)B * G;
  dim3 gi((N + kTpb - 1) / kTpb, l + 1, (B + kKsKT - 1) / kKsKT);
  const double sbytes = 8.0 * N * ((double)B * G * l * (l + 1) + 2.0 * G * l * (l + 1) + 2.0 * B * (l + 1));
  const double sops = 2.0 * N * B * G * l * (l + 1);
  if (kKsKT == 1 && l <= 8) {
    dim3 gt((N + kTpb - 1) / kTpb, l + 1, B);
#define KSS_GO(LV) \
  case LV: \
    LAUNCH_BO(c, "k_ks_inner", sbytes, sops, \
              k_ks_inner_sum_t<LV><<<gt, kTpb, 0, c.stream>>>(c.primes, D, B, G, c.L(), N, km, acc)); \
    break;
    switch (l) { KSS_GO(1) KSS_GO(2) KSS_GO(3) KSS_GO(4) KSS_GO(5) KSS_GO(6) KSS_GO(7) KSS_GO(8) }
#undef KSS_GO
  } else {
    LAUNCH_BO(c, "k_ks_inner", sbytes, sops,
              k_ks_inner_sum<<<gi, kTpb, 0, c.stream>>>(c.primes, D, B, G, l, c.L(), N, km, acc));
  }
}

// one rank's share of merge_maps (config 3 across GPUs): maps
// [B][M] are global maps lo .. lo+M-1 of each image; map j is rotated right
// by j*w.  acc = the extended-basis key inner products of the share's
// rotations, C = its Q-basis part (k_merge_c_part).  The element-wise sum of
// every share's (acc, C), reduced mod q, ModDown(acc) + C is the merged
// ciphertext -- bit-identical to eval_merge (the sums precede the rounding).
void eval_merge_partial(Context& c, const CtBatch& maps, int M, int lo, int64_t w, u64d* acc, u64d* C) {
  const int B = maps.count / M, l = maps.level, N = c.N(), S = c.S();
  const size_t st = maps.stride();
  const int first = lo == 0 ? 1 : 0, G = M - first;
  if (M > HEGPU_MAX_BATCH_PERIOD) fail(HEGPU_ERR_CAPACITY, "merge_maps: too many maps in one share");
  KeyRowMap kc{};
  kc.period = M;
  for (int j = 0; j < M; ++j) kc.shift[j] = (int)((S - ((int64_t)(lo + j) * w) % S) % S);
  if (G > 0) {
    KeyRowMap kg{};
    kg.period = G;
    for (int g = 0; g < G; ++g) {
      kg.shift[g] = kc.shift[first + g];
      kg.key[g] = c.rot_key(kg.shift[g]).data;
    }
    kg.grp = G;
    kg.grp_stride = (long)(M * st);
    u64d* tmp = c.alloc((size_t)B * G * l * N);
    u64d* D = c.alloc((size_t)B * G * l * (l + 1) * N);
    ks_modup(c, maps.d + first * st + (size_t)l * N, (long)st, B * G, l, &kg, tmp, D);
    ks_inner_sum(c, D, B, G, l, kg, acc);
    c.free(tmp);
    c.free(D);
  } else {
    CK(cudaMemsetAsync(acc, 0, (size_t)B * 2 * (l + 1) * N * 8, c.stream));
  }
  dim3 gc((N + kTpb - 1) / kTpb, 2 * l, B);
  LAUNCH_B(c, "k_merge_c", 8.0 * N * ((double)B * (M + 1) * l + 2.0 * B * l),
           k_merge_c_part<<<gc, kTpb, 0, c.stream>>>(c.primes, maps.d, B, M, first, l, N, kc, C));
}

// merge_maps with one lazy ModDown per image; km carries
// the nmaps-1 shifts / keys (period nmaps-1)
void eval_merge(Context& c, const CtBatch& maps, int nmaps, const KeyRowMap& km, CtBatch& out) {
  const int B = out.count, l = maps.level, N = c.N(), G = nmaps - 1;
  const size_t st = maps.stride();
  u64d* tmp = c.alloc((size_t)B * G * l * N);
  u64d* D = c.alloc((size_t)B * G * l * (l + 1) * N);
  u64d* acc = c.alloc((size_t)B * 2 * (l + 1) * N);
  u64d* C = c.alloc((size_t)B * 2 * l * N);
  u64d* tmpP = c.alloc((size_t)B * 2 * N);
  KeyRowMap kg = km;
  kg.grp = G;
  kg.grp_stride = (long)(nmaps * st);
  ks_modup(c, maps.d + st + (size_t)l * N, (long)st, B * G, l, &kg, tmp, D);
  ks_inner_sum(c, D, B, G, l, km, acc);
  dim3 gc((N + kTpb - 1) / kTpb, 2 * l, B);
  LAUNCH_B(c, "k_merge_c", 8.0 * N * ((double)B * (nmaps + 1) * l + 2.0 * B * l),
           k_merge_c<<<gc, kTpb, 0, c.stream>>>(c.primes, maps.d, B, nmaps, l, N, km, C));
  DropArgs d{};
  d.src = acc; d.src_b = 2L * (l + 1) * N; d.src_p = (long)(l + 1) * N; d.src_limbs = l + 1;
  d.dst = out.d; d.dst_b = (long)out.stride(); d.dst_p = (long)l * N;
  d.pd = c.L(); d.nl = l;
  d.add = C; d.add_b = 2L * l * N; d.add_p = (long)l * N; d.add_mask = 3; d.shifts = nullptr;
  drop_last_limb(c, B, d, tmpP);
  c.free(tmp); c.free(D); c.free(acc); c.free(C); c.free(tmpP);
}

void eval_square_impl(Context& c, const CtBatch& a, CtBatch& out, bool rescale);

void eval_square(Context& c, const CtBatch& a, CtBatch& out) { eval_square_impl(c, a, out, false); }

// square + relinearise + rescale with the ModDown and the rescale fused
// (drop_last_limb fuse_rescale, ntt.cu §4.8): out at level l - 1
void eval_square_rescale(Context& c, const CtBatch& a, CtBatch& out) { eval_square_impl(c, a, out, true); }

void eval_square_impl(Context& c, const CtBatch& a, CtBatch& out, bool rescale) {
  if (!c.has_relin) fail(HEGPU_ERR_KEY, "square: no relinearisation key");
  const int l = a.level, N = c.N(), B = a.count;
  if (rescale && l < 2) fail(HEGPU_ERR_CAPACITY, "square: no prime left to drop");
  u64d* d01 = c.alloc((size_t)B * 2 * l * N);
  u64d* d2 = c.alloc((size_t)B * l * N);
  u64d* tmp = c.alloc((size_t)B * l * N);
  u64d* D = c.alloc((size_t)B * l * (l + 1) * N);
  u64d* acc = c.alloc((size_t)B * 2 * (l + 1) * N);
  u64d* tmpP = c.alloc((size_t)B * 2 * N);
  launch_tensor_square(c, a.d, d01, d2, B, l);
  ks_modup(c, d2, (long)l * N, B, l, nullptr, tmp, D);
  KeyRowMap km{};
  km.period = 1;
  km.key[0] = c.relin.data;
  ks_inner(c, D, B, l, km, acc);
  DropArgs d{};
  d.src = acc; d.src_b = 2L * (l + 1) * N; d.src_p = (long)(l + 1) * N; d.src_limbs = l + 1;
  d.dst = out.d; d.dst_b = (long)out.stride(); d.dst_p = (long)(rescale ? l - 1 : l) * N;
  d.pd = c.L(); d.nl = rescale ? l - 1 : l;
  d.add = d01; d.add_b = 2L * l * N; d.add_p = (long)l * N; d.add_mask = 3; d.shifts = nullptr;
  d.fuse_rescale = rescale ? 1 : 0;
  drop_last_limb(c, B, d, tmpP);
  c.free(d01); c.free(d2); c.free(tmp); c.free(D); c.free(acc); c.free(tmpP);
}

}  // namespace hegpu
