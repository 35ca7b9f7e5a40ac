// eval.cu -- pointwise RNS kernels, the key-switch inner product, the
// conv-pack MAC, the Halevi-Shoup diagonal accumulation, and the evaluator
// compositions (rescale, Galois rotation, square + relinearise).
//
// Reference semantics: add / mul (proj/src/slotvec.cpp:97-109), rotate_right
// / rotate_left (:42-66), square_layer (proj/src/convlower.cpp:141-143),
// conv_packed_forward (:39-74), hs_matvec (proj/src/matvec.cpp:82-105).  The
// CKKS math (hybrid key switch, alpha = 1, one special prime) is fixed in
// DESIGN.md §3 and restated by oracle/ckks_oracle.c.
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

// key-switch inner product: acc[b][p][t] = sum_j D[b][j][t] * key_b[j][p][pi(t)]
__global__ void k_ks_inner(PrimeTable pt, const u64d* __restrict__ D, int l, int L, int N, KeyRowMap km,
                           u64d* __restrict__ acc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y, b = blockIdx.z;
  if (k >= N) return;
  const int pi = t == l ? L : t;
  const DevPrime pr = pt.p[pi];
  const u64d* key = km.key[b % km.period];
  const size_t kp = (size_t)(L + 1) * N;  // one key poly over all primes
  u64d lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
  uint32_t t0 = 0, t1 = 0;
  for (int j = 0; j < l; ++j) {
    const u64d d = D[(((size_t)b * l + j) * (l + 1) + t) * N + k];
    const u64d* kj = key + (size_t)j * 2 * kp + (size_t)pi * N + k;
    mad192(lo0, hi0, t0, d, __ldg(kj));
    mad192(lo1, hi1, t1, d, __ldg(kj + kp));
  }
  u64d* o = acc + ((size_t)b * 2 * (l + 1) + t) * N + k;
  o[0] = red192(lo0, hi0, t0, pr);
  o[(size_t)(l + 1) * N] = red192(lo1, hi1, t1, pr);
}

// conv-pack MAC (convlower.cpp:39-74): CO output maps per thread, taps
// streamed 8 at a time so each thread keeps 8 independent loads in flight.
template <int CO>
__global__ void __launch_bounds__(kTpb) k_conv_mac(PrimeTable pt, const u64d* __restrict__ taps, int ntaps, int l,
                                                   int N, const u64d* __restrict__ w, int c_out,
                                                   const u64d* __restrict__ bias, u64d* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % l, poly = blockIdx.y / l;
  const int groups = (c_out + CO - 1) / CO;
  const int b = blockIdx.z / groups, cg = blockIdx.z % groups;
  if (k >= N) return;
  const DevPrime pr = pt.p[t];
  const size_t ct_words = (size_t)2 * l * N;
  const u64d* tp = taps + (size_t)b * ntaps * ct_words + (size_t)poly * l * N + (size_t)t * N + k;
  u64d lo[CO], hi[CO];
  uint32_t top[CO];
#pragma unroll
  for (int c = 0; c < CO; ++c) lo[c] = hi[c] = 0, top[c] = 0;
  const int nco = c_out - cg * CO < CO ? c_out - cg * CO : CO;
  int s = 0;
  for (; s + 8 <= ntaps; s += 8) {
    u64d x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(tp + (size_t)(s + u) * ct_words);
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < CO; ++c)
        if (c < nco) mad192(lo[c], hi[c], top[c], x[u], __ldg(w + ((size_t)(cg * CO + c) * ntaps + s + u) * l + t));
  }
  for (; s < ntaps; ++s) {
    const u64d x = __ldg(tp + (size_t)s * ct_words);
#pragma unroll
    for (int c = 0; c < CO; ++c)
      if (c < nco) mad192(lo[c], hi[c], top[c], x, __ldg(w + ((size_t)(cg * CO + c) * ntaps + s) * l + t));
  }
#pragma unroll
  for (int c = 0; c < CO; ++c) {
    if (c >= nco) break;
    const int co = cg * CO + c;
    u64d v = red192(lo[c], hi[c], top[c], pr);
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
constexpr int kHsBT = 4;    // images per thread

template <int LV>
__global__ void __launch_bounds__(kHsKB) k_hs_diag(PrimeTable pt, const u64d* __restrict__ v,
                                                   const u64d* __restrict__ D, int B, int L, int N,
                                                   HsDiagTable tab, u64d* __restrict__ acc,
                                                   u64d* __restrict__ cacc) {
  extern __shared__ u64d win[];  // [BT][LV + 1][W]
  const int S = N >> 1;
  const int KB = kHsKB < S ? kHsKB : S;
  const int kb = blockIdx.y, t = blockIdx.z, b0 = blockIdx.x * kHsBT;
  const int k0 = kb * KB, k = k0 + threadIdx.x;
  const bool active = threadIdx.x < KB;
  const int half = k0 >= S ? S : 0;
  const int pi = t == LV ? L : t;
  const DevPrime pr = pt.p[pi];
  const bool has_c = t < LV;
  const int Wmax = KB + kHsCW;
  const int nrow = has_c ? LV + 1 : LV;  // D digits (+ c0)
  const size_t ln = (size_t)LV * N;

  u64d a_lo[kHsBT][2], a_hi[kHsBT][2], c_lo[kHsBT][2], c_hi[kHsBT][2];
  uint32_t a_tp[kHsBT][2], c_tp[kHsBT][2];
#pragma unroll
  for (int bb = 0; bb < kHsBT; ++bb)
#pragma unroll
    for (int p = 0; p < 2; ++p) a_lo[bb][p] = a_hi[bb][p] = c_lo[bb][p] = c_hi[bb][p] = 0, a_tp[bb][p] = c_tp[bb][p] = 0;

  for (int ch = 0; ch < tab.nchunk; ++ch) {
    const int i0 = __ldg(tab.chunk + ch), i1 = __ldg(tab.chunk + ch + 1);
    const int r_lo = __ldg(tab.r + i0), r_hi = __ldg(tab.r + i1 - 1);
    const int W = KB + r_hi - r_lo;
    // stage window positions k0 - r_hi + w (mod S, inside this half)
    __syncthreads();
    for (int e = threadIdx.x; e < kHsBT * nrow * W; e += blockDim.x) {
      const int w = e % W, rb = e / W, row = rb % nrow, bb = rb / nrow;
      const int b = b0 + bb;
      int pos = k0 - half - r_hi + w;
      pos %= S;
      if (pos < 0) pos += S;
      pos += half;
      u64d val = 0;
      if (b < B)
        val = row < LV ? D[(((size_t)b * LV + row) * (LV + 1) + t) * N + pos]
                       : v[(size_t)b * 2 * ln + (size_t)t * N + pos];
      win[(size_t)(bb * (LV + 1) + row) * Wmax + w] = val;
    }
    __syncthreads();
    if (!active) continue;
    for (int i = i0; i < i1; ++i) {
      const int r = __ldg(tab.r + i);
      const int wo = threadIdx.x + (r_hi - r);
      const u64d m = has_c ? __ldg(tab.masks + ((size_t)i * (LV + 1) + t) * N + k) : 0ull;
      if (r == 0) {
        if (has_c) {
#pragma unroll
          for (int bb = 0; bb < kHsBT; ++bb) {
            const int b = b0 + bb;
            if (b >= B) break;
            mad192(c_lo[bb][0], c_hi[bb][0], c_tp[bb][0], win[(size_t)(bb * (LV + 1) + LV) * Wmax + wo], m);
            mad192(c_lo[bb][1], c_hi[bb][1], c_tp[bb][1], v[(size_t)b * 2 * ln + ln + (size_t)t * N + k], m);
          }
        }
        continue;
      }
      const u64d* fk = tab.fkeys[i] + (size_t)t * N + k;
      const size_t kp = (size_t)(LV + 1) * N;
      u64d kv[LV][2];
#pragma unroll
      for (int j = 0; j < LV; ++j) {
        kv[j][0] = __ldg(fk + (size_t)j * 2 * kp);
        kv[j][1] = __ldg(fk + (size_t)j * 2 * kp + kp);
      }
#pragma unroll
      for (int bb = 0; bb < kHsBT; ++bb) {
#pragma unroll
        for (int j = 0; j < LV; ++j) {
          const u64d d = win[(size_t)(bb * (LV + 1) + j) * Wmax + wo];
          mad192(a_lo[bb][0], a_hi[bb][0], a_tp[bb][0], d, kv[j][0]);
          mad192(a_lo[bb][1], a_hi[bb][1], a_tp[bb][1], d, kv[j][1]);
        }
        if (has_c) mad192(c_lo[bb][0], c_hi[bb][0], c_tp[bb][0], win[(size_t)(bb * (LV + 1) + LV) * Wmax + wo], m);
      }
    }
  }
  if (!active) return;
#pragma unroll
  for (int bb = 0; bb < kHsBT; ++bb) {
    const int b = b0 + bb;
    if (b >= B) break;
    u64d* ab = acc + (size_t)b * 2 * (LV + 1) * N + (size_t)t * N + k;
    ab[0] = red192(a_lo[bb][0], a_hi[bb][0], a_tp[bb][0], pr);
    ab[(size_t)(LV + 1) * N] = red192(a_lo[bb][1], a_hi[bb][1], a_tp[bb][1], pr);
    if (has_c) {
      u64d* cb = cacc + (size_t)b * 2 * ln + (size_t)t * N + k;
      cb[0] = red192(c_lo[bb][0], c_hi[bb][0], c_tp[bb][0], pr);
      cb[ln] = red192(c_lo[bb][1], c_hi[bb][1], c_tp[bb][1], pr);
    }
  }
}

// fused key: fk[j][p][t] = key[j][p][pi(t)] * m[t]   (t over the ext basis)
__global__ void k_fuse_key(PrimeTable pt, const u64d* __restrict__ key, const u64d* __restrict__ m, int l, int L,
                           int N, u64d* __restrict__ fk) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % (l + 1), jp = blockIdx.y / (l + 1);  // jp = j * 2 + p
  if (k >= N) return;
  const int pi = t == l ? L : t;
  const DevPrime pr = pt.p[pi];
  const u64d kv = key[((size_t)jp * (L + 1) + pi) * N + k];
  fk[((size_t)jp * (l + 1) + t) * N + k] = mont_mul(kv, m[(size_t)t * N + k], pr.q, pr.qneg_inv);
}

unsigned grid_for(size_t total) {
  size_t g = (total + kTpb - 1) / kTpb;
  return (unsigned)(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

template <int LV>
void launch_hs_lv(Context& c, const u64d* v, int B, const u64d* D, const HsDiagTable& t, u64d* acc, u64d* cacc) {
  const int N = c.N(), S = N / 2;
  const int KB = kHsKB < S ? kHsKB : S;
  dim3 grid((B + kHsBT - 1) / kHsBT, N / KB, LV + 1);
  const size_t sm = (size_t)kHsBT * (LV + 1) * (KB + kHsCW) * 8;
  static size_t done = 0;
  if (sm > 48 * 1024 && sm > done) {
    CK(cudaFuncSetAttribute(k_hs_diag<LV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    done = sm;
  }
  // fused keys + masks (c-part limbs) once; v, D read once; acc, cacc written once
  const double NB = 8.0 * N;
  const double bytes = NB * (t.keyed * LV * 2.0 * (LV + 1) + t.ndiag * LV + B * (LV * (LV + 1.0) + 2.0 * LV) +
                             B * (2.0 * (LV + 1) + 2.0 * LV));
  LAUNCH_B(c, "k_hs_diag", bytes, k_hs_diag<LV><<<grid, kHsKB, sm, c.stream>>>(c.primes, v, D, B, c.L(), N, t, acc, cacc));
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
  dim3 grid((c.N() + kTpb - 1) / kTpb, l + 1, B);
  double kb = 0;  // distinct keys read once each
  for (int i = 0; i < keys.period && i < B; ++i) kb += 8.0 * l * 2 * (l + 1) * c.N();
  LAUNCH_B(c, "k_ks_inner", 8.0 * B * (l + 2) * (l + 1) * c.N() + kb, k_ks_inner<<<grid, kTpb, 0, c.stream>>>(c.primes, D, l, c.L(), c.N(), keys, acc));
}

void launch_conv_mac(Context& c, const u64d* taps, int B, int ntaps, int l, const u64d* w, int c_out,
                     const u64d* bias, u64d* out) {
  // taps read once, maps written once, bias plaintexts read once
  const double bytes = 8.0 * c.N() * l * (2.0 * B * ntaps + 2.0 * B * c_out + c_out);
  if (c_out <= 4) {
    dim3 grid((c.N() + kTpb - 1) / kTpb, 2 * l, B * ((c_out + 3) / 4));
    LAUNCH_B(c, "k_conv_mac", bytes,
           k_conv_mac<4><<<grid, kTpb, 0, c.stream>>>(c.primes, taps, ntaps, l, c.N(), w, c_out, bias, out));
  } else {
    dim3 grid((c.N() + kTpb - 1) / kTpb, 2 * l, B * ((c_out + 7) / 8));
    LAUNCH_B(c, "k_conv_mac", bytes,
           k_conv_mac<8><<<grid, kTpb, 0, c.stream>>>(c.primes, taps, ntaps, l, c.N(), w, c_out, bias, out));
  }
}

void launch_fuse_key(Context& c, const u64d* key, const u64d* mask, int l, u64d* fk) {
  dim3 grid((c.N() + kTpb - 1) / kTpb, 2 * l * (l + 1));
  LAUNCH(c, "k_fuse_key", k_fuse_key<<<grid, kTpb, 0, c.stream>>>(c.primes, key, mask, l, c.L(), c.N(), fk));
}

void launch_hs_diag(Context& c, const u64d* v, int B, int l, const u64d* D, const HsDiagTable& t, u64d* acc,
                    u64d* cacc) {
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

void eval_square(Context& c, const CtBatch& a, CtBatch& out) {
  if (!c.has_relin) fail(HEGPU_ERR_KEY, "square: no relinearisation key");
  const int l = a.level, N = c.N(), B = a.count;
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
  d.dst = out.d; d.dst_b = (long)out.stride(); d.dst_p = (long)l * N;
  d.pd = c.L(); d.nl = l;
  d.add = d01; d.add_b = 2L * l * N; d.add_p = (long)l * N; d.add_mask = 3; d.shifts = nullptr;
  drop_last_limb(c, B, d, tmpP);
  c.free(d01); c.free(d2); c.free(tmp); c.free(D); c.free(acc); c.free(tmpP);
}

}  // namespace hegpu
