// eval.cu -- pointwise RNS kernels, the key-switch inner product, and the
// evaluator compositions (rescale, Galois rotation, square + relinearise).
//
// Reference semantics: add / mul (proj/src/slotvec.cpp:97-109), rotate_right
// / rotate_left (:42-66), square_layer (proj/src/convlower.cpp:141-143).
// The CKKS math (hybrid key switch, alpha = 1, one special prime) is fixed
// in DESIGN.md §3.6 and restated by oracle/ckks_oracle.c.
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
  for (int j = 0; j < l; ++j) {
    const u64d d = D[(((size_t)b * l + j) * (l + 1) + t) * N + k];
    const u64d* kj = key + (size_t)j * 2 * kp + (size_t)pi * N + k;
    mac128(lo0, hi0, d, __ldg(kj));
    mac128(lo1, hi1, d, __ldg(kj + kp));
  }
  u64d* o = acc + ((size_t)b * 2 * (l + 1) + t) * N + k;
  o[0] = mont_reduce128(lo0, hi0, pr.q, pr.qneg_inv);
  o[(size_t)(l + 1) * N] = mont_reduce128(lo1, hi1, pr.q, pr.qneg_inv);
}

// conv-pack MAC (convlower.cpp:39-74): up to 8 output maps per thread
template <int CO>
__global__ void k_conv_mac(PrimeTable pt, const u64d* __restrict__ taps, int ntaps, int l, int N,
                           const u64d* __restrict__ w, int c_out, const u64d* __restrict__ bias,
                           u64d* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y % l, poly = blockIdx.y / l;
  const int b = blockIdx.z / ((c_out + CO - 1) / CO), cg = blockIdx.z % ((c_out + CO - 1) / CO);
  if (k >= N) return;
  const DevPrime pr = pt.p[t];
  const size_t ct_words = (size_t)2 * l * N;
  const u64d* tp = taps + (size_t)b * ntaps * ct_words + (size_t)poly * l * N + (size_t)t * N + k;
  u64d acc[CO], lo[CO], hi[CO];
#pragma unroll
  for (int c = 0; c < CO; ++c) acc[c] = lo[c] = hi[c] = 0;
  for (int s0 = 0; s0 < ntaps; s0 += 7) {
    const int s1 = s0 + 7 < ntaps ? s0 + 7 : ntaps;
    for (int s = s0; s < s1; ++s) {
      const u64d x = tp[(size_t)s * ct_words];
#pragma unroll
      for (int c = 0; c < CO; ++c) {
        const int co = cg * CO + c;
        if (co < c_out) mac128(lo[c], hi[c], x, __ldg(w + ((size_t)co * ntaps + s) * l + t));
      }
    }
#pragma unroll
    for (int c = 0; c < CO; ++c) {
      acc[c] = add_mod_d(acc[c], mont_reduce128(lo[c], hi[c], pr.q, pr.qneg_inv), pr.q);
      lo[c] = hi[c] = 0;
    }
  }
#pragma unroll
  for (int c = 0; c < CO; ++c) {
    const int co = cg * CO + c;
    if (co >= c_out) break;
    u64d v = acc[c];
    if (poly == 0 && bias)
      v = add_mod_d(v, mont_mul(bias[((size_t)co * l + t) * N + k], 1ull, pr.q, pr.qneg_inv), pr.q);
    out[((size_t)b * c_out + co) * ct_words + (size_t)poly * l * N + (size_t)t * N + k] = v;
  }
}

// Halevi-Shoup diagonal accumulation over the hoisted ModUp digits D of v.c1
// (DESIGN.md §4.3): for each diagonal i with left shift s_i and mask m_i
//   acc (ext basis) += m_i * sum_j sigma_i(D_j) * key_i[j]
//   cacc            += m_i * sigma_i(v.c0)         (s_i == 0: m_i * v)
__global__ void k_hs_diag(PrimeTable pt, const u64d* __restrict__ v, const u64d* __restrict__ D, int l, int L,
                          int N, int ndiag, const u64d* __restrict__ masks, const int* __restrict__ shifts,
                          const u64d* const* __restrict__ keys, u64d* __restrict__ acc, u64d* __restrict__ cacc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  const int t = blockIdx.y, b = blockIdx.z;
  if (k >= N) return;
  const int S = N >> 1;
  const int pi = t == l ? L : t;
  const DevPrime pr = pt.p[pi];
  const u64d q = pr.q, qn = pr.qneg_inv;
  const size_t kp = (size_t)(L + 1) * N;
  const size_t ln = (size_t)l * N;
  const u64d* Db = D + (size_t)b * l * (l + 1) * N + (size_t)t * N;
  const u64d* c0 = v + (size_t)b * 2 * ln + (size_t)t * N;
  const u64d* c1 = c0 + ln;
  u64d a0 = 0, a1 = 0, x0 = 0, x1 = 0;
  for (int i = 0; i < ndiag; ++i) {
    const int s = __ldg(shifts + i);
    const u64d m = __ldg(masks + ((size_t)i * (l + 1) + t) * N + k);
    if (s == 0) {
      if (t < l) {
        x0 = add_mod_d(x0, mont_mul(c0[k], m, q, qn), q);
        x1 = add_mod_d(x1, mont_mul(c1[k], m, q, qn), q);
      }
      continue;
    }
    const int ps = shifted_pos(k, s, S);
    const u64d* key = keys[i] + (size_t)pi * N + k;
    u64d lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
    for (int j = 0; j < l; ++j) {
      const u64d d = Db[(size_t)j * (l + 1) * N + ps];
      const u64d* kj = key + (size_t)j * 2 * kp;
      mac128(lo0, hi0, d, __ldg(kj));
      mac128(lo1, hi1, d, __ldg(kj + kp));
    }
    const u64d ip0 = mont_reduce128(lo0, hi0, q, qn), ip1 = mont_reduce128(lo1, hi1, q, qn);
    a0 = add_mod_d(a0, mont_mul(ip0, m, q, qn), q);
    a1 = add_mod_d(a1, mont_mul(ip1, m, q, qn), q);
    if (t < l) x0 = add_mod_d(x0, mont_mul(c0[ps], m, q, qn), q);
  }
  u64d* ab = acc + (size_t)b * 2 * (l + 1) * N + (size_t)t * N + k;
  ab[0] = a0;
  ab[(size_t)(l + 1) * N] = a1;
  if (t < l) {
    u64d* cb = cacc + (size_t)b * 2 * ln + (size_t)t * N + k;
    cb[0] = x0;
    cb[ln] = x1;
  }
}

unsigned grid_for(size_t total) {
  size_t g = (total + kTpb - 1) / kTpb;
  return (unsigned)(g < 148 * 16 ? (g ? g : 1) : 148 * 16);
}

}  // namespace

void launch_add(Context& c, const u64d* a, const u64d* b, u64d* out, int count, int l) {
  const size_t total = (size_t)count * 2 * l * c.N();
  k_add<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, b, out, total, l, c.N());
  c.launches++;
  CK(cudaGetLastError());
}

void launch_add_plain(Context& c, const u64d* a, const u64d* p, long p_stride, u64d* out, int count, int l) {
  const size_t total = (size_t)count * 2 * l * c.N();
  k_add_plain<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, p, p_stride, out, total, l, c.N());
  c.launches++;
  CK(cudaGetLastError());
}

void launch_mul_plain(Context& c, const u64d* a, const u64d* p, long p_stride, u64d* out, int count, int l) {
  const size_t total = (size_t)count * 2 * l * c.N();
  k_mul_plain<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, p, p_stride, out, total, l, c.N());
  c.launches++;
  CK(cudaGetLastError());
}

void launch_tensor_square(Context& c, const u64d* a, u64d* d01, u64d* d2, int count, int l) {
  const size_t total = (size_t)count * l * c.N();
  k_tensor_square<<<grid_for(total), kTpb, 0, c.stream>>>(c.primes, a, d01, d2, total, l, c.N());
  c.launches++;
  CK(cudaGetLastError());
}

void ks_inner(Context& c, const u64d* D, int B, int l, const KeyRowMap& keys, u64d* acc) {
  dim3 grid((c.N() + kTpb - 1) / kTpb, l + 1, B);
  k_ks_inner<<<grid, kTpb, 0, c.stream>>>(c.primes, D, l, c.L(), c.N(), keys, acc);
  c.launches++;
  CK(cudaGetLastError());
}

void launch_conv_mac(Context& c, const u64d* taps, int B, int ntaps, int l, const u64d* w, int c_out,
                     const u64d* bias, u64d* out) {
  const int groups = (c_out + 7) / 8;
  dim3 grid((c.N() + kTpb - 1) / kTpb, 2 * l, B * groups);
  k_conv_mac<8><<<grid, kTpb, 0, c.stream>>>(c.primes, taps, ntaps, l, c.N(), w, c_out, bias, out);
  c.launches++;
  CK(cudaGetLastError());
}

void launch_hs_diag(Context& c, const u64d* v, int B, int l, const u64d* D, const HsDiagTable& t, u64d* acc,
                    u64d* cacc) {
  dim3 grid((c.N() + kTpb - 1) / kTpb, l + 1, B);
  k_hs_diag<<<grid, kTpb, 0, c.stream>>>(c.primes, v, D, l, c.L(), c.N(), t.ndiag, t.masks, t.shifts, t.keys,
                                         acc, cacc);
  c.launches++;
  CK(cudaGetLastError());
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
