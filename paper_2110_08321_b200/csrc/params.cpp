// params.cpp -- prime chain, roots of unity and NTT tables (host).
// DESIGN.md §3.1-3.3 fixes the rules; slot_src is the device-layout map.
#include <cmath>

#include "core.hpp"

namespace hegpu {

u64 pow_mod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  for (; e; e >>= 1) {
    if (e & 1) r = mul_mod(r, a, q);
    a = mul_mod(a, a, q);
  }
  return r;
}

bool is_prime_u64(u64 n) {
  static const u64 kBases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 b : kBases) {
    if (n == b) return true;
    if (n % b == 0) return false;
  }
  u64 d = n - 1;
  int s = 0;
  while (!(d & 1)) d >>= 1, ++s;
  for (u64 b : kBases) {
    u64 x = pow_mod(b, d, n);
    if (x == 1 || x == n - 1) continue;
    bool witness = true;
    for (int i = 1; i < s && witness; ++i) {
      x = mul_mod(x, x, n);
      if (x == n - 1) witness = false;
    }
    if (witness) return false;
  }
  return true;
}

unsigned bit_reverse(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1u);
  return r;
}

u64 residue_of_double(double x, u64 q) {
  const bool neg = x < 0;
  const double ax = std::fabs(x);
  u64 r;
  if (ax < 18446744073709551616.0) {
    r = static_cast<u64>(ax) % q;
  } else {
    int e = 0;
    const double m = std::frexp(ax, &e);
    const u64 mant = static_cast<u64>(std::ldexp(m, 53));
    r = mul_mod(mant % q, pow_mod(2, static_cast<u64>(e - 53), q), q);
  }
  return neg ? neg_mod(r, q) : r;
}

Params::Params(const hegpu_params& p) {
  if (p.log_n < 3 || p.log_n > 16) fail(HEGPU_ERR_ARG, "log_n must be in [3, 16]");
  if (p.n_q < 1 || p.n_q > HEGPU_MAX_Q) fail(HEGPU_ERR_ARG, "n_q out of range");
  log_n = p.log_n;
  n = 1 << log_n;
  slots = n / 2;
  m2n = 2 * n;
  L = p.n_q;
  seed = p.seed;
  primes.resize(L + 1);
  // largest unused primes below 2^bits with q == 1 (mod 2N), in request order
  for (int i = 0; i <= L; ++i) {
    const int bits = i < L ? p.q_bits[i] : p.p_bits;
    // <= 60 bits: the lazy NTT keeps values below 8q < 2^63
    if (bits <= log_n + 1 || bits > 60) fail(HEGPU_ERR_ARG, "prime bit size out of range (<= 60)");
    u64 c = (1ULL << bits) - (u64)m2n + 1;
    for (;; c -= (u64)m2n) {
      bool used = false;
      for (int j = 0; j < i; ++j) used = used || primes[j].q == c;
      if (!used && is_prime_u64(c)) break;
    }
    primes[i].q = c;
  }
  for (Prime& pr : primes) {
    const u64 q = pr.q;
    for (u64 x = 2;; ++x) {
      const u64 g = pow_mod(x, (q - 1) / (u64)m2n, q);
      if (pow_mod(g, (u64)n, q) == q - 1) { pr.psi = g; break; }
    }
    pr.ninv = inv_mod((u64)n, q);
    u64 inv = 1;  // -q^{-1} mod 2^64 by Newton iteration
    for (int it = 0; it < 6; ++it) inv *= 2 - q * inv;
    pr.qneg_inv = (u64)0 - inv;
    pr.r_mod = (u64)(((u128)1 << 64) % q);
    pr.r2_mod = mul_mod(pr.r_mod, pr.r_mod, q);
    pr.w.resize(n); pr.wp.resize(n); pr.iw.resize(n); pr.iwp.resize(n);
    const u64 ipsi = inv_mod(pr.psi, q);
    u64 pw = 1, ipw = 1;
    std::vector<u64> pows(n), ipows(n);
    for (int k = 0; k < n; ++k) { pows[k] = pw; ipows[k] = ipw; pw = mul_mod(pw, pr.psi, q); ipw = mul_mod(ipw, ipsi, q); }
    for (int k = 0; k < n; ++k) {
      const unsigned e = bit_reverse((unsigned)k, log_n);
      pr.w[k] = pows[e];   pr.wp[k] = shoup_pre(pr.w[k], q);
      pr.iw[k] = ipows[e]; pr.iwp[k] = shoup_pre(pr.iw[k], q);
    }
  }
  ksi_re.resize(m2n + 1);
  ksi_im.resize(m2n + 1);
  for (int k = 0; k < m2n; ++k) {
    const double ang = 2.0 * M_PI * (double)k / (double)m2n;
    ksi_re[k] = std::cos(ang);
    ksi_im[k] = std::sin(ang);
  }
  ksi_re[m2n] = ksi_re[0];
  ksi_im[m2n] = ksi_im[0];
  rot_group.resize(slots);
  for (u64 j = 0, g = 1; j < (u64)slots; ++j, g = g * 5 % (u64)m2n) rot_group[j] = g;
  // device layout: position p < S holds the evaluation at psi^(5^p), p >= S
  // at psi^(-5^(p-S)); in the wire (bit-reversed) order that is index
  // brv((e - 1) / 2).
  slot_src.resize(n);
  for (int p2 = 0; p2 < n; ++p2) {
    u64 e = rot_group[p2 % slots];
    if (p2 >= slots) e = (u64)m2n - e;
    slot_src[p2] = bit_reverse((unsigned)((e - 1) / 2), log_n);
  }
}

u64 Params::galois_left(int64_t r) const {
  int64_t s = slots;
  r %= s;
  if (r < 0) r += s;
  return pow_mod(5, (u64)r, (u64)m2n);
}

void host_ntt(const Params& P, int pi, u64* a) {
  const Prime& pr = P.primes[pi];
  const u64 q = pr.q;
  for (int m = 1, t = P.n >> 1; m < P.n; m <<= 1, t >>= 1) {
    for (int i = 0; i < m; ++i) {
      const u64 w = pr.w[m + i], wp = pr.wp[m + i];
      u64* x = a + 2 * i * t;
      for (int j = 0; j < t; ++j) {
        const u64 u = x[j], v = shoup_mul(x[j + t], w, wp, q);
        x[j] = add_mod(u, v, q);
        x[j + t] = sub_mod(u, v, q);
      }
    }
  }
}

void host_intt(const Params& P, int pi, u64* a) {
  const Prime& pr = P.primes[pi];
  const u64 q = pr.q;
  for (int t = 1, h = P.n >> 1; h >= 1; t <<= 1, h >>= 1) {
    for (int i = 0; i < h; ++i) {
      const u64 w = pr.iw[h + i], wp = pr.iwp[h + i];
      u64* x = a + 2 * i * t;
      for (int j = 0; j < t; ++j) {
        const u64 u = x[j], v = x[j + t];
        x[j] = add_mod(u, v, q);
        x[j + t] = shoup_mul(sub_mod(u, v, q), w, wp, q);
      }
    }
  }
  const u64 nw = pr.ninv, nwp = shoup_pre(pr.ninv, q);
  for (int k = 0; k < P.n; ++k) a[k] = shoup_mul(a[k], nw, nwp, q);
}

}  // namespace hegpu
