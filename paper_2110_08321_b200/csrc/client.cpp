// client.cpp -- host-side client of the engine: CKKS encoding (canonical
// embedding over the 5^j slot order), symmetric encryption, decryption and
// key generation.  In the reference these are the free `pack` / `conv_pack`
// client steps (proj/src/slotvec.cpp:26-40, proj/src/convlower.cpp:9-37);
// here they produce RNS limbs in the wire format of include/hegpu.h.
#include <cmath>
#include <cstring>

#include "core.hpp"

namespace hegpu {

Client::Client(const Params& p) : P_(p) {
  const int N = P_.n, np = P_.np();
  s_.resize((size_t)np * N);
  std::vector<int> sv(N);
  const Stream st(P_.seed, kTagSecret);
  for (int k = 0; k < N; ++k) sv[k] = st.ternary((u64)k);
  for (int pi = 0; pi < np; ++pi) small_to_ntt(pi, sv.data(), s_.data() + (size_t)pi * N);
  qinv_.assign(np, std::vector<u64>(np, 0));
  for (int i = 0; i < np; ++i)
    for (int j = 0; j < np; ++j)
      if (i != j) qinv_[i][j] = inv_mod(P_.q(j) % P_.q(i), P_.q(i));
}

void Client::small_to_ntt(int pi, const int* v, u64* out) const {
  const u64 q = P_.q(pi);
  for (int k = 0; k < P_.n; ++k) out[k] = v[k] >= 0 ? (u64)v[k] : q - (u64)(-v[k]);
  host_ntt(P_, pi, out);
}

// ---- encoding ------------------------------------------------------------
static void swap_bitrev(std::vector<double>& re, std::vector<double>& im, int size) {
  int bits = 0;
  while ((1 << bits) < size) ++bits;
  for (int i = 0; i < size; ++i) {
    const int j = (int)bit_reverse((unsigned)i, bits);
    if (i < j) { std::swap(re[i], re[j]); std::swap(im[i], im[j]); }
  }
}

// Inverse of the slot evaluation map z_j = m(zeta^(5^j)) on S complex slots
// (the published special-FFT recursion of CKKS).  The FP
// operation sequence is part of the spec: built with -ffp-contract=off.
void Client::fft_inv(std::vector<double>& re, std::vector<double>& im) const {
  const int size = P_.slots, M = P_.m2n;
  for (int len = size; len >= 2; len >>= 1) {
    const int half = len >> 1, quad = len << 2, gap = M / quad;
    for (int base = 0; base < size; base += len) {
      for (int j = 0; j < half; ++j) {
        const long idx = (long)(quad - (int)(P_.rot_group[j] % (u64)quad)) * gap;
        const double ar = re[base + j], ai = im[base + j];
        const double br = re[base + j + half], bi = im[base + j + half];
        const double sr = ar + br, si = ai + bi;
        const double dr = ar - br, di = ai - bi;
        const double kr = P_.ksi_re[idx], ki = P_.ksi_im[idx];
        re[base + j] = sr;
        im[base + j] = si;
        re[base + j + half] = dr * kr - di * ki;
        im[base + j + half] = dr * ki + di * kr;
      }
    }
  }
  swap_bitrev(re, im, size);
  for (int i = 0; i < size; ++i) { re[i] /= size; im[i] /= size; }
}

void Client::fft_fwd(std::vector<double>& re, std::vector<double>& im) const {
  const int size = P_.slots, M = P_.m2n;
  swap_bitrev(re, im, size);
  for (int len = 2; len <= size; len <<= 1) {
    const int half = len >> 1, quad = len << 2, gap = M / quad;
    for (int base = 0; base < size; base += len) {
      for (int j = 0; j < half; ++j) {
        const long idx = (long)(P_.rot_group[j] % (u64)quad) * gap;
        const double ur = re[base + j], ui = im[base + j];
        const double br = re[base + j + half], bi = im[base + j + half];
        const double kr = P_.ksi_re[idx], ki = P_.ksi_im[idx];
        const double vr = br * kr - bi * ki, vi = br * ki + bi * kr;
        re[base + j] = ur + vr;
        im[base + j] = ui + vi;
        re[base + j + half] = ur - vr;
        im[base + j + half] = ui - vi;
      }
    }
  }
}

void Client::encode_coeffs(const double* z, int len, double scale, double* coeffs) const {
  const int S = P_.slots;
  if (len > S) fail(HEGPU_ERR_CAPACITY, "encode: " + std::to_string(len) + " values exceed " +
                                            std::to_string(S) + " slots");
  std::vector<double> re(S, 0.0), im(S, 0.0);
  for (int j = 0; j < len; ++j) re[j] = z[j];
  fft_inv(re, im);
  for (int k = 0; k < S; ++k) {
    coeffs[k] = std::rint(re[k] * scale);
    coeffs[k + S] = std::rint(im[k] * scale);
  }
}

void Client::coeffs_to_limbs(const double* coeffs, int level, bool with_p, u64* out) const {
  const int N = P_.n;
  const int nl = level + (with_p ? 1 : 0);
  for (int l = 0; l < nl; ++l) {
    const int pi = l < level ? l : P_.L;
    u64* o = out + (size_t)l * N;
    for (int k = 0; k < N; ++k) o[k] = residue_of_double(coeffs[k], P_.q(pi));
    host_ntt(P_, pi, o);
  }
}

void Client::encode(const double* z, int len, double scale, int level, bool with_p, u64* out) const {
  std::vector<double> co(P_.n);
  encode_coeffs(z, len, scale, co.data());
  coeffs_to_limbs(co.data(), level, with_p, out);
}

double Client::crt_centered(const u64* r, int l) const {
  u64 a[HEGPU_MAX_Q + 1];
  for (int i = 0; i < l; ++i) {
    const u64 q = P_.q(i);
    u64 t = r[i];
    for (int j = 0; j < i; ++j) t = mul_mod(sub_mod(t, a[j] % q, q), qinv_[i][j], q);
    a[i] = t;
  }
  // x > (Q-1)/2 iff its mixed-radix digits exceed ((q_i-1)/2)_i lexicographically
  bool neg = false;
  for (int i = l - 1; i >= 0; --i) {
    const u64 h = (P_.q(i) - 1) / 2;
    if (a[i] != h) { neg = a[i] > h; break; }
  }
  if (neg) {  // Q - x, digit-wise on (Q-1) - x, plus one
    u64 carry = 1;
    for (int i = 0; i < l; ++i) {
      u64 d = P_.q(i) - 1 - a[i] + carry;
      carry = d == P_.q(i);
      a[i] = carry ? 0 : d;
    }
  }
  double v = (double)a[l - 1];
  for (int i = l - 2; i >= 0; --i) v = v * (double)P_.q(i) + (double)a[i];
  return neg ? -v : v;
}

void Client::decode(const u64* pt, int level, double scale, double* slots) const {
  const int N = P_.n, S = P_.slots;
  std::vector<u64> tmp(pt, pt + (size_t)level * N);
  for (int l = 0; l < level; ++l) host_intt(P_, l, tmp.data() + (size_t)l * N);
  std::vector<double> re(S), im(S);
  u64 r[HEGPU_MAX_Q + 1];
  for (int k = 0; k < N; ++k) {
    for (int l = 0; l < level; ++l) r[l] = tmp[(size_t)l * N + k];
    const double v = crt_centered(r, level) / scale;
    if (k < S) re[k] = v; else im[k - S] = v;
  }
  fft_fwd(re, im);
  for (int j = 0; j < S; ++j) slots[j] = re[j];
}

// ---- encryption ------------------------------------------------------------
void Client::encrypt(const u64* pt, int level, u64 nonce, u64* ct) const {
  const int N = P_.n;
  std::vector<int> ev(N);
  std::vector<u64> e(N);
  const Stream es(P_.seed, tag_enc(nonce, 1, 0));
  for (int k = 0; k < N; ++k) ev[k] = es.cbd21((u64)k);
  for (int t = 0; t < level; ++t) {
    const u64 q = P_.q(t);
    small_to_ntt(t, ev.data(), e.data());
    const Stream as(P_.seed, tag_enc(nonce, 0, t));
    const u64* st = s_.data() + (size_t)t * N;
    const u64* m = pt + (size_t)t * N;
    u64* c0 = ct + (size_t)t * N;
    u64* c1 = ct + ((size_t)level + t) * N;
    for (int k = 0; k < N; ++k) {
      const u64 a = as.uniform((u64)k, q);
      c1[k] = a;
      c0[k] = add_mod(sub_mod(e[k], mul_mod(a, st[k], q), q), m[k], q);
    }
  }
}

size_t Client::compact_bytes(int level) const {
  size_t n = (size_t)level * 8;
  for (int i = 0; i < level; ++i) n += (size_t)P_.n * limb_bytes(i);
  return n;
}

void Client::encrypt_compact(const u64* pt, int level, u64 nonce, uint8_t* out) const {
  const int N = P_.n;
  std::vector<u64> ct((size_t)2 * level * N);
  encrypt(pt, level, nonce, ct.data());
  u64* keys = reinterpret_cast<u64*>(out);
  for (int t = 0; t < level; ++t) keys[t] = Stream(P_.seed, tag_enc(nonce, 0, (u64)t)).key;
  // c0 in the DEVICE SLOT ORDER (position p = wire index slot_src[p]), so the
  // device expansion is a linear unpack
  uint8_t* o = out + (size_t)level * 8;
  for (int t = 0; t < level; ++t) {
    const int nb = limb_bytes(t);
    const u64* c0 = ct.data() + (size_t)t * N;
    for (int p = 0; p < N; ++p) {
      const u64 v = c0[P_.slot_src[p]];
      for (int b = 0; b < nb; ++b) *o++ = (uint8_t)(v >> (8 * b));
    }
  }
}

void Client::decrypt(const u64* ct, int level, u64* pt) const {
  const int N = P_.n;
  for (int t = 0; t < level; ++t) {
    const u64 q = P_.q(t);
    for (int k = 0; k < N; ++k) {
      const size_t i = (size_t)t * N + k;
      pt[i] = add_mod(ct[i], mul_mod(ct[(size_t)level * N + i], s_[i], q), q);
    }
  }
}

// ---- key generation ----------------------------------------------------------
// Hybrid key switching with one special prime P and one-limb digits: digit j
// of key s' -> s encrypts P * s' in limb j only (the CRT idempotent gadget),
// so the same key serves every level.
void Client::gen_ksk(u64 kind, u64 g, const u64* sp, u64* key) const {
  const int N = P_.n, L = P_.L, np = P_.np();
  const u64 P = P_.q(L);
  std::vector<int> ev(N);
  std::vector<u64> e(N);
  for (int j = 0; j < L; ++j) {
    const Stream es(P_.seed, tag_ksk(kind, g, (u64)j, 1, 0));
    for (int k = 0; k < N; ++k) ev[k] = es.cbd21((u64)k);
    for (int t = 0; t < np; ++t) {
      const u64 q = P_.q(t);
      small_to_ntt(t, ev.data(), e.data());
      const Stream as(P_.seed, tag_ksk(kind, g, (u64)j, 0, (u64)t));
      u64* b = key + (((size_t)j * 2 + 0) * np + t) * N;
      u64* a = key + (((size_t)j * 2 + 1) * np + t) * N;
      const u64* st = s_.data() + (size_t)t * N;
      const u64* spt = sp + (size_t)t * N;
      const u64 pm = P % q;
      for (int k = 0; k < N; ++k) {
        a[k] = as.uniform((u64)k, q);
        u64 v = sub_mod(e[k], mul_mod(a[k], st[k], q), q);
        if (t == j) v = add_mod(v, mul_mod(pm, spt[k], q), q);
        b[k] = v;
      }
    }
  }
}

void Client::automorph_wire(u64 g, const u64* in, u64* out, int nlimbs) const {
  const int N = P_.n;
  for (int k = 0; k < N; ++k) {
    const u64 e = (2 * (u64)bit_reverse((unsigned)k, P_.log_n) + 1) * g % (u64)P_.m2n;
    const unsigned src = bit_reverse((unsigned)((e - 1) / 2), P_.log_n);
    for (int l = 0; l < nlimbs; ++l) out[(size_t)l * N + k] = in[(size_t)l * N + src];
  }
}

void Client::gen_galois_key(u64 g, u64* key) const {
  std::vector<u64> sp(s_.size());
  automorph_wire(g, s_.data(), sp.data(), P_.np());
  gen_ksk(kKindGalois, g, sp.data(), key);
}

void Client::gen_relin_key(u64* key) const {
  std::vector<u64> sp(s_.size());
  const int N = P_.n;
  for (int t = 0; t < P_.np(); ++t)
    for (int k = 0; k < N; ++k) {
      const size_t i = (size_t)t * N + k;
      sp[i] = mul_mod(s_[i], s_[i], P_.q(t));
    }
  gen_ksk(kKindRelin, 0, sp.data(), key);
}

}  // namespace hegpu
