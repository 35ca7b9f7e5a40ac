// core.hpp -- host-side parameter set, modular arithmetic and randomness of
// the hegpu engine (product code; independent of oracle/).
//
// The CKKS conventions are fixed by DESIGN.md §3 (primes, psi, NTT order,
// PRNG streams, encoding); the CPU oracle restates the same specification
// separately so the two can be compared limb for limb.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hegpu.h"

namespace hegpu {

using u64 = uint64_t;
using u128 = unsigned __int128;

// ---- errors (proj/include/hesim/errors.hpp:9-26) -------------------------
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// ---- scalar modular arithmetic (host) ------------------------------------
inline u64 mul_mod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
inline u64 add_mod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
inline u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
inline u64 neg_mod(u64 a, u64 q) { return a ? q - a : 0; }
u64 pow_mod(u64 a, u64 e, u64 q);
inline u64 inv_mod(u64 a, u64 q) { return pow_mod(a % q, q - 2, q); }
inline u64 shoup_pre(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
inline u64 shoup_mul(u64 a, u64 w, u64 wp, u64 q) {
  u64 h = (u64)(((u128)a * wp) >> 64);
  u64 r = a * w - h * q;
  return r >= q ? r - q : r;
}
bool is_prime_u64(u64 n);
unsigned bit_reverse(unsigned x, int bits);
// exact residue of an integer-valued double (any magnitude)
u64 residue_of_double(double x, u64 q);

// ---- parameter set -------------------------------------------------------
struct Prime {
  u64 q;
  u64 psi;          // primitive 2N-th root (DESIGN.md §3.2 rule)
  u64 ninv;         // N^{-1} mod q
  u64 qneg_inv;     // -q^{-1} mod 2^64 (Montgomery)
  u64 r_mod;        // 2^64 mod q
  u64 r2_mod;       // 2^128 mod q
  std::vector<u64> w, wp;    // psi^{brv(k)} and Shoup companions
  std::vector<u64> iw, iwp;  // psi^{-brv(k)} and Shoup companions
};

struct Params {
  int log_n = 0, n = 0, slots = 0, m2n = 0;  // N, S = N/2, 2N
  int L = 0;                                  // Q primes; P is index L
  std::vector<Prime> primes;                  // L + 1
  std::vector<uint32_t> slot_src;  // slot-order position p -> bit-reversed index
  std::vector<double> ksi_re, ksi_im;  // exp(2 pi i k / 2N), k in [0, 2N]
  std::vector<u64> rot_group;          // 5^j mod 2N, j < S
  u64 seed = 0;

  explicit Params(const hegpu_params& p);
  int np() const { return L + 1; }
  u64 q(int i) const { return primes[i].q; }
  // Galois element for a left rotation by r slots (5^r mod 2N)
  u64 galois_left(int64_t r) const;
  u64 galois_right(int64_t r) const { return galois_left((int64_t)slots - (r % slots)); }
};

// host NTT (bit-reversed output)
void host_ntt(const Params& P, int pi, u64* a);
void host_intt(const Params& P, int pi, u64* a);

// ---- counter-based randomness ----------------------------
inline u64 sm_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
struct Stream {
  u64 key;
  Stream(u64 seed, u64 tag)
      : key(sm_mix(sm_mix(seed) ^ (tag * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL))) {}
  u64 word(u64 k) const { return sm_mix(key + (k + 1) * 0x9E3779B97F4A7C15ULL); }
  int ternary(u64 k) const { return (int)(word(k) % 3) - 1; }
  int cbd21(u64 k) const {
    u64 w = word(k);
    return __builtin_popcountll(w & 0x1FFFFFULL) - __builtin_popcountll((w >> 32) & 0x1FFFFFULL);
  }
  u64 uniform(u64 k, u64 q) const { return (u64)(((u128)word(k) * q) >> 64); }
};
constexpr u64 kTagSecret = 1ULL << 56;
inline u64 tag_ksk(u64 kind, u64 g, u64 j, u64 comp, u64 t) {
  return (kind << 56) | (g << 24) | (j << 16) | (comp << 8) | t;
}
inline u64 tag_enc(u64 nonce, u64 comp, u64 t) {
  return (4ULL << 56) | ((nonce & 0xFFFFFFFFFFULL) << 12) | (comp << 8) | t;
}
constexpr u64 kKindGalois = 2, kKindRelin = 3;

// ---- client (host) -------------------------------------------------------
class Client {
 public:
  explicit Client(const Params& p);
  const Params& params() const { return P_; }
  // FP64 part of the encoding: slot values -> rounded coefficients
  void encode_coeffs(const double* z, int len, double scale, double* coeffs) const;
  // coefficients -> wire limbs (level [+P])
  void coeffs_to_limbs(const double* coeffs, int level, bool with_p, u64* out) const;
  void encode(const double* z, int len, double scale, int level, bool with_p, u64* out) const;
  void decode(const u64* pt, int level, double scale, double* slots) const;
  void encrypt(const u64* pt, int level, u64 nonce, u64* ct) const;
  // compact fresh ciphertext: the level a-stream keys, then
  // c0 limb i packed in ceil(bits(q_i) / 8) bytes per coefficient; c1 = a is
  // regenerated from the stream keys on the device.  Expands to exactly the
  // ciphertext encrypt() produces.
  size_t compact_bytes(int level) const;
  void encrypt_compact(const u64* pt, int level, u64 nonce, uint8_t* out) const;
  int limb_bytes(int i) const { return (64 - __builtin_clzll(P_.q(i)) + 7) / 8; }
  void decrypt(const u64* ct, int level, u64* pt) const;
  // key-switching key s' -> s, wire layout [L][2][L+1][N]
  void gen_ksk(u64 kind, u64 g, const u64* sprime, u64* key) const;
  void gen_galois_key(u64 g, u64* key) const;
  void gen_relin_key(u64* key) const;
  size_t key_words() const { return (size_t)P_.L * 2 * P_.np() * P_.n; }
  // automorphism X -> X^g on wire-format NTT limbs
  void automorph_wire(u64 g, const u64* in, u64* out, int nlimbs) const;

 private:
  void small_to_ntt(int pi, const int* v, u64* out) const;
  double crt_centered(const u64* r, int l) const;
  void fft_inv(std::vector<double>& re, std::vector<double>& im) const;
  void fft_fwd(std::vector<double>& re, std::vector<double>& im) const;
  const Params& P_;
  std::vector<u64> s_;  // secret, (L+1) limbs, wire NTT form
  std::vector<std::vector<u64>> qinv_;  // qinv_[i][j] = q_j^{-1} mod q_i
};

}  // namespace hegpu
