/*
 * oracle/ckks_oracle.c -- TEST INFRASTRUCTURE ONLY.  See ckks_oracle.h for
 * the parity status ("parity unpinned" at the CKKS limb level) and the
 * shared conventions.  Deliberately simple: straight loops, __int128 modular
 * products, one limb at a time.  Compiled with -ffp-contract=off so the FP64
 * encoder performs exactly the operations written.
 *
 * Reference anchors (slot semantics these limbs must decrypt to):
 *   rotate_right/left  proj/src/slotvec.cpp:42-66   -> ock_rotate + ock_galois_*
 *   add / mul          proj/src/slotvec.cpp:97-109  -> ock_add / ock_add_pc / ock_mul_pc
 *   square_layer       proj/src/convlower.cpp:141-143 -> ock_square (+ rescale)
 *   conv_packed_forward proj/src/convlower.cpp:39-74 -> ock_conv_mac (+ rescale)
 *   merge_maps         proj/src/convlower.cpp:145-160 -> ock_merge
 *   hs_matvec          proj/src/matvec.cpp:82-105   -> ock_hs_hoisted + rescale + folds
 */
#include "ckks_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

#define MAXP 40


struct ock_ctx {
  int logN, N, S, M, L, np;
  u64 q[MAXP];
  u64 psi[MAXP];
  u64 ninv[MAXP];
  u64 *psi_rev[MAXP], *ipsi_rev[MAXP];
  u64 *psi_sh[MAXP], *ipsi_sh[MAXP];   /* Shoup companions of the twiddles */
  u64 qinv_mod[MAXP][MAXP]; /* q_j^{-1} mod q_i */
  double *ksi_re, *ksi_im;  /* M+1 */
  u64* rot_group;           /* S entries 5^j mod M */
};

/* ---------------------------------------------------------------- arith */
/* general a * b mod q: x86-64 compiles the 128 / 64 remainder to one DIV,
 * measured faster here than a Barrett reduction with runtime shift counts;
 * products by a constant (NTT twiddles, N^-1, q^-1, conv weights) use Shoup
 * (mulmod_sh) */
static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
/* Shoup product with a precomputed companion w' = floor(w 2^64 / q) */
static inline u64 mulmod_sh(u64 a, u64 w, u64 wp, u64 q) {
  const u64 h = (u64)(((u128)a * wp) >> 64);
  u64 r = a * w - h * q;
  return r >= q ? r - q : r;
}
static inline u64 addmod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static inline u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static inline u64 negmod(u64 a, u64 q) { return a ? q - a : 0; }
static u64 powmod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }

static int is_prime(u64 n) {
  static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; i++) {
    if (n == bases[i]) return 1;
    if (n % bases[i] == 0) return 0;
  }
  u64 d = n - 1;
  int r = 0;
  while ((d & 1) == 0) { d >>= 1; r++; }
  for (int i = 0; i < 12; i++) {
    u64 x = powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int comp = 1;
    for (int k = 1; k < r; k++) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = 0; break; }
    }
    if (comp) return 0;
  }
  return 1;
}

static unsigned brv(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
  return r;
}

/* exact residue of an integer-valued double */
static u64 dmod(double x, u64 q) {
  int neg = x < 0;
  double ax = fabs(x);
  u64 r;
  if (ax < 18446744073709551616.0) {
    r = ((u64)ax) % q;
  } else {
    int e;
    double m = frexp(ax, &e);
    u64 mant = (u64)ldexp(m, 53);
    r = mulmod(mant % q, powmod(2, (u64)(e - 53), q), q);
  }
  return neg ? negmod(r, q) : r;
}

/* --------------------------------------------------------------- context */
ock_ctx* ock_create(int logN, int L, const int* qbits, int pbits) {
  if (L + 1 > MAXP || logN < 2 || logN > 17) return NULL;
  ock_ctx* c = (ock_ctx*)calloc(1, sizeof(ock_ctx));
  c->logN = logN;
  c->N = 1 << logN;
  c->S = c->N / 2;
  c->M = 2 * c->N;
  c->L = L;
  c->np = L + 1;
  for (int i = 0; i < c->np; i++) {
    int b = i < L ? qbits[i] : pbits;
    u64 cand = (1ULL << b) - (u64)c->M + 1;
    for (;;) {
      int used = 0;
      for (int j = 0; j < i; j++) used |= (c->q[j] == cand);
      if (!used && is_prime(cand)) break;
      cand -= (u64)c->M;
    }
    c->q[i] = cand;
  }
  for (int i = 0; i < c->np; i++) {
    u64 q = c->q[i];
    for (u64 x = 2;; x++) {
      u64 g = powmod(x, (q - 1) / (u64)c->M, q);
      if (powmod(g, (u64)c->N, q) == q - 1) { c->psi[i] = g; break; }
    }
    c->ninv[i] = invmod((u64)c->N, q);
    c->psi_rev[i] = (u64*)malloc(sizeof(u64) * c->N);
    c->ipsi_rev[i] = (u64*)malloc(sizeof(u64) * c->N);
    u64 ipsi = invmod(c->psi[i], q);
    c->psi_sh[i] = (u64*)malloc(sizeof(u64) * c->N);
    c->ipsi_sh[i] = (u64*)malloc(sizeof(u64) * c->N);
    for (int k = 0; k < c->N; k++) {
      unsigned e = brv((unsigned)k, logN);
      c->psi_rev[i][k] = powmod(c->psi[i], e, q);
      c->ipsi_rev[i][k] = powmod(ipsi, e, q);
      c->psi_sh[i][k] = (u64)(((u128)c->psi_rev[i][k] << 64) / q);
      c->ipsi_sh[i][k] = (u64)(((u128)c->ipsi_rev[i][k] << 64) / q);
    }
    for (int j = 0; j < c->np; j++)
      c->qinv_mod[i][j] = (i == j) ? 0 : invmod(c->q[j] % q, q);
  }
  c->ksi_re = (double*)malloc(sizeof(double) * (c->M + 1));
  c->ksi_im = (double*)malloc(sizeof(double) * (c->M + 1));
  for (int k = 0; k < c->M; k++) {
    double ang = 2.0 * M_PI * (double)k / (double)c->M;
    c->ksi_re[k] = cos(ang);
    c->ksi_im[k] = sin(ang);
  }
  c->ksi_re[c->M] = c->ksi_re[0];
  c->ksi_im[c->M] = c->ksi_im[0];
  c->rot_group = (u64*)malloc(sizeof(u64) * c->S);
  u64 g = 1;
  for (int j = 0; j < c->S; j++) { c->rot_group[j] = g; g = (g * 5) % (u64)c->M; }
  return c;
}

void ock_destroy(ock_ctx* c) {
  if (!c) return;
  for (int i = 0; i < c->np; i++) {
    free(c->psi_rev[i]); free(c->ipsi_rev[i]); free(c->psi_sh[i]); free(c->ipsi_sh[i]);
  }
  free(c->ksi_re); free(c->ksi_im); free(c->rot_group);
  free(c);
}
uint64_t ock_prime(const ock_ctx* c, int i) { return c->q[i]; }
uint64_t ock_psi(const ock_ctx* c, int i) { return c->psi[i]; }
int ock_N(const ock_ctx* c) { return c->N; }

/* ------------------------------------------------------------------- NTT */
void ock_ntt(const ock_ctx* c, int pi, u64* a) {
  const u64 q = c->q[pi];
  const u64* w = c->psi_rev[pi];
  const u64* wsh = c->psi_sh[pi];
  int t = c->N;
  for (int m = 1; m < c->N; m <<= 1) {
    t >>= 1;
    for (int i = 0; i < m; i++) {
      int j1 = 2 * i * t;
      u64 s = w[m + i], sp = wsh[m + i];
      for (int j = j1; j < j1 + t; j++) {
        u64 U = a[j], V = mulmod_sh(a[j + t], s, sp, q);
        a[j] = addmod(U, V, q);
        a[j + t] = submod(U, V, q);
      }
    }
  }
}

void ock_intt(const ock_ctx* c, int pi, u64* a) {
  const u64 q = c->q[pi];
  const u64* w = c->ipsi_rev[pi];
  const u64* wsh = c->ipsi_sh[pi];
  int t = 1;
  for (int m = c->N; m > 1; m >>= 1) {
    int h = m >> 1, j1 = 0;
    for (int i = 0; i < h; i++) {
      u64 s = w[h + i], sp = wsh[h + i];
      for (int j = j1; j < j1 + t; j++) {
        u64 U = a[j], V = a[j + t];
        a[j] = addmod(U, V, q);
        a[j + t] = mulmod_sh(submod(U, V, q), s, sp, q);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  const u64 ni = c->ninv[pi], nip = (u64)(((u128)ni << 64) / q);
  for (int j = 0; j < c->N; j++) a[j] = mulmod_sh(a[j], ni, nip, q);
}

/* ---------------------------------------------------------- automorphism */
uint64_t ock_galois_left(const ock_ctx* c, int64_t r) {
  int64_t S = c->S;
  r %= S;
  if (r < 0) r += S;
  return powmod(5, (u64)r, (u64)c->M);
}
uint64_t ock_galois_right(const ock_ctx* c, int64_t r) {
  return ock_galois_left(c, (int64_t)c->S - (r % (int64_t)c->S));
}

void ock_automorph_ntt(const ock_ctx* c, u64 g, const u64* in, u64* out,
                       int nlimbs) {
  const int N = c->N;
  for (int k = 0; k < N; k++) {
    u64 e = (2 * (u64)brv((unsigned)k, c->logN) + 1) * g % (u64)c->M;
    unsigned src = brv((unsigned)((e - 1) / 2), c->logN);
    for (int l = 0; l < nlimbs; l++) out[(size_t)l * N + k] = in[(size_t)l * N + src];
  }
}

void ock_automorph_coeff(const ock_ctx* c, int pi, u64 g, const u64* in,
                         u64* out) {
  const u64 q = c->q[pi];
  for (int i = 0; i < c->N; i++) {
    u64 e = (u64)i * g % (u64)c->M;
    if (e < (u64)c->N) out[e] = in[i];
    else out[e - c->N] = negmod(in[i], q);
  }
}

/* -------------------------------------------------------------- encoding */
static void bit_reverse_c(double* re, double* im, int size) {
  int bits = 0;
  while ((1 << bits) < size) bits++;
  for (int i = 0; i < size; i++) {
    int j = (int)brv((unsigned)i, bits);
    if (i < j) {
      double t = re[i]; re[i] = re[j]; re[j] = t;
      t = im[i]; im[i] = im[j]; im[j] = t;
    }
  }
}

/* inverse "special" FFT over the 5^j slot ordering (published HEAAN/CKKS
 * algorithm, restated) */
static void fft_special_inv(const ock_ctx* c, double* re, double* im, int size) {
  for (int len = size; len >= 1; len >>= 1) {
    int lenh = len >> 1, lenq = len << 2, gap = c->M / lenq;
    for (int i = 0; i < size; i += len) {
      for (int j = 0; j < lenh; j++) {
        long idx = (long)(lenq - (int)(c->rot_group[j] % (u64)lenq)) * gap;
        double ar = re[i + j], ai = im[i + j];
        double br = re[i + j + lenh], bi = im[i + j + lenh];
        double ur = ar + br, ui = ai + bi;
        double vr = ar - br, vi = ai - bi;
        double kr = c->ksi_re[idx], ki = c->ksi_im[idx];
        re[i + j] = ur;
        im[i + j] = ui;
        re[i + j + lenh] = vr * kr - vi * ki;
        im[i + j + lenh] = vr * ki + vi * kr;
      }
    }
  }
  bit_reverse_c(re, im, size);
  for (int i = 0; i < size; i++) { re[i] /= size; im[i] /= size; }
}

static void fft_special(const ock_ctx* c, double* re, double* im, int size) {
  bit_reverse_c(re, im, size);
  for (int len = 2; len <= size; len <<= 1) {
    int lenh = len >> 1, lenq = len << 2, gap = c->M / lenq;
    for (int i = 0; i < size; i += len) {
      for (int j = 0; j < lenh; j++) {
        long idx = (long)(c->rot_group[j] % (u64)lenq) * gap;
        double ur = re[i + j], ui = im[i + j];
        double br = re[i + j + lenh], bi = im[i + j + lenh];
        double kr = c->ksi_re[idx], ki = c->ksi_im[idx];
        double vr = br * kr - bi * ki, vi = br * ki + bi * kr;
        re[i + j] = ur + vr;
        im[i + j] = ui + vi;
        re[i + j + lenh] = ur - vr;
        im[i + j + lenh] = ui - vi;
      }
    }
  }
}

void ock_encode_fp(const ock_ctx* c, const double* z, int len, double scale,
                   double* coeffs) {
  const int S = c->S;
  double* re = (double*)calloc(S, sizeof(double));
  double* im = (double*)calloc(S, sizeof(double));
  for (int j = 0; j < len && j < S; j++) re[j] = z[j];
  fft_special_inv(c, re, im, S);
  for (int k = 0; k < S; k++) {
    coeffs[k] = rint(re[k] * scale);
    coeffs[k + S] = rint(im[k] * scale);
  }
  free(re); free(im);
}

void ock_encode_coeffs(const ock_ctx* c, const double* coeffs, int level,
                       int with_p, u64* out) {
  const int N = c->N;
  int nl = level + (with_p ? 1 : 0);
  for (int l = 0; l < nl; l++) {
    int pi = l < level ? l : c->L;
    u64* o = out + (size_t)l * N;
    for (int k = 0; k < N; k++) o[k] = dmod(coeffs[k], c->q[pi]);
    ock_ntt(c, pi, o);
  }
}

void ock_encode(const ock_ctx* c, const double* z, int len, double scale,
                int level, int with_p, u64* out) {
  double* co = (double*)malloc(sizeof(double) * c->N);
  ock_encode_fp(c, z, len, scale, co);
  ock_encode_coeffs(c, co, level, with_p, out);
  free(co);
}

void ock_encode_direct(const ock_ctx* c, const double* z, int len, double scale,
                       double* coeffs) {
  /* m_k = (2/N) Re( sum_j scale*z_j * zeta^{-5^j k} ), zeta = exp(i pi / N) */
  const int N = c->N, S = c->S;
  for (int k = 0; k < N; k++) {
    double acc = 0.0;
    for (int j = 0; j < len && j < S; j++) {
      u64 e = (c->rot_group[j] * (u64)k) % (u64)c->M;
      double ang = -M_PI * (double)e / (double)N;
      acc += z[j] * cos(ang);
    }
    coeffs[k] = 2.0 * scale * acc / (double)N;
  }
}

/* centered CRT composition of residues r[0..l) to a double (Garner) */
static double crt_centered(const ock_ctx* c, const u64* r, int l) {
  u64 a[MAXP];
  for (int i = 0; i < l; i++) {
    u64 q = c->q[i], t = r[i];
    for (int j = 0; j < i; j++) {
      t = submod(t, a[j] % q, q);
      t = mulmod(t, c->qinv_mod[i][j], q);
    }
    a[i] = t;
  }
  /* compare with (Q-1)/2 whose mixed-radix digits are (q_i-1)/2 */
  int neg = 0;
  for (int i = l - 1; i >= 0; i--) {
    u64 h = (c->q[i] - 1) / 2;
    if (a[i] > h) { neg = 1; break; }
    if (a[i] < h) { neg = 0; break; }
  }
  if (neg) { /* Q - x = (Q-1) - x + 1 digit-wise */
    u64 carry = 1;
    for (int i = 0; i < l; i++) {
      u64 d = c->q[i] - 1 - a[i] + carry;
      if (d == c->q[i]) { d = 0; carry = 1; } else carry = 0;
      a[i] = d;
    }
  }
  double v = (double)a[l - 1];
  for (int i = l - 2; i >= 0; i--) v = v * (double)c->q[i] + (double)a[i];
  return neg ? -v : v;
}

void ock_decode(const ock_ctx* c, const u64* pt, int level, double scale,
                double* slots) {
  const int N = c->N, S = c->S;
  u64* tmp = (u64*)malloc(sizeof(u64) * (size_t)N * level);
  memcpy(tmp, pt, sizeof(u64) * (size_t)N * level);
  for (int l = 0; l < level; l++) ock_intt(c, l, tmp + (size_t)l * N);
  double* re = (double*)malloc(sizeof(double) * S);
  double* im = (double*)malloc(sizeof(double) * S);
  u64 r[MAXP];
  for (int k = 0; k < N; k++) {
    for (int l = 0; l < level; l++) r[l] = tmp[(size_t)l * N + k];
    double v = crt_centered(c, r, level) / scale;
    if (k < S) re[k] = v; else im[k - S] = v;
  }
  fft_special(c, re, im, S);
  for (int j = 0; j < S; j++) slots[j] = re[j];
  free(re); free(im); free(tmp);
}

/* ------------------------------------------------------------------ PRNG */
static inline u64 sm_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
static inline u64 stream_key(u64 seed, u64 tag) {
  return sm_mix(sm_mix(seed) ^ (tag * 0xD1B54A32D192ED03ULL + 0x632BE59BD9B4E019ULL));
}
static inline u64 stream_word(u64 key, u64 k) {
  return sm_mix(key + (k + 1) * 0x9E3779B97F4A7C15ULL);
}
static inline int sample_ternary(u64 key, u64 k) { return (int)(stream_word(key, k) % 3) - 1; }
static inline int sample_cbd(u64 key, u64 k) {
  u64 w = stream_word(key, k);
  return __builtin_popcountll(w & 0x1FFFFFULL) - __builtin_popcountll((w >> 32) & 0x1FFFFFULL);
}
static inline u64 sample_uniform(u64 key, u64 k, u64 q) {
  return (u64)(((u128)stream_word(key, k) * q) >> 64);
}

#define TAG_SECRET (1ULL << 56)
#define TAG_KSK(kind, g, j, comp, t) \
  (((u64)(kind) << 56) | ((u64)(g) << 24) | ((u64)(j) << 16) | ((u64)(comp) << 8) | (u64)(t))
#define TAG_ENC(nonce, comp, t) \
  ((4ULL << 56) | (((u64)(nonce) & 0xFFFFFFFFFFULL) << 12) | ((u64)(comp) << 8) | (u64)(t))

/* small signed coefficients -> NTT limb for prime pi */
static void small_to_ntt(const ock_ctx* c, int pi, const int* v, u64* out) {
  u64 q = c->q[pi];
  for (int k = 0; k < c->N; k++) out[k] = v[k] >= 0 ? (u64)v[k] : q - (u64)(-v[k]);
  ock_ntt(c, pi, out);
}

void ock_secret(const ock_ctx* c, u64 seed, u64* s) {
  int* v = (int*)malloc(sizeof(int) * c->N);
  u64 key = stream_key(seed, TAG_SECRET);
  for (int k = 0; k < c->N; k++) v[k] = sample_ternary(key, (u64)k);
  for (int pi = 0; pi < c->np; pi++) small_to_ntt(c, pi, v, s + (size_t)pi * c->N);
  free(v);
}

void ock_gen_ksk(const ock_ctx* c, u64 seed, u64 kind, u64 g, const u64* s,
                 const u64* sp, u64* key) {
  const int N = c->N, L = c->L, np = c->np;
  int* ev = (int*)malloc(sizeof(int) * N);
  u64* e = (u64*)malloc(sizeof(u64) * N);
  const u64 P = c->q[L];
  for (int j = 0; j < L; j++) {
    u64 ekey = stream_key(seed, TAG_KSK(kind, g, j, 1, 0));
    for (int k = 0; k < N; k++) ev[k] = sample_cbd(ekey, (u64)k);
    for (int t = 0; t < np; t++) {
      u64 q = c->q[t];
      small_to_ntt(c, t, ev, e);
      u64 akey = stream_key(seed, TAG_KSK(kind, g, j, 0, t));
      u64* b = key + (((size_t)j * 2 + 0) * np + t) * N;
      u64* a = key + (((size_t)j * 2 + 1) * np + t) * N;
      const u64* st = s + (size_t)t * N;
      const u64* spt = sp + (size_t)t * N;
      u64 pmod = P % q;
      for (int k = 0; k < N; k++) {
        a[k] = sample_uniform(akey, (u64)k, q);
        u64 v = submod(e[k], mulmod(a[k], st[k], q), q);
        if (t == j) v = addmod(v, mulmod(pmod, spt[k], q), q);
        b[k] = v;
      }
    }
  }
  free(ev); free(e);
}

void ock_gen_galois_key(const ock_ctx* c, u64 seed, const u64* s, u64 g, u64* key) {
  u64* sp = (u64*)malloc(sizeof(u64) * (size_t)c->N * c->np);
  ock_automorph_ntt(c, g, s, sp, c->np);
  ock_gen_ksk(c, seed, 2, g, s, sp, key);
  free(sp);
}

void ock_gen_relin_key(const ock_ctx* c, u64 seed, const u64* s, u64* key) {
  const size_t n = (size_t)c->N * c->np;
  u64* sp = (u64*)malloc(sizeof(u64) * n);
  for (int t = 0; t < c->np; t++)
    for (int k = 0; k < c->N; k++) {
      size_t i = (size_t)t * c->N + k;
      sp[i] = mulmod(s[i], s[i], c->q[t]);
    }
  ock_gen_ksk(c, seed, 3, 0, s, sp, key);
  free(sp);
}

void ock_encrypt(const ock_ctx* c, u64 seed, u64 nonce, const u64* s,
                 const u64* pt, int l, u64* ct) {
  const int N = c->N;
  int* ev = (int*)malloc(sizeof(int) * N);
  u64* e = (u64*)malloc(sizeof(u64) * N);
  u64 ekey = stream_key(seed, TAG_ENC(nonce, 1, 0));
  for (int k = 0; k < N; k++) ev[k] = sample_cbd(ekey, (u64)k);
  for (int t = 0; t < l; t++) {
    u64 q = c->q[t];
    small_to_ntt(c, t, ev, e);
    u64 akey = stream_key(seed, TAG_ENC(nonce, 0, t));
    u64* c0 = ct + (size_t)t * N;
    u64* c1 = ct + ((size_t)l + t) * N;
    const u64* st = s + (size_t)t * N;
    const u64* m = pt + (size_t)t * N;
    for (int k = 0; k < N; k++) {
      u64 a = sample_uniform(akey, (u64)k, q);
      c1[k] = a;
      c0[k] = addmod(submod(e[k], mulmod(a, st[k], q), q), m[k], q);
    }
  }
  free(ev); free(e);
}

void ock_decrypt(const ock_ctx* c, const u64* s, const u64* ct, int l, u64* pt) {
  const int N = c->N;
  for (int t = 0; t < l; t++) {
    u64 q = c->q[t];
    for (int k = 0; k < N; k++) {
      size_t i = (size_t)t * N + k;
      pt[i] = addmod(ct[i], mulmod(ct[(size_t)l * N + i], s[i], q), q);
    }
  }
}

/* -------------------------------------------------------------- evaluator */
void ock_add(const ock_ctx* c, const u64* a, const u64* b, int l, u64* out) {
  const int N = c->N;
  for (int p = 0; p < 2; p++)
    for (int t = 0; t < l; t++)
      for (int k = 0; k < N; k++) {
        size_t i = ((size_t)p * l + t) * N + k;
        out[i] = addmod(a[i], b[i], c->q[t]);
      }
}

void ock_add_pc(const ock_ctx* c, const u64* a, const u64* pt, int l, u64* out) {
  const size_t n = (size_t)c->N * l;
  for (size_t i = 0; i < n; i++) out[i] = addmod(a[i], pt[i], c->q[i / c->N]);
  if (out != a) memcpy(out + n, a + n, sizeof(u64) * n);
}

void ock_mul_pc(const ock_ctx* c, const u64* a, const u64* pt, int l, u64* out) {
  const int N = c->N;
  for (int p = 0; p < 2; p++)
    for (int t = 0; t < l; t++)
      for (int k = 0; k < N; k++) {
        size_t i = ((size_t)p * l + t) * N + k;
        out[i] = mulmod(a[i], pt[(size_t)t * N + k], c->q[t]);
      }
}

/* divide an (nl+1)-limb polynomial by its last prime `qd` (index pd) with a
 * centered lift of the dropped residue; `src` limbs 0..nl-1 use primes
 * prime_of[0..nl-1]. out gets nl limbs. */
static void drop_last(const ock_ctx* c, const u64* src, const int* prime_of,
                      int nl, int pd, u64* out) {
  const int N = c->N;
  const u64 qd = c->q[pd];
  u64* last = (u64*)malloc(sizeof(u64) * N);
  u64* x = (u64*)malloc(sizeof(u64) * N);
  memcpy(last, src + (size_t)nl * N, sizeof(u64) * N);
  ock_intt(c, pd, last);
  for (int t = 0; t < nl; t++) {
    int pi = prime_of[t];
    u64 q = c->q[pi];
    for (int k = 0; k < N; k++) {
      u64 r = last[k];
      x[k] = (r > qd / 2) ? negmod((qd - r) % q, q) : r % q;
    }
    ock_ntt(c, pi, x);
    u64 inv = invmod(qd % q, q);
    const u64* s = src + (size_t)t * N;
    u64* o = out + (size_t)t * N;
    const u64 invp = (u64)(((u128)inv << 64) / q);
    for (int k = 0; k < N; k++) o[k] = mulmod_sh(submod(s[k], x[k], q), inv, invp, q);
  }
  free(last); free(x);
}

void ock_rescale(const ock_ctx* c, const u64* a, int l, u64* out) {
  int prime_of[MAXP] = {0};
  for (int t = 0; t < l; t++) prime_of[t] = t;
  const size_t N = c->N;
  for (int p = 0; p < 2; p++)
    drop_last(c, a + (size_t)p * l * N, prime_of, l - 1, l - 1,
              out + (size_t)p * (l - 1) * N);
}

/* ModUp of d (l limbs, NTT) into D[j][t] (l digits x (l+1) ext limbs) */
static void modup(const ock_ctx* c, const u64* d, int l, u64* D) {
  const int N = c->N;
  u64* coef = (u64*)malloc(sizeof(u64) * N);
  for (int j = 0; j < l; j++) {
    memcpy(coef, d + (size_t)j * N, sizeof(u64) * N);
    ock_intt(c, j, coef);
    for (int t = 0; t <= l; t++) {
      int pi = t < l ? t : c->L;
      u64* o = D + ((size_t)j * (l + 1) + t) * N;
      if (pi == j) { memcpy(o, d + (size_t)j * N, sizeof(u64) * N); continue; }
      for (int k = 0; k < N; k++) o[k] = coef[k] % c->q[pi];
      ock_ntt(c, pi, o);
    }
  }
  free(coef);
}

/* inner product of D (optionally permuted by g) with key at level l,
 * ACC[2][l+1][N] (ext basis) */
static void key_inner(const ock_ctx* c, const u64* D, int l, const u64* key,
                      u64* ACC) {
  const int N = c->N, np = c->np;
  memset(ACC, 0, sizeof(u64) * 2 * (size_t)(l + 1) * N);
  for (int p = 0; p < 2; p++)
    for (int t = 0; t <= l; t++) {
      int pi = t < l ? t : c->L;
      u64 q = c->q[pi];
      u64* acc = ACC + ((size_t)p * (l + 1) + t) * N;
      /* lazy reduction: the l products (< 2^122 each, l < 64) are summed in
       * 128 bits and reduced once -- the same residue as reducing each term */
      for (int k = 0; k < N; k++) {
        u128 s = 0;
        for (int j = 0; j < l; j++)
          s += (u128)D[((size_t)j * (l + 1) + t) * N + k] * key[(((size_t)j * 2 + p) * np + pi) * N + k];
        acc[k] = (u64)(s % q);
      }
    }
}

/* ModDown of ACC[2][l+1][N] -> out[2][l][N] */
static void moddown(const ock_ctx* c, const u64* ACC, int l, u64* out) {
  int prime_of[MAXP] = {0};
  for (int t = 0; t < l; t++) prime_of[t] = t;
  const size_t N = c->N;
  for (int p = 0; p < 2; p++)
    drop_last(c, ACC + (size_t)p * (l + 1) * N, prime_of, l, c->L,
              out + (size_t)p * l * N);
}

static void keyswitch(const ock_ctx* c, const u64* d, int l, const u64* key,
                      u64* out) {
  const size_t N = c->N;
  u64* D = (u64*)malloc(sizeof(u64) * (size_t)l * (l + 1) * N);
  u64* ACC = (u64*)malloc(sizeof(u64) * 2 * (size_t)(l + 1) * N);
  modup(c, d, l, D);
  key_inner(c, D, l, key, ACC);
  moddown(c, ACC, l, out);
  free(D); free(ACC);
}

void ock_rotate(const ock_ctx* c, const u64* a, int l, u64 g, const u64* key,
                u64* out) {
  const size_t N = c->N, n = (size_t)l * N;
  u64* ra = (u64*)malloc(sizeof(u64) * 2 * n);
  u64* ks = (u64*)malloc(sizeof(u64) * 2 * n);
  ock_automorph_ntt(c, g, a, ra, 2 * l);
  keyswitch(c, ra + n, l, key, ks);
  for (int t = 0; t < l; t++)
    for (size_t k = 0; k < N; k++) {
      size_t i = (size_t)t * N + k;
      out[i] = addmod(ra[i], ks[i], c->q[t]);
      out[n + i] = ks[n + i];
    }
  free(ra); free(ks);
}

void ock_square(const ock_ctx* c, const u64* a, int l, const u64* rlk, u64* out) {
  const size_t N = c->N, n = (size_t)l * N;
  u64* d2 = (u64*)malloc(sizeof(u64) * n);
  u64* ks = (u64*)malloc(sizeof(u64) * 2 * n);
  u64* d0 = (u64*)malloc(sizeof(u64) * n);
  u64* d1 = (u64*)malloc(sizeof(u64) * n);
  for (size_t i = 0; i < n; i++) {
    u64 q = c->q[i / N];
    u64 c0 = a[i], c1 = a[n + i];
    d0[i] = mulmod(c0, c0, q);
    d1[i] = mulmod(addmod(c0, c0, q), c1, q);
    d2[i] = mulmod(c1, c1, q);
  }
  keyswitch(c, d2, l, rlk, ks);
  for (size_t i = 0; i < n; i++) {
    u64 q = c->q[i / N];
    out[i] = addmod(d0[i], ks[i], q);
    out[n + i] = addmod(d1[i], ks[n + i], q);
  }
  free(d2); free(ks); free(d0); free(d1);
}

void ock_conv_mac(const ock_ctx* c, const u64* taps, int ntaps, int l,
                  const double* weights, int c_out, double wscale,
                  const u64* bias_pts, u64* maps) {
  const size_t N = c->N, n = (size_t)l * N;
  for (int co = 0; co < c_out; co++) {
    u64* o = maps + (size_t)co * 2 * n;
    memset(o, 0, sizeof(u64) * 2 * n);
    for (int t = 0; t < ntaps; t++) {
      double wi = rint(weights[(size_t)co * ntaps + t] * wscale);
      const u64* tp = taps + (size_t)t * 2 * n;
      for (int p = 0; p < 2; p++)
        for (int li = 0; li < l; li++) {
          u64 q = c->q[li], W = dmod(wi, q), Wp = (u64)(((u128)W << 64) / q);
          for (size_t k = 0; k < N; k++) {
            size_t i = (size_t)p * n + (size_t)li * N + k;
            o[i] = addmod(o[i], mulmod_sh(tp[i], W, Wp, q), q);
          }
        }
    }
    if (bias_pts) ock_add_pc(c, o, bias_pts + (size_t)co * n, l, o);
  }
}

/* merge_maps with one lazy ModDown:
 *   out = map_0 + sum_j rot_right(map_j, j w)
 *       = (map_0.c0 + sum_j sigma_j(map_j.c0), map_0.c1) + ModDown(sum_j IP_j)
 * where IP_j is the extended-basis key-switch inner product of
 * sigma_j(map_j.c1). */
void ock_merge(const ock_ctx* c, const u64* maps, int nmaps, int l, int64_t w,
               const u64* keys, u64* out) {
  const size_t N = c->N, n = 2 * (size_t)l * N, ne = (size_t)(l + 1) * N;
  const size_t ksz = (size_t)c->L * 2 * c->np * N;
  u64* ra = (u64*)malloc(sizeof(u64) * n);
  u64* D = (u64*)malloc(sizeof(u64) * (size_t)l * ne);
  u64* IP = (u64*)malloc(sizeof(u64) * 2 * ne);
  u64* ACC = (u64*)calloc(2 * ne, sizeof(u64));
  u64* md = (u64*)malloc(sizeof(u64) * n);
  memcpy(out, maps, sizeof(u64) * n);
  for (int j = 1; j < nmaps; j++) {
    ock_automorph_ntt(c, ock_galois_right(c, (int64_t)j * w), maps + (size_t)j * n, ra, 2 * l);
    modup(c, ra + (size_t)l * N, l, D);
    key_inner(c, D, l, keys + (size_t)(j - 1) * ksz, IP);
    for (int p = 0; p < 2; p++)
      for (int t = 0; t <= l; t++) {
        u64 q = c->q[t < l ? t : c->L];
        for (size_t k = 0; k < N; k++) {
          size_t i = (size_t)p * ne + (size_t)t * N + k;
          ACC[i] = addmod(ACC[i], IP[i], q);
        }
      }
    for (int t = 0; t < l; t++)
      for (size_t k = 0; k < N; k++) {
        size_t i = (size_t)t * N + k;
        out[i] = addmod(out[i], ra[i], c->q[t]);
      }
  }
  if (nmaps > 1) {
    moddown(c, ACC, l, md);
    for (int p = 0; p < 2; p++)
      for (int t = 0; t < l; t++)
        for (size_t k = 0; k < N; k++) {
          size_t i = (size_t)p * l * N + (size_t)t * N + k;
          out[i] = addmod(out[i], md[i], c->q[t]);
        }
  }
  free(ra); free(D); free(IP); free(ACC); free(md);
}

/* Double-hoisted Halevi-Shoup diagonal sum:
 *   out = sum_i mask'_i (.) rot_right(v, r_i),   mask'_i = rot_right(mask_i, r_i)
 * One ModUp of v.c1, one ModDown of the summed extended-basis products. */
void ock_hs_hoisted(const ock_ctx* c, const u64* v, int l, int ndiag,
                    const int64_t* rots, const u64* masks_ext, const u64* keys,
                    u64* out) {
  const size_t N = c->N, n = (size_t)l * N, ne = (size_t)(l + 1) * N;
  const size_t ksz = (size_t)c->L * 2 * c->np * N;
  u64* D = (u64*)malloc(sizeof(u64) * l * ne);
  u64* Dg = (u64*)malloc(sizeof(u64) * l * ne);
  u64* IP = (u64*)malloc(sizeof(u64) * 2 * ne);
  u64* ACC = (u64*)calloc(2 * ne, sizeof(u64));
  u64* C = (u64*)calloc(2 * n, sizeof(u64));
  u64* c0g = (u64*)malloc(sizeof(u64) * n);
  u64* md = (u64*)malloc(sizeof(u64) * 2 * n);
  modup(c, v + n, l, D);
  int kidx = 0;
  for (int i = 0; i < ndiag; i++) {
    const u64* m = masks_ext + (size_t)i * ne;
    if (rots[i] == 0) {
      for (int p = 0; p < 2; p++)
        for (int t = 0; t < l; t++)
          for (size_t k = 0; k < N; k++) {
            size_t idx = (size_t)t * N + k; u64 q = c->q[t];
            C[p * n + idx] = addmod(C[p * n + idx], mulmod(v[p * n + idx], m[idx], q), q);
          }
      continue;
    }
    u64 g = ock_galois_right(c, rots[i]);
    const u64* key = keys + (size_t)(kidx++) * ksz;
    ock_automorph_ntt(c, g, D, Dg, l * (l + 1));
    key_inner(c, Dg, l, key, IP);
    for (int p = 0; p < 2; p++)
      for (int t = 0; t <= l; t++) {
        int pi = t < l ? t : c->L;
        u64 q = c->q[pi];
        for (size_t k = 0; k < N; k++) {
          size_t idx = (size_t)p * ne + (size_t)t * N + k;
          ACC[idx] = addmod(ACC[idx], mulmod(IP[idx], m[(size_t)t * N + k], q), q);
        }
      }
    ock_automorph_ntt(c, g, v, c0g, l);
    for (int t = 0; t < l; t++)
      for (size_t k = 0; k < N; k++) {
        size_t idx = (size_t)t * N + k;
        u64 q = c->q[t];
        C[idx] = addmod(C[idx], mulmod(c0g[idx], m[idx], q), q);
      }
  }
  moddown(c, ACC, l, md);
  for (int p = 0; p < 2; p++)
    for (int t = 0; t < l; t++)
      for (size_t k = 0; k < N; k++) {
        size_t idx = (size_t)p * n + (size_t)t * N + k;
        out[idx] = addmod(C[idx], md[idx], c->q[t]);
      }
  free(D); free(Dg); free(IP); free(ACC); free(C); free(c0g); free(md);
}
