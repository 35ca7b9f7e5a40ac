/*
 * oracle/ckks_oracle.h -- TEST INFRASTRUCTURE ONLY (the limb-level checker).
 *
 * A plain-C CPU restatement of the RNS-CKKS evaluator that the B200 path
 * implements.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product (libhegpu.so) never links it.
 *
 * Parity status: the reference (`hesim`) is a plaintext slot simulator with
 * no CKKS (reference SPEC.md:8,89,101; proj/README.md:3-7), and the paper's
 * SEAL is not vendored.  CKKS limbs therefore have no
 * reference oracle: this file is builder-authored from the CKKS literature
 * ("parity unpinned" at the limb level).  What IS pinned against the
 * reference is the slot semantics the limbs decrypt to (rotation direction
 * proj/src/slotvec.cpp:42-66, HS layout proj/src/matvec.cpp:45-105, conv
 * packing proj/src/convlower.cpp:9-74, merge :145-160) and the HOP counts;
 * see oracle/hesim_oracle.py and tests/test_oracle_*.py.
 *
 * Conventions (shared, by specification, with the CUDA path):
 *   - primes: largest primes below 2^bits with p == 1 (mod 2N), requested in
 *     order q_0..q_{L-1} then the special prime P (index L); no repeats.
 *   - psi: for x = 2,3,..: g = x^((p-1)/2N); first g with g^N == -1.
 *   - NTT: Cooley-Tukey with psi powers in bit-reversed order, natural
 *     input, bit-reversed output (slot k holds a(psi^(2*brv(k)+1))); all
 *     residues canonical in [0, p).
 *   - a polynomial at level l is l limbs of N words (limb i mod prime i);
 *     a ciphertext is [2][l][N]; the extended basis appends the P limb.
 *   - everything integer is exact, so any evaluation order gives identical
 *     limbs; the only roundings are rescale / ModDown (centered lift of the
 *     dropped residue) and FP64 encoding (fixed operation order, no FMA).
 */
#ifndef CKKS_ORACLE_H
#define CKKS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ock_ctx ock_ctx;

ock_ctx* ock_create(int logN, int L, const int* qbits, int pbits);
void ock_destroy(ock_ctx* c);
uint64_t ock_prime(const ock_ctx* c, int i);
uint64_t ock_psi(const ock_ctx* c, int i);
int ock_N(const ock_ctx* c);

/* single-limb transforms, prime index pi (0..L-1 = q_i, L = P) */
void ock_ntt(const ock_ctx* c, int pi, uint64_t* a);
void ock_intt(const ock_ctx* c, int pi, uint64_t* a);

/* automorphism X -> X^g applied to nlimbs NTT-domain limbs (limb-agnostic) */
void ock_automorph_ntt(const ock_ctx* c, uint64_t g, const uint64_t* in,
                       uint64_t* out, int nlimbs);
/* same in the coefficient domain for prime pi */
void ock_automorph_coeff(const ock_ctx* c, int pi, uint64_t g,
                         const uint64_t* in, uint64_t* out);
uint64_t ock_galois_left(const ock_ctx* c, int64_t r);  /* 5^r mod 2N */
uint64_t ock_galois_right(const ock_ctx* c, int64_t r); /* 5^(S-r) */

/* FP64 canonical-embedding encode of len real slot values at `scale`,
 * producing `level` limbs (+ the P limb when with_p) in the NTT domain. */
void ock_encode(const ock_ctx* c, const double* z, int len, double scale,
                int level, int with_p, uint64_t* out);
/* integer-valued coefficient vector (doubles) -> NTT limbs */
void ock_encode_coeffs(const ock_ctx* c, const double* coeffs, int level,
                       int with_p, uint64_t* out);
/* FP64 coefficient vector (before rounding) of an encoding */
void ock_encode_fp(const ock_ctx* c, const double* z, int len, double scale,
                   double* coeffs_out);
void ock_decode(const ock_ctx* c, const uint64_t* pt, int level, double scale,
                double* slots_out);
/* reference O(N*S) canonical embedding (small N only) */
void ock_encode_direct(const ock_ctx* c, const double* z, int len,
                       double scale, double* coeffs_out);

/* keys: s is (L+1) limbs NTT domain */
void ock_secret(const ock_ctx* c, uint64_t seed, uint64_t* s_out);
/* key-switching key from s' (L+1 limbs NTT) to s: layout [L][2][L+1][N] */
void ock_gen_ksk(const ock_ctx* c, uint64_t seed, uint64_t kind, uint64_t g,
                 const uint64_t* s, const uint64_t* sprime, uint64_t* key);
void ock_gen_galois_key(const ock_ctx* c, uint64_t seed, const uint64_t* s,
                        uint64_t g, uint64_t* key);
void ock_gen_relin_key(const ock_ctx* c, uint64_t seed, const uint64_t* s,
                       uint64_t* key);

void ock_encrypt(const ock_ctx* c, uint64_t seed, uint64_t nonce,
                 const uint64_t* s, const uint64_t* pt, int level,
                 uint64_t* ct);
void ock_decrypt(const ock_ctx* c, const uint64_t* s, const uint64_t* ct,
                 int level, uint64_t* pt);

/* evaluator (all NTT domain, level l) */
void ock_add(const ock_ctx* c, const uint64_t* a, const uint64_t* b, int l,
             uint64_t* out);
void ock_add_pc(const ock_ctx* c, const uint64_t* a, const uint64_t* pt, int l,
                uint64_t* out);
void ock_mul_pc(const ock_ctx* c, const uint64_t* a, const uint64_t* pt, int l,
                uint64_t* out);
void ock_rescale(const ock_ctx* c, const uint64_t* a, int l, uint64_t* out);
void ock_rotate(const ock_ctx* c, const uint64_t* a, int l, uint64_t g,
                const uint64_t* key, uint64_t* out);
void ock_square(const ock_ctx* c, const uint64_t* a, int l,
                const uint64_t* rlk, uint64_t* out);
void ock_conv_mac(const ock_ctx* c, const uint64_t* taps, int ntaps, int l,
                  const double* weights, int c_out, double wscale,
                  const uint64_t* bias_pts, uint64_t* maps_out);
void ock_merge(const ock_ctx* c, const uint64_t* maps, int nmaps, int l,
               int64_t w, const uint64_t* keys, uint64_t* out);
void ock_hs_hoisted(const ock_ctx* c, const uint64_t* v, int l, int ndiag,
                    const int64_t* rots, const uint64_t* masks_ext,
                    const uint64_t* keys, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
