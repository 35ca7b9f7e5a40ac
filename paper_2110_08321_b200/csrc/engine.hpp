// engine.hpp -- device-side engine state shared by the CUDA translation
// units and the C-ABI (csrc/capi.cu).
//
// Device layout: an NTT-domain limb is stored in SLOT ORDER
// (position p < S holds a(psi^(5^p)), p >= S holds a(psi^(-5^(p-S)))), so
// the Galois automorphism X -> X^(5^s) is a cyclic shift by s inside each
// half -- every rotation becomes coalesced streaming instead of a gather.
// Plaintexts, keys and HS masks are kept in Montgomery form.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "core.hpp"
#include "modarith.cuh"

namespace hegpu {

#define HEGPU_MAX_BATCH_PERIOD 64

// per-launch description of which key / shift row b uses (b % period)
struct KeyRowMap {
  int period;
  int shift[HEGPU_MAX_BATCH_PERIOD];             // left shift s (0 = none)
  const u64d* key[HEGPU_MAX_BATCH_PERIOD];       // device key (Montgomery)
  // optional grouped input rows (merge): row b reads src + (b / grp) *
  // grp_stride + (b % grp) * src_stride; grp = 0 means b * src_stride
  int grp;
  long grp_stride;
};

struct DeviceKey {
  u64d* data = nullptr;  // [L][2][L+1][N], slot order, Montgomery form
  int shift = 0;         // left rotation amount (Galois 5^shift)
  std::vector<u64> wire; // host wire copy (exported for tests)
};

struct Meter {
  std::vector<std::pair<std::string, std::array<int64_t, 5>>> stages;
  std::array<int64_t, 5> total{};
  int cur = -1;
  void begin(const std::string& label);
  void bump(int field, int64_t n);
};

struct Context {
  hegpu_params hp{};
  std::unique_ptr<Params> P;
  std::unique_ptr<Client> client;
  int device = 0;
  cudaStream_t stream = nullptr;
  PrimeTable primes{};
  u64d* d_tw = nullptr;          // [np][2][N] (w, w') pairs: forward, inverse
  double* d_twd = nullptr;       // [np][2][N] w as doubles (FP64 NTT path, primes < 2^45)
  double* d_fpq = nullptr;       // [np][2] (q, 1/q), or (0, 0) for primes on the integer path
  bool fp_all = false;           // every prime on the FP64 path: the FP64-only NTT builds run
  u64d* d_consts = nullptr;      // [np]: ninv, ninv' ; then [np][np]: qinv(value, shoup)
  uint32_t* d_slot_src = nullptr;  // [N]
  std::map<int, DeviceKey> rot_keys;  // keyed by left shift in [1, S)
  DeviceKey relin;
  bool has_relin = false;
  Meter meter;
  std::string last_error;
  int64_t launches = 0;
  size_t ws_bytes = 0;
  // per-kernel event timing (hegpu_kernel_timer): every launch of the named
  // kernel is bracketed by two events on the context stream
  std::string ktimer_name;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ktimer_events;
  size_t ktimer_used = 0;
  double ktimer_bytes = 0;
  double ktimer_ops = 0;  // algorithmic modular multiply(-accumulate)s
  // key-switch work actually executed (hegpu_ks_counters): ModUps, key
  // inner products, ModDowns, rescaled ciphertexts
  std::array<int64_t, 4> ks{};

  int N() const { return P->n; }
  int S() const { return P->slots; }
  int L() const { return P->L; }
  const u64d* ninv_tab() const { return d_consts; }
  const u64d* qinv_tab() const { return d_consts + 2 * (size_t)P->np(); }
  u64d* alloc(size_t words);
  void free(u64d* p);
  const DeviceKey& rot_key(int shift);
};

struct CtBatch {
  Context* ctx;
  int count, level;
  double scale;
  u64d* d;  // [count][2][level][N]
  size_t words() const { return (size_t)count * 2 * level * ctx->N(); }
  size_t stride() const { return (size_t)2 * level * ctx->N(); }
};

struct PtBatch {
  Context* ctx;
  int count, level, with_p;
  double scale;
  u64d* d;  // [count][level + with_p][N], Montgomery form
  int limbs() const { return level + with_p; }
  size_t words() const { return (size_t)count * limbs() * ctx->N(); }
};

// ---------------------------------------------------------------- launchers
void check_cuda(cudaError_t e, const char* what);
#define CK(x) ::hegpu::check_cuda((x), #x)

enum { KS_MODUP = 0, KS_INNER = 1, KS_MODDOWN = 2, KS_RESCALE = 3 };

// every C-ABI call binds the context's device first, so contexts on
// different GPUs can be driven from one thread (single-process multi-GPU)
inline void bind_device(const Context* c) {
  if (c && c->device >= 0 && c->stream) {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != c->device) check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
  }
}
inline int current_device() {
  int d = 0;
  check_cuda(cudaGetDevice(&d), "cudaGetDevice");
  return d;
}
// one-time per-device setup (cudaFuncSetAttribute and device attributes are
// per device): true the first time it is asked for the current device
struct PerDeviceOnce {
  unsigned long long mask = 0;
  bool first() {
    const unsigned long long bit = 1ull << (current_device() & 63);
    if (mask & bit) return false;
    mask |= bit;
    return true;
  }
};
// streaming multiprocessors of the current device (cached per device)
inline int device_sms() {
  static int sms[64] = {0};
  const int d = current_device() & 63;
  if (!sms[d]) check_cuda(cudaDeviceGetAttribute(&sms[d], cudaDevAttrMultiProcessorCount, d), "sm count");
  return sms[d];
}

// Brackets one kernel launch: counts it and, when the context's kernel
// timer names this kernel, records start/stop events around it.
struct Launch {
  Context& c;
  cudaEvent_t stop = nullptr;
  // bytes: the launch's ALGORITHMIC HBM bytes (each operand read or written
  // once), accumulated for the timed kernel -> roofline achieved GB/s;
  // ops: its algorithmic modular multiplies (MAC terms / butterflies)
  Launch(Context& cc, const char* name, double bytes = 0.0, double ops = 0.0) : c(cc) {
    ++c.launches;
    if (!c.ktimer_name.empty() && c.ktimer_name == name) {
      c.ktimer_bytes += bytes;
      c.ktimer_ops += ops;
      if (c.ktimer_used == c.ktimer_events.size()) {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        c.ktimer_events.emplace_back(a, b);
      }
      auto& ev = c.ktimer_events[c.ktimer_used++];
      CK(cudaEventRecord(ev.first, c.stream));
      stop = ev.second;
    }
  }
  void end() {
    if (stop) CK(cudaEventRecord(stop, c.stream));
    CK(cudaGetLastError());
  }
};
// LAUNCH_B(ctx, "k_name", bytes, k_name<<<grid, block, smem, ctx.stream>>>(args...));
#define LAUNCH_B(ctx, name, bytes, ...)          \
  do {                                           \
    ::hegpu::Launch _launch(ctx, name, (bytes)); \
    __VA_ARGS__;                                 \
    _launch.end();                               \
  } while (0)
#define LAUNCH(ctx, name, ...) LAUNCH_B(ctx, name, 0.0, __VA_ARGS__)
// LAUNCH_BO: as LAUNCH_B plus the launch's algorithmic modular-multiply count
#define LAUNCH_BO(ctx, name, bytes, ops, ...)             \
  do {                                                    \
    ::hegpu::Launch _launch(ctx, name, (bytes), (ops));   \
    __VA_ARGS__;                                          \
    _launch.end();                                        \
  } while (0)

// compact fresh ciphertexts (io.cu): bytes per ct, device expansion
size_t compact_ct_bytes(Context& c, int level);
void launch_expand_compact(Context& c, const uint8_t* src, int count, int level, u64d* dst);
struct CompactLayout;
CompactLayout compact_layout(Context& c, int level);
// twiddle tables [np][fwd, inv][N] of (w, w') pairs -> c.d_tw
void upload_twiddles(Context& c);
bool ntt_fp_enabled();
// coefficient rows -> slot-order NTT rows; row r uses limb r % nl (limb l ->
// prime l, or P for l == p_limb when p_limb >= 0)
void launch_ntt_rows(Context& c, const u64d* src, u64d* dst, int rows, int nl, int p_limb);
// slot-order NTT rows -> coefficient rows (x N^{-1}); 2-level row map
void launch_intt_rows(Context& c, const u64d* src, u64d* dst, int n_outer, int n_inner,
                      long src_outer, long src_inner, long dst_outer, long dst_inner,
                      const int* prime_of_inner /* n_inner entries, host */);
// wire (bit-reversed) <-> slot order permutation on count*limbs rows
void launch_wire_to_slot(Context& c, const u64d* src, u64d* dst, size_t rows, int to_mont,
                         int nl, int p_limb);
void launch_slot_to_wire(Context& c, const u64d* src, u64d* dst, size_t rows, int from_mont,
                         int nl, int p_limb);

// key switching pieces (ks.cu)
struct KsWork {
  u64d* tmp;  // [B][l][N] coefficient digits
  u64d* D;    // [B][l][l+1][N] ModUp digits, slot order
  u64d* acc;  // [B][2][l+1][N] extended-basis accumulators
  u64d* tmpP; // [B][2][N] dropped-limb coefficients
};
// d rows: poly at src + b*src_stride (l limbs); keys/shifts per b % period
void ks_modup(Context& c, const u64d* src, long src_stride, int B, int l, const KeyRowMap* shifts,
              u64d* tmp, u64d* D);
void ks_inner(Context& c, const u64d* D, int B, int l, const KeyRowMap& keys, u64d* acc);
// out[b][p][t] = (src[b][p][t] - lift(src[b][p][last])) * inv + add[b][p][t](shifted)
struct DropArgs {
  const u64d* src; long src_b, src_p; int src_limbs;  // last limb is dropped
  u64d* dst; long dst_b, dst_p;
  int pd;          // prime index of the dropped limb
  int nl;          // output limbs (primes 0..nl-1)
  const u64d* add; long add_b, add_p; int add_mask;  // add term per poly (bit p)
  const KeyRowMap* shifts;  // shift for add reads of poly 0 (may be null)
  // ModDown (pd = P) followed by the rescale that drops q_{l-1}, fused
  // (ntt.cu k_md_intt / k_md_ntt): dst gets nl = l - 1 limbs; add unshifted
  int fuse_rescale;
};
void drop_last_limb(Context& c, int B, const DropArgs& a, u64d* tmpP);
// the two NTT builds (ntt.cu: 16 words/thread, ntt_r8.cu: 8 for N <= 2^13)
void launch_ntt_rows_r8(Context& c, const u64d* src, u64d* dst, int rows, int nl, int p_limb);
void launch_ntt_rows_r16(Context& c, const u64d* src, u64d* dst, int rows, int nl, int p_limb);
void launch_intt_rows_r8(Context& c, const u64d* src, u64d* dst, int n_outer, int n_inner, long so, long si,
                         long dox, long di, const int* prime_of_inner);
void launch_intt_rows_r16(Context& c, const u64d* src, u64d* dst, int n_outer, int n_inner, long so, long si,
                          long dox, long di, const int* prime_of_inner);
void ks_modup_r8(Context& c, const u64d* src, long src_stride, int B, int l, const KeyRowMap* shifts, u64d* tmp,
                 u64d* D);
void ks_modup_r16(Context& c, const u64d* src, long src_stride, int B, int l, const KeyRowMap* shifts, u64d* tmp,
                  u64d* D);
void drop_last_limb_r8(Context& c, int B, const DropArgs& a, u64d* tmpP);
void drop_last_limb_r16(Context& c, int B, const DropArgs& a, u64d* tmpP);
// FP64-only builds (every prime < 2^45): ntt_fp16.cu, ntt_fp8.cu
#define HEGPU_NTT_DECL(S)                                                                                   \
  void launch_ntt_rows##S(Context& c, const u64d* src, u64d* dst, int rows, int nl, int p_limb);            \
  void launch_intt_rows##S(Context& c, const u64d* src, u64d* dst, int n_outer, int n_inner, long so, long si, \
                           long dox, long di, const int* prime_of_inner);                                 \
  void ks_modup##S(Context& c, const u64d* src, long src_stride, int B, int l, const KeyRowMap* shifts,      \
                   u64d* tmp, u64d* D);                                                                     \
  void drop_last_limb##S(Context& c, int B, const DropArgs& a, u64d* tmpP);
HEGPU_NTT_DECL(_fp16)
HEGPU_NTT_DECL(_fp8)
#undef HEGPU_NTT_DECL
void drop_last_limb_fp16n(Context& c, int B, const DropArgs& a, u64d* tmpP);  // ntt_fp16n.cu

// pointwise (eval.cu)
void launch_add(Context& c, const u64d* a, const u64d* b, u64d* out, int count, int l);
void launch_add_plain(Context& c, const u64d* a, const u64d* p, long p_stride, u64d* out, int count, int l);
void launch_mul_plain(Context& c, const u64d* a, const u64d* p, long p_stride, u64d* out, int count, int l);
void launch_tensor_square(Context& c, const u64d* a, u64d* d01, u64d* d2, int count, int l);
// the same MAC on the int8 tensor cores (conv_imma.cu); wa: per limb, map
// pair, 4-tap block and lane the A fragment (uint4) of the byte planes of
// W * 2^(8i) mod q
bool conv_imma_supported(Context& c);
// the same MAC on tcgen05 (conv_tc.cu): positions as MMA rows, weight byte
// planes as accumulator columns; wb from conv_tc_weights
bool conv_tc_supported(Context& c, int ntaps, int c_out, int l);
std::vector<uint8_t> conv_tc_weights(Context& c, int ntaps, int c_out, int l, const std::vector<u64>& ws);
void launch_conv_tc(Context& c, const u64d* taps, int B, int ntaps, int l, const uint8_t* wb, int c_out,
                    const u64d* bias, u64d* out);
// limb t packs 3 maps x 5 weight-byte planes per MMA row tile (q_t < 2^40)
bool conv_imma_triples(Context& c, int t, int c_out);
void launch_conv_imma(Context& c, const u64d* taps, int B, int ntaps, int l, const uint32_t* wa, int cps, int kbn,
                      int c_out, const u64d* bias, u64d* out);
// out[b] = sum_s taps[b][s] * pw[s] + pbias (poly 0): per-position plaintext
// weights (the merged first layer), pw split-31 Montgomery, pbias standard
void launch_conv_pt(Context& c, const u64d* taps, int B, int ntaps, int regions, int l, const u64d* pw,
                    const u64d* pbias, u64d* out);
// masked-constant conv over every output map in one launch: taps [ntaps][B]
// (tap-major), pw [c_out][ntaps][l][N] split-31 Montgomery, pbias [c_out][l][N]
// standard form, out [c_out][B] (map-major), all at level l
void launch_conv_masked(Context& c, const u64d* taps, int B, int ntaps, int c_out, int l, const u64d* pw,
                        const u64d* pbias, u64d* out);
void launch_conv_mac(Context& c, const u64d* taps, int B, int ntaps, int l, const u64d* wmont /*[c_out][ntaps][l]*/,
                     int c_out, const u64d* bias /*[c_out][l][N] mont*/, u64d* out);
struct HsDiagTable {
  int ndiag;
  int keyed;                 // diagonals with r > 0 (carry a fused key)
  const int* r;              // [ndiag] device: right rotation r_i, ascending
  // fused keys key_i * mask_i of the keyed diagonals, contiguous:
  // diagonal i (>= first_keyed) at fk + (i - first_keyed) * fk_words, [l][2][l+1][N]
  const u64d* fk;
  size_t fk_words;
  int first_keyed;           // 1 when diagonal 0 has r = 0 (no key), else 0
  int own_c1;                // this run carries diagonal 0's c1 * mask term (the range starts at 0)
  const u64d* masks;         // [ndiag][l+1][N] mont, slot order
  int nchunk;
  const int* chunk;          // [nchunk + 1] diagonal ranges with r span < hs_chunk_span()
  int unit_masks = 0;        // every mask is 1 (the fold's hoisted rotation sum)
};
int hs_chunk_span();
void launch_hs_diag(Context& c, const u64d* v, int B, int l, const u64d* D, const HsDiagTable& t,
                    u64d* acc, u64d* cacc);
void launch_fuse_key(Context& c, const u64d* key, const u64d* mask, int l, u64d* fk);
// the same accumulation on the int8 tensor cores (hs_imma.cu): one chunk of
// kept diagonals with r in [r_lo, r_hi], its A fragments wt ([l+1][N][ns][32]
// uint4: byte planes of the fused keys and P * masks per position)
struct HsImmaChunk {
  int r_lo, r_hi, ns;
  int keyed, ndiag;  // kept diagonals in the chunk (with a key / all)
  u64d* wt;
};
int hs_imma_chunk_span(int l);
// the same accumulation on tcgen05 (hs_tc.cu): per chunk of kept diagonals
// with r in [r_lo, r_hi] (span <= hs_tc_chunk_span), A tables `at` built by
// launch_hs_tc_tiles (hs_tc_table_bytes); ce [np][8] = 2^(8e) R mod q, pR[t] = P R mod q_t
bool hs_tc_enabled();
constexpr int kHsTcMaxLevel = 8;  // k_hs_tc<J> is instantiated for J = l + 1 <= 9
int hs_tc_chunk_span(int l);
size_t hs_tc_table_bytes(Context& c, int l, int span);
void launch_hs_tc_tiles(Context& c, int l, const struct HsDiagTable& t, const u64d* pR, const int* rdiag, int r_lo,
                        int r_hi, uint8_t* at);
void launch_hs_tc(Context& c, const u64d* v, int B, int l, const u64d* D, int r_lo, int r_hi, const uint8_t* at,
                  const u64d* ce, int accumulate, u64d* acc, int keyed, int ndiag);
bool hs_imma_supported(Context& c, int l);
size_t hs_imma_tile_words(Context& c, int l, const HsImmaChunk& ch);
// rdiag[r] = kept diagonal index of right rotation r (or -1); pmod[t] = P mod q_t
void launch_hs_imma_tiles(Context& c, int l, const HsDiagTable& t, const u64d* pmod, const int* rdiag,
                          const HsImmaChunk& ch, u64d* wt);
// acc (= or += when accumulate) for one chunk; ec: [np][2][4][2] epilogue constants
void launch_hs_imma(Context& c, const u64d* v, int B, int l, const u64d* D, const HsImmaChunk& ch,
                    const u64d* ec, int accumulate, u64d* acc);
// cacc of the tensor-core path: 0, or diagonal 0's c1 * m0 in part 1
void launch_hs_cacc(Context& c, const u64d* v, const u64d* m0, int B, int l, int c1_term, u64d* cacc);
// re-pack Montgomery multiplier words x -> (x mod 2^31) | (x >> 31) << 32
void launch_split31(Context& c, u64d* p, size_t words);
// x -> x mod q(limb) for rows of nl limbs (limb p_limb is the special prime P);
// x < 2^64 (e.g. a sum of partial accumulators from several GPUs)
void launch_reduce_rows(Context& c, u64d* p, size_t words, int nl, int p_limb);

// high-level evaluator (eval.cu)
void eval_rescale(Context& c, const CtBatch& a, CtBatch& out);
// out = rot(a) for B ciphertexts at level l (strided), per-row shift/key
void eval_rotate(Context& c, const u64d* a, long a_stride, int B, int l, const KeyRowMap& km, u64d* out,
                 long out_stride);
void eval_square(Context& c, const CtBatch& a, CtBatch& out);  // tensor + relin, no rescale
void eval_square_rescale(Context& c, const CtBatch& a, CtBatch& out);  // tensor + relin + rescale (fused)
void eval_merge(Context& c, const CtBatch& maps, int nmaps, const KeyRowMap& km, CtBatch& out);
// one rank's share (maps lo .. lo+M-1 per image) of a merge: acc [B][2][l+1][N], C [B][2][l][N]
void eval_merge_partial(Context& c, const CtBatch& maps, int M, int lo, int64_t w, u64d* acc, u64d* C);

}  // namespace hegpu
