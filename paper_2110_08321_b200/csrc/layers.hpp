// layers.hpp -- the reference's layer kernels on the CKKS engine:
//   ConvLayer   conv_packed_forward  proj/src/convlower.cpp:39-74
//   merge_maps  merge_maps           proj/src/convlower.cpp:145-160
//   square_layer square_layer        proj/src/convlower.cpp:141-143
//   HsPlan      extract_diagonals + hs_matvec  proj/src/matvec.cpp:45-105
#pragma once
#include <map>
#include <memory>

#include "engine.hpp"

namespace hegpu {

// conv-pack MAC with scalar weights round(w * q_{l-1}) (the tap ciphertexts
// are zero beyond the used slots, so the reference's masked constant
// plaintext and the scalar agree up to encryption noise),
// the per-map bias plaintext on the first w_used slots, then one rescale.
struct ConvLayer {
  int ntaps, c_out, level;
  u64d* w = nullptr;     // [c_out][ntaps][level] Montgomery scalars
  u64d* bias = nullptr;  // [c_out][level][N] Montgomery, slot order
  uint32_t* wa = nullptr;  // tensor-core A fragments (launch_conv_imma)
  uint8_t* wtc = nullptr;  // tcgen05 weight operand images (launch_conv_tc), null if unsupported
  int cps = 0, kbn = 0;    // map pairs, 4-tap blocks
  ConvLayer(Context& c, int ntaps, int c_out, const double* weights, const double* bias_vals, int w_used,
            int level, double tap_scale);
  ~ConvLayer();
  ConvLayer(const ConvLayer&) = delete;
  ConvLayer& operator=(const ConvLayer&) = delete;
  void run(Context& c, const CtBatch& taps, CtBatch& maps);  // mac + rescale
  // the multiply-accumulate alone: prod [B][c_out] at `level` (scale x q_top)
  void mac(Context& c, const CtBatch& taps, CtBatch& prod);
  // the same on B images of compact fresh taps (device bytes at `level`):
  // expanded into full ciphertexts first (io.cu), then the MAC
  void mac_compact(Context& c, const uint8_t* taps, int B, double tap_scale, CtBatch& prod);
  // merged mode (the stage driver's Conv1 + Flat1): the
  // client packs every tap replicated at the c_out map offsets co * w_used,
  // the weights become block plaintexts P_s (W[co][s] on block co, scale
  // q_{level-1}) and the bias one block plaintext, so the MAC lands each map
  // at its merged slots: ONE ciphertext per image, no merge rotations
  void make_merged(Context& c, const double* weights, const double* bias_vals, int w_used, double tap_scale,
                   int regions = 1);
  bool merged = false;
  int regions = 1;  // merged: taps per input ciphertext (tap s in region s % regions, offset region * c_out * w)
  int cts_per_image() const { return merged ? (ntaps + regions - 1) / regions : ntaps; }
  u64d* pw = nullptr;     // [ntaps][level][N] split-31 Montgomery block plaintexts
  u64d* pbias = nullptr;  // [level][N] standard-form block bias (product scale)
  int out_per_image() const { return merged ? 1 : c_out; }
  Context* ctx;
};

// conv_packed_forward with the reference's MASKED constant plaintexts
// pt(w[co,t] on slots < w_used) (convlower.cpp:55-63) for taps whose slots
// beyond w_used are not zero -- the RepackConv stage's rotated group
// ciphertexts (netcompile.cpp:352-379).  taps [ntaps][B] tap-major at
// `level`, maps [c_out][B] map-major at level - 1 (MAC + bias + rescale).
struct MaskedConv {
  int ntaps = 0, c_out = 0, level = 0;
  u64d* pw = nullptr;     // [c_out][ntaps][level][N] split-31 Montgomery, scale q_{level-1}
  u64d* pbias = nullptr;  // [c_out][level][N] standard form, scale tap_scale * q_{level-1}
  Context* ctx = nullptr;
  MaskedConv(Context& c, int ntaps, int c_out, const double* weights, const double* bias_vals, int w_used, int level,
             double tap_scale);
  ~MaskedConv();
  MaskedConv(const MaskedConv&) = delete;
  MaskedConv& operator=(const MaskedConv&) = delete;
  void run(Context& c, const CtBatch& taps, CtBatch& maps);
};

void merge_maps(Context& c, const CtBatch& maps, int nmaps, int64_t w, CtBatch& out);
void square_layer(Context& c, const CtBatch& a, CtBatch& out);  // tensor + relin + rescale

struct HsDiag {
  int index;      // diagonal i of extract_diagonals
  int64_t right;  // right rotation (= i)
  int shift;      // device left shift (S - i) mod S
};

struct HsPlan {
  int m = 0, n = 0, m_eff = 0, folds = 0, level = 0;
  std::vector<HsDiag> diag;   // kept (non-zero) diagonals in order
  u64d* masks = nullptr;      // [kept][level+1][N] Montgomery, slot order
  int* d_r = nullptr;         // [kept] right rotations
  int* d_chunk = nullptr;     // chunk boundaries
  int nchunk = 0;
  std::vector<int> h_chunk;   // chunk boundaries (host copy)
  std::map<std::pair<int, int>, std::pair<int*, int>> sub_chunks;  // diagonal range -> (device chunks, count)
  u64d* fkeys = nullptr;      // [keyed][level][2][level+1][N] key_i * mask_i (first run)
  bool keys_resolved = false;
  // tensor-core path (hs_imma.cu): chunks with their A fragments, built on
  // the first run with a batch of >= hs_imma_min_batch() images
  std::vector<HsImmaChunk> imma;
  u64d* imma_ec = nullptr;    // [np][2][4][2] epilogue constants
  u64d* imma_pmod = nullptr;  // [level] P mod q_t
  int* d_rdiag = nullptr;     // [S] right rotation -> kept diagonal (or -1)
  bool imma_built = false;
  void ensure_imma(Context& c);
  void ensure_imma_consts(Context& c);
  // the tcgen05 path (hs_tc.cu): chunks (r_lo, r_hi, keyed, ndiag) with their A tables
  struct TcChunk {
    int r_lo, r_hi, keyed, ndiag;
    uint8_t* at;
  };
  std::vector<TcChunk> tc;
  u64d* tc_ce = nullptr;  // [np][8] 2^(8e) R mod q
  u64d* tc_pR = nullptr;  // [level] P R mod q_t
  bool tc_built = false, tc_unfit = false;
  // builds the A tables on first use; false if they do not fit the free
  // device memory (the caller falls back to the integer kernels)
  bool ensure_tc(Context& c);
  bool use_imma(Context& c, int B, int i_lo, int i_hi) const;
  // the log-depth fold (matvec.cpp:101-103) as hoisted rotation sums: the
  // `folds` doublings in groups of <= kMaxFoldGroup (fold_groups), each a
  // unit-mask plan over rot_left(., m_eff 2^offset u), u < 2^size, at level - 1
  static constexpr int kMaxFoldGroup = 5;
  std::vector<std::unique_ptr<HsPlan>> fold;
  bool unit_masks = false;  // a rotation-sum plan (build_rotsum)
  std::vector<int> fold_groups() const;
  std::vector<int64_t> fold_rights(int offset, int size) const;  // ascending, 0 first
  void build_rotsum(Context& c, const std::vector<int64_t>& rights, int level);
  void build(Context& c, const double* A, int m, int n, int level, bool skip_zero);
  void release();
  std::vector<int64_t> right_rotations() const;  // diagonals, then folds
  void run(Context& c, const CtBatch& v, CtBatch& out);
  // distributed HS (config 3): the extended-basis accumulators of the kept
  // diagonals [i_lo, i_hi) -- acc [B][2][l+1][N], cacc [B][2][l][N] -- and the
  // finish (ModDown, rescale, folds) on accumulators summed over nparts
  // such ranges (entries < nparts * q, reduced here)
  void ensure_keys(Context& c);
  void accumulate(Context& c, const CtBatch& v, int i_lo, int i_hi, u64d* acc, u64d* cacc);
  void finish(Context& c, int B, double v_scale, u64d* acc, u64d* cacc, int nparts, CtBatch& out);
  size_t acc_words(int B, int N) const { return (size_t)B * (2 * (level + 1) + 2 * level) * N; }
  Context* ctx = nullptr;
};

// LoLa comparators (lola.cu): kind 0 = lola_dense_matvec, 1 = lola_stacked_matvec
// (proj/src/matvec.cpp:107-166).  Input at `level`, outputs at level - 2:
// dense -> B * m ciphertexts (image-major, A[i] . x in slot 0), stacked ->
// B ciphertexts (row i in slot slot_of_row(i)).
struct LolaPlan {
  int kind = 0, m = 0, n = 0, level = 0, delta = 1, folds = 0, k = 1, batches = 0;
  u64d* rows = nullptr;   // [batches][level][N] product plaintexts (scale q_{level-1})
  u64d* masks = nullptr;  // [1 or batches][level-1][N] clearing masks (scale q_{level-2})
  void build(Context& c, int kind, const double* A, int m, int n, int level);
  void release();
  std::vector<int64_t> right_rotations() const;
  int out_count(int B) const;
  int64_t slot_of_row(int i) const;
  void run(Context& c, const CtBatch& v, CtBatch& out);
  Context* ctx = nullptr;
};

}  // namespace hegpu
