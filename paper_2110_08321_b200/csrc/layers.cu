// layers.cu -- conv-pack, merge, square and Halevi-Shoup layers on the
// CKKS engine (reference semantics: proj/src/convlower.cpp:39-74,141-160,
// proj/src/matvec.cpp:45-105).
#include <algorithm>
#include <cmath>
#include <string>

#include "layers.hpp"

namespace hegpu {

namespace {

void need(bool ok, int code, const std::string& msg) {
  if (!ok) fail(code, msg);
}

// host wire limbs -> device slot order, Montgomery
void upload_mont(Context& c, const std::vector<u64>& wire, u64d* dst, size_t rows, int nl, int p_limb) {
  u64d* stage = c.alloc(wire.size());
  CK(cudaMemcpyAsync(stage, wire.data(), wire.size() * 8, cudaMemcpyHostToDevice, c.stream));
  launch_wire_to_slot(c, stage, dst, rows, 1, nl, p_limb);
  c.free(stage);
  CK(cudaStreamSynchronize(c.stream));
}

int ceil_log2(int64_t x) {
  int b = 0;
  while ((int64_t{1} << b) < x) ++b;
  return b;
}
int64_t next_pow2(int64_t x) {
  int64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}
// proj/src/matvec.cpp:29-33
bool plain_branch_fits(int64_t m, int64_t n, int64_t S) {
  if (S < m + n - 1) return false;
  const int b = ceil_log2((m + n - 1 + m - 1) / m);
  return (m << b) <= S;
}

}  // namespace

// ------------------------------------------------------------------ conv ----
ConvLayer::ConvLayer(Context& c, int nt, int co_n, const double* weights, const double* bias_vals, int w_used,
                     int lvl, double tap_scale)
    : ntaps(nt), c_out(co_n), level(lvl), ctx(&c) {
  need(level >= 2, HEGPU_ERR_CAPACITY, "conv_packed_forward: no prime left to rescale");
  const Params& P = *c.P;
  const u64 qlast = P.q(level - 1);
  std::vector<u64> w((size_t)c_out * ntaps * level);
  for (int co = 0; co < c_out; ++co)
    for (int t = 0; t < ntaps; ++t) {
      const double x = std::rint(weights[(size_t)co * ntaps + t] * (double)qlast);
      for (int li = 0; li < level; ++li) {
        const u64 q = P.q(li);
        const u64 wm = mul_mod(residue_of_double(x, q), P.primes[li].r_mod, q);  // Montgomery form
        w[((size_t)co * ntaps + t) * level + li] = (wm & 0x7FFFFFFFull) | ((wm >> 31) << 32);  // split-31
      }
    }
  CK(cudaMalloc((void**)&this->w, w.size() * 8));
  CK(cudaMemcpy(this->w, w.data(), w.size() * 8, cudaMemcpyHostToDevice));
  // tensor-core operand: per limb, map pair cp, 4-tap block kb and lane, the
  // m16n8k32 A fragment whose (row, col) = (map 2cp + row / 8, byte plane
  // e = row % 8; tap 4kb + col / 8, tap byte i = col % 8) holds byte e of
  // W[co][s] * 2^(8i) mod q (standard form)
  cps = (c_out + 1) / 2;
  kbn = (ntaps + 3) / 4;
  {
    std::vector<u64> ws((size_t)level * c_out * ntaps * 8);  // [li][co][s][i]
    for (int li = 0; li < level; ++li) {
      const u64 q = P.q(li);
      for (int co = 0; co < c_out; ++co)
        for (int s = 0; s < ntaps; ++s) {
          // Montgomery form: the kernel's single reduction divides by R
          u64 v = mul_mod(residue_of_double(std::rint(weights[(size_t)co * ntaps + s] * (double)qlast), q),
                          P.primes[li].r_mod, q);
          for (int i = 0; i < 8; ++i) {
            ws[(((size_t)li * c_out + co) * ntaps + s) * 8 + i] = v;
            v = mul_mod(v, 256 % q, q);
          }
        }
    }
    if (conv_tc_supported(c, ntaps, c_out, level)) {
      const std::vector<uint8_t> img = conv_tc_weights(c, ntaps, c_out, level, ws);
      CK(cudaMalloc((void**)&wtc, img.size()));
      CK(cudaMemcpy(wtc, img.data(), img.size(), cudaMemcpyHostToDevice));
    }
    // limbs of primes < 2^40 (5-byte weight digits) pack rows as 3 maps x 5
    // planes (row 15 unused; conv_imma.cu MPT = 3), the others 2 maps x 8
    auto byte_at = [&](int li, int row, int col, int cp, int kb) -> uint32_t {
      const bool tri = conv_imma_triples(c, li, c_out);
      if (tri && row >= 15) return 0u;
      const int co = tri ? 3 * cp + row / 5 : 2 * cp + row / 8, e = tri ? row % 5 : row % 8;
      const int s = 4 * kb + col / 8, i = col % 8;
      if (co >= c_out || s >= ntaps) return 0u;
      return (uint32_t)((ws[(((size_t)li * c_out + co) * ntaps + s) * 8 + i] >> (8 * e)) & 0xFF);
    };
    std::vector<uint32_t> wa_h((size_t)level * cps * kbn * 32 * 4);
    for (int li = 0; li < level; ++li)
      for (int cp = 0; cp < cps; ++cp)
        for (int kb = 0; kb < kbn; ++kb)
          for (int lane = 0; lane < 32; ++lane) {
            const int r = lane / 4, c0 = 4 * (lane % 4);
            uint32_t reg[4] = {0, 0, 0, 0};
            const int rows[4] = {r, r + 8, r, r + 8}, cols[4] = {c0, c0, 16 + c0, 16 + c0};
            for (int q4 = 0; q4 < 4; ++q4)
              for (int bb = 0; bb < 4; ++bb) reg[q4] |= byte_at(li, rows[q4], cols[q4] + bb, cp, kb) << (8 * bb);
            uint32_t* dst = wa_h.data() + ((((size_t)li * cps + cp) * kbn + kb) * 32 + lane) * 4;
            for (int q4 = 0; q4 < 4; ++q4) dst[q4] = reg[q4];
          }
    CK(cudaMalloc((void**)&wa, wa_h.size() * 4));
    CK(cudaMemcpy(wa, wa_h.data(), wa_h.size() * 4, cudaMemcpyHostToDevice));
  }
  // bias[co] on the first w_used slots (convlower.cpp:68-71), at the product scale
  const int N = P.n;
  std::vector<u64> wire((size_t)c_out * level * N);
  std::vector<double> z(w_used);
  for (int co = 0; co < c_out; ++co) {
    std::fill(z.begin(), z.end(), bias_vals ? bias_vals[co] : 0.0);
    c.client->encode(z.data(), w_used, tap_scale * (double)qlast, level, false, wire.data() + (size_t)co * level * N);
  }
  CK(cudaMalloc((void**)&bias, wire.size() * 8));
  upload_mont(c, wire, bias, (size_t)c_out * level, level, -1);
}

void ConvLayer::make_merged(Context& c, const double* weights, const double* bias_vals, int w_used,
                            double tap_scale, int regs) {
  const int N = c.N(), S = c.S();
  const size_t F = (size_t)c_out * w_used;
  need((int64_t)regs * F <= S, HEGPU_ERR_CAPACITY, "merged conv: regions * c_out * d_out^2 exceeds the slots");
  regions = regs;
  const double qlast = (double)c.P->q(level - 1);
  std::vector<u64> wire((size_t)ntaps * level * N);
#pragma omp parallel for schedule(dynamic)
  for (int t = 0; t < ntaps; ++t) {
    // P_t: W[co][t] on block co of tap t's region
    const size_t off = (size_t)(t % regions) * F;
    std::vector<double> z(off + F, 0.0);
    for (int co = 0; co < c_out; ++co)
      std::fill_n(z.data() + off + (size_t)co * w_used, w_used, weights[(size_t)co * ntaps + t]);
    c.client->encode(z.data(), (int)z.size(), qlast, level, false, wire.data() + (size_t)t * level * N);
  }
  // the R taps of one tap ciphertext meet the same input limb, so their
  // plaintexts are summed once here (exact mod q; linear through the NTT):
  // the MAC runs G = ceil(ntaps / R) products per slot instead of ntaps
  const int G = (ntaps + regions - 1) / regions;
  std::vector<u64> gw((size_t)G * level * N, 0);
  for (int g = 0; g < G; ++g)
    for (int t = 0; t < level; ++t) {
      const u64 q = c.P->q(t);
      u64* dst = gw.data() + ((size_t)g * level + t) * N;
      for (int s = g * regions; s < std::min(ntaps, (g + 1) * regions); ++s) {
        const u64* src = wire.data() + ((size_t)s * level + t) * N;
        for (int k = 0; k < N; ++k) {
          const u64 v = dst[k] + src[k] % q;
          dst[k] = v >= q ? v - q : v;
        }
      }
    }
  CK(cudaMalloc((void**)&pw, gw.size() * 8));
  upload_mont(c, gw, pw, (size_t)G * level, level, -1);
  launch_split31(c, pw, gw.size());
  std::vector<double> zb((size_t)c_out * w_used);
  for (int co = 0; co < c_out; ++co)
    std::fill_n(zb.data() + (size_t)co * w_used, w_used, bias_vals ? bias_vals[co] : 0.0);
  std::vector<u64> bw((size_t)level * N);
  c.client->encode(zb.data(), (int)zb.size(), tap_scale * qlast, level, false, bw.data());
  CK(cudaMalloc((void**)&pbias, bw.size() * 8));
  u64d* stage = c.alloc(bw.size());
  CK(cudaMemcpyAsync(stage, bw.data(), bw.size() * 8, cudaMemcpyHostToDevice, c.stream));
  launch_wire_to_slot(c, stage, pbias, (size_t)level, 0, level, -1);  // standard form
  c.free(stage);
  CK(cudaStreamSynchronize(c.stream));
  merged = true;
}

MaskedConv::MaskedConv(Context& c, int ntaps_, int c_out_, const double* weights, const double* bias_vals,
                       int w_used, int level_, double tap_scale)
    : ntaps(ntaps_), c_out(c_out_), level(level_), ctx(&c) {
  const int N = c.N();
  need(w_used >= 0 && w_used <= c.S(), HEGPU_ERR_CAPACITY, "masked conv: w exceeds the slots");
  need(level >= 2 && level <= c.L(), HEGPU_ERR_CAPACITY, "masked conv: level must leave a prime to rescale");
  const double qlast = (double)c.P->q(level - 1);
  const size_t rows = (size_t)c_out * ntaps;
  std::vector<u64> wire(rows * level * N), bw((size_t)c_out * level * N);
#pragma omp parallel for schedule(dynamic)
  for (long r = 0; r < (long)rows; ++r) {
    std::vector<double> z(w_used, weights[r]);
    c.client->encode(z.data(), w_used, qlast, level, false, wire.data() + (size_t)r * level * N);
  }
#pragma omp parallel for schedule(dynamic)
  for (int co = 0; co < c_out; ++co) {
    std::vector<double> z(w_used, bias_vals ? bias_vals[co] : 0.0);
    c.client->encode(z.data(), w_used, tap_scale * qlast, level, false, bw.data() + (size_t)co * level * N);
  }
  CK(cudaMalloc((void**)&pw, wire.size() * 8));
  upload_mont(c, wire, pw, rows * level, level, -1);
  launch_split31(c, pw, wire.size());
  CK(cudaMalloc((void**)&pbias, bw.size() * 8));
  u64d* stage = c.alloc(bw.size());
  CK(cudaMemcpyAsync(stage, bw.data(), bw.size() * 8, cudaMemcpyHostToDevice, c.stream));
  launch_wire_to_slot(c, stage, pbias, (size_t)c_out * level, 0, level, -1);  // standard form
  c.free(stage);
  CK(cudaStreamSynchronize(c.stream));
}

MaskedConv::~MaskedConv() {
  cudaStreamSynchronize(ctx->stream);
  cudaFree(pw);
  cudaFree(pbias);
}

void MaskedConv::run(Context& c, const CtBatch& taps, CtBatch& maps) {
  const int B = taps.count / ntaps, N = c.N();
  u64d* prod = c.alloc((size_t)B * c_out * 2 * level * N);
  launch_conv_masked(c, taps.d, B, ntaps, c_out, level, pw, pbias, prod);
  CtBatch pb{&c, B * c_out, level, taps.scale * (double)c.P->q(level - 1), prod};
  eval_rescale(c, pb, maps);
  maps.scale = taps.scale;
  c.free(prod);
}

ConvLayer::~ConvLayer() {
  cudaStreamSynchronize(ctx->stream);
  cudaFree(pw);
  cudaFree(pbias);
  cudaFree(w);
  cudaFree(bias);
  cudaFree(wa);
  cudaFree(wtc);
}

#ifndef HEGPU_CONV_IMMA
#define HEGPU_CONV_IMMA 1  // conv MAC on the int8 tensor cores (conv_imma.cu)
#endif

void ConvLayer::mac(Context& c, const CtBatch& taps, CtBatch& prod) {
  const int B = taps.count / ntaps;
  if (merged) launch_conv_pt(c, taps.d, taps.count / cts_per_image(), ntaps, regions, level, pw, pbias, prod.d);
  else if (wtc) launch_conv_tc(c, taps.d, B, ntaps, level, wtc, c_out, bias, prod.d);
  else if (HEGPU_CONV_IMMA && conv_imma_supported(c))
    launch_conv_imma(c, taps.d, B, ntaps, level, wa, cps, kbn, c_out, bias, prod.d);
  else
    launch_conv_mac(c, taps.d, B, ntaps, level, w, c_out, bias, prod.d);
  prod.scale = taps.scale * (double)c.P->q(level - 1);
}

void ConvLayer::mac_compact(Context& c, const uint8_t* taps, int B, double tap_scale, CtBatch& prod) {
  // measured: expanding into full taps and streaming them through the MAC
  // beats decoding c0 / hashing c1 inside the register-heavy MAC kernel
  u64d* full = c.alloc((size_t)B * cts_per_image() * 2 * level * c.N());
  launch_expand_compact(c, taps, B * cts_per_image(), level, full);
  if (merged) launch_conv_pt(c, full, B, ntaps, regions, level, pw, pbias, prod.d);
  else if (wtc) launch_conv_tc(c, full, B, ntaps, level, wtc, c_out, bias, prod.d);
  else if (HEGPU_CONV_IMMA && conv_imma_supported(c))
    launch_conv_imma(c, full, B, ntaps, level, wa, cps, kbn, c_out, bias, prod.d);
  else
    launch_conv_mac(c, full, B, ntaps, level, w, c_out, bias, prod.d);
  c.free(full);
  prod.scale = tap_scale * (double)c.P->q(level - 1);
}

void ConvLayer::run(Context& c, const CtBatch& taps, CtBatch& maps) {
  const int B = taps.count / cts_per_image(), l = level, N = c.N(), mo = out_per_image();
  CtBatch prod{&c, B * mo, l, 0, c.alloc((size_t)B * mo * 2 * l * N)};
  mac(c, taps, prod);
  eval_rescale(c, prod, maps);
  maps.scale = taps.scale;
  c.free(prod.d);
}

// ----------------------------------------------------------------- merge ----
void merge_maps(Context& c, const CtBatch& maps, int nmaps, int64_t w, CtBatch& out) {
  const int S = c.S();
  const size_t st = maps.stride();
  out.scale = maps.scale;
  if (nmaps == 1) {
    CK(cudaMemcpyAsync(out.d, maps.d, (size_t)out.count * st * 8, cudaMemcpyDeviceToDevice, c.stream));
    return;
  }
  if (nmaps - 1 > HEGPU_MAX_BATCH_PERIOD) fail(HEGPU_ERR_CAPACITY, "merge_maps: too many maps");
  // all c-1 rotations in one batched key switch with a single ModDown
  KeyRowMap km{};
  km.period = nmaps - 1;
  for (int j = 1; j < nmaps; ++j) {
    const int shift = (int)((S - ((int64_t)j * w) % S) % S);
    km.shift[j - 1] = shift;
    km.key[j - 1] = c.rot_key(shift).data;
  }
  eval_merge(c, maps, nmaps, km, out);
}

// ---------------------------------------------------------------- square ----
void square_layer(Context& c, const CtBatch& a, CtBatch& out) {
  const int B = a.count, l = a.level;
  (void)B;
  eval_square_rescale(c, a, out);
  out.scale = a.scale * a.scale / (double)c.P->q(l - 1);
}

// -------------------------------------------------------------------- HS ----
void HsPlan::build(Context& c, const double* A, int m_, int n_, int lvl, bool skip_zero) {
  ctx = &c;
  m = m_;
  n = n_;
  level = lvl;
  const int S = c.S(), N = c.N();
  // proj/src/matvec.cpp:35-41, 48-53
  need(m >= 1 && n >= 1, HEGPU_ERR_SHAPE, "hs_matvec: empty matrix");
  need(m <= S && n <= S, HEGPU_ERR_CAPACITY,
       "matrix " + std::to_string(m) + "x" + std::to_string(n) + " exceeds " + std::to_string(S) + " slots");
  const bool plain = plain_branch_fits(m, n, S);
  m_eff = plain ? m : (int)next_pow2(m);
  need(m_eff <= S, HEGPU_ERR_CAPACITY,
       "padded row count " + std::to_string(m_eff) + " exceeds " + std::to_string(S) + " slots");
  folds = plain ? ceil_log2((m + n - 1 + m - 1) / m) : ceil_log2(S / m_eff);
  // generalized diagonals, pre-rotated: mask'_i = rot_right(mask_i, i)
  std::vector<std::vector<double>> kept;
  for (int i = 0; i < m_eff; ++i) {
    std::vector<double> mk(S, 0.0);
    bool nz = false;
    for (int j = 0; j < n; ++j) {
      const int row = (i + j) % m_eff;
      if (row < m) {
        const double v = A[(size_t)row * n + j];
        mk[(j + i) % S] = v;
        nz = nz || v != 0.0;
      }
    }
    if (skip_zero && !nz) continue;
    diag.push_back(HsDiag{i, i, (S - i) % S});
    kept.push_back(std::move(mk));
  }
  const int nl = level + 1;
  const double scale = (double)c.P->q(level - 1);
  std::vector<u64> wire(kept.size() * nl * (size_t)N);
#pragma omp parallel for schedule(dynamic)
  for (long i = 0; i < (long)kept.size(); ++i)
    c.client->encode(kept[i].data(), S, scale, level, true, wire.data() + (size_t)i * nl * N);
  if (!kept.empty()) {
    CK(cudaMalloc((void**)&masks, wire.size() * 8));
    upload_mont(c, wire, masks, kept.size() * nl, nl, level);
    launch_split31(c, masks, wire.size());
    CK(cudaStreamSynchronize(c.stream));
  }
  // right rotations (ascending) and chunks whose r span fits one smem window
  std::vector<int> r(diag.size()), chunk{0};
  for (size_t i = 0; i < diag.size(); ++i) {
    r[i] = (int)diag[i].right;
    if (i > 0 && r[i] - r[chunk.back()] >= hs_chunk_span()) chunk.push_back((int)i);
  }
  chunk.push_back((int)diag.size());
  if (diag.empty()) chunk = {0};
  nchunk = (int)chunk.size() - 1;
  CK(cudaMalloc((void**)&d_r, (r.size() + 1) * sizeof(int)));
  if (!r.empty()) CK(cudaMemcpy(d_r, r.data(), r.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMalloc((void**)&d_chunk, chunk.size() * sizeof(int)));
  CK(cudaMemcpy(d_chunk, chunk.data(), chunk.size() * sizeof(int), cudaMemcpyHostToDevice));
  h_chunk = chunk;
}

void HsPlan::release() {
  if (ctx) cudaStreamSynchronize(ctx->stream);
  for (auto& f : fold) f->release();
  fold.clear();
  cudaFree(masks);
  cudaFree(d_r);
  cudaFree(d_chunk);
  for (auto& e : sub_chunks) cudaFree(e.second.first);
  sub_chunks.clear();
  cudaFree(fkeys);
  for (HsImmaChunk& ch : imma) cudaFree(ch.wt);
  imma.clear();
  for (TcChunk& ch : tc) cudaFree(ch.at);
  tc.clear();
  cudaFree(tc_ce);
  cudaFree(tc_pR);
  tc_ce = tc_pR = nullptr;
  tc_built = false;
  cudaFree(imma_ec);
  cudaFree(imma_pmod);
  cudaFree(d_rdiag);
  imma_ec = imma_pmod = nullptr;
  d_rdiag = nullptr;
  imma_built = false;
  masks = nullptr;
  d_r = d_chunk = nullptr;
  fkeys = nullptr;
}

// the fold's doublings in ceil(folds / 5) groups of near-equal size, larger
// first: a group of a doublings is one hoisted sum of 2^a - 1 key inner
// products, so 7 doublings cost 15 + 7 inner products and two ModUp /
// ModDown pairs instead of 127 (the config-1 m = 64, n = 4096 point);
// oracle/ckks_pipeline.fold_groups mirrors it
std::vector<int> HsPlan::fold_groups() const {
  std::vector<int> g;
  if (folds <= 0) return g;
  const int n = (folds + kMaxFoldGroup - 1) / kMaxFoldGroup;
  for (int i = 0; i < n; ++i) g.push_back(folds / n + (i < folds % n ? 1 : 0));
  return g;
}

std::vector<int64_t> HsPlan::fold_rights(int offset, int size) const {
  // s += rot_left(s, m_eff 2^t) for t = folds-1..0 sums rot_left(s, m_eff u)
  // over u < 2^folds (distinct: m_eff 2^folds <= S in both branches); the
  // group of `size` doublings from `offset` sums rot_left(s, m_eff 2^offset u)
  const int64_t S = ctx->S(), step = (int64_t)m_eff << offset;
  std::vector<int64_t> r;
  for (int64_t u = 0; u < (int64_t{1} << size); ++u) r.push_back((S - (step * u) % S) % S);
  std::sort(r.begin(), r.end());
  return r;
}

std::vector<int64_t> HsPlan::right_rotations() const {
  std::vector<int64_t> r;
  for (const HsDiag& d : diag)
    if (d.right) r.push_back(d.right);
  int off = 0;
  for (int a : fold_groups()) {
    for (int64_t f : fold_rights(off, a))
      if (f) r.push_back(f);  // the fold's hoisted rotations
    off += a;
  }
  return r;
}

void HsPlan::build_rotsum(Context& c, const std::vector<int64_t>& rights, int lvl) {
  ctx = &c;
  level = lvl;
  m = n = m_eff = 0;
  folds = 0;
  unit_masks = true;
  const int S = c.S(), N = c.N(), nl = level + 1;
  for (int64_t r : rights) diag.push_back(HsDiag{(int)diag.size(), r, (int)((S - r) % S)});
  // unit masks: Montgomery 1 = 2^64 mod q per limb (limb `level` is P), split-31
  std::vector<u64> mk(diag.size() * (size_t)nl * N);
  for (int t = 0; t < nl; ++t) {
    const u64 q = c.P->q(t == level ? c.L() : t);
    const u64 one = (u64)(((u128)1 << 64) % q);
    const u64 sp = (one & 0x7FFFFFFFull) | ((one >> 31) << 32);
    for (size_t i = 0; i < diag.size(); ++i) std::fill_n(mk.data() + (i * nl + t) * N, N, sp);
  }
  CK(cudaMalloc((void**)&masks, mk.size() * 8));
  CK(cudaMemcpy(masks, mk.data(), mk.size() * 8, cudaMemcpyHostToDevice));
  std::vector<int> r(diag.size()), chunk{0};
  for (size_t i = 0; i < diag.size(); ++i) {
    r[i] = (int)diag[i].right;
    if (i > 0 && r[i] - r[chunk.back()] >= hs_chunk_span()) chunk.push_back((int)i);
  }
  chunk.push_back((int)diag.size());
  nchunk = (int)chunk.size() - 1;
  CK(cudaMalloc((void**)&d_r, (r.size() + 1) * sizeof(int)));
  CK(cudaMemcpy(d_r, r.data(), r.size() * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMalloc((void**)&d_chunk, chunk.size() * sizeof(int)));
  CK(cudaMemcpy(d_chunk, chunk.data(), chunk.size() * sizeof(int), cudaMemcpyHostToDevice));
  h_chunk = chunk;
}

void HsPlan::ensure_keys(Context& c) {
  if (keys_resolved) return;
  const int l = level, N = c.N(), S = c.S();
  // fuse each diagonal's Galois key with its mask once (offline work):
  // fk_i[j][p][t] = key_i[j][p][t] * mask'_i[t] over the level-l ext basis
  for (int t = folds - 1; t >= 0; --t) c.rot_key((int)(((int64_t)m_eff << t) % S));
  const size_t fk_words = (size_t)l * 2 * (l + 1) * N;
  size_t nkeyed = 0;
  for (const HsDiag& d : diag) nkeyed += d.shift != 0;
  if (nkeyed) CK(cudaMalloc((void**)&fkeys, nkeyed * fk_words * 8));
  size_t slot = 0;  // only diagonal 0 can be unkeyed (r ascending)
  for (size_t i = 0; i < diag.size(); ++i) {
    if (!diag[i].shift) continue;
    launch_fuse_key(c, c.rot_key(diag[i].shift).data, masks + i * (size_t)(l + 1) * N, l,
                    fkeys + slot++ * fk_words);
  }
  CK(cudaStreamSynchronize(c.stream));
  keys_resolved = true;
}

// HEGPU_HS_IMMA=0 keeps the integer-pipe kernel for every batch
static int hs_imma_min_batch() {
  static int mb = -1;
  if (mb < 0) {
    const char* e = getenv("HEGPU_HS_IMMA");
    mb = e && atoi(e) == 0 ? 1 << 30 : 8;
    if (e && atoi(e) > 1) mb = atoi(e);  // HEGPU_HS_IMMA=<min batch>
  }
  return mb;
}

// narrow diagonal bands (e.g. a 10-row output layer) stay on the integer
// kernel: the MMA band is too short to amortise the window staging and the
// byte-plane epilogue (HEGPU_HS_IMMA_MINSPAN, default 32 rotations)
static int hs_imma_min_span() {
  static int ms = -1;
  if (ms < 0) {
    const char* e = getenv("HEGPU_HS_IMMA_MINSPAN");
    ms = e ? atoi(e) : 32;
  }
  return ms;
}

bool HsPlan::use_imma(Context& c, int B, int i_lo, int i_hi) const {
  if (diag.empty()) return false;
  const int64_t span = diag.back().right - diag.front().right + 1;
  // dense bands only: the fragments cover the whole rotation span (a sparse
  // band -- e.g. a convolution's matrix -- would store mostly zero tiles)
  // the tcgen05 kernel is instantiated up to level 8 (J = l + 1 <= 9), the mma.sync one up to 6
  const bool level_ok = hs_imma_supported(c, level) ||
                        (hs_tc_enabled() && level >= 1 && level <= kHsTcMaxLevel && hs_imma_supported(c, 6));
  return B >= hs_imma_min_batch() && i_lo == 0 && i_hi == (int)diag.size() && span >= hs_imma_min_span() &&
         4 * (int64_t)diag.size() >= span && level_ok;
}

// shared by the mma.sync and tcgen05 paths: epilogue constants, P mod q_t,
// and the right rotation -> kept diagonal map
void HsPlan::ensure_imma_consts(Context& c) {
  if (d_rdiag) return;
  ensure_keys(c);
  const int l = level, S = c.S(), np = c.P->np();
  // epilogue constants 2^(24 g + 32 h) mod q with Shoup companions
  std::vector<u64> ec((size_t)np * 16);
  for (int pi = 0; pi < np; ++pi) {
    const u64 q = c.P->q(pi);
    for (int h = 0; h < 2; ++h)
      for (int g = 0; g < 4; ++g) {
        u128 w = 1;
        for (int e = 0; e < 24 * g + 32 * h; ++e) w = (w * 2) % q;
        ec[((size_t)pi * 2 + h) * 8 + 2 * g] = (u64)w;
        ec[((size_t)pi * 2 + h) * 8 + 2 * g + 1] = (u64)((w << 64) / q);
      }
  }
  std::vector<u64> pm(l);
  for (int t = 0; t < l; ++t) pm[t] = c.P->q(c.L()) % c.P->q(t);
  std::vector<int> rd(S, -1);
  for (size_t i = 0; i < diag.size(); ++i) rd[diag[i].right] = (int)i;
  CK(cudaMalloc((void**)&imma_ec, ec.size() * 8));
  CK(cudaMemcpy(imma_ec, ec.data(), ec.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc((void**)&imma_pmod, pm.size() * 8));
  CK(cudaMemcpy(imma_pmod, pm.data(), pm.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc((void**)&d_rdiag, rd.size() * sizeof(int)));
  CK(cudaMemcpy(d_rdiag, rd.data(), rd.size() * sizeof(int), cudaMemcpyHostToDevice));
}

void HsPlan::ensure_imma(Context& c) {
  if (imma_built) return;
  ensure_imma_consts(c);
  const int l = level, N = c.N(), J = l + 1;
  // chunks of kept diagonals whose r span fits the kernel's window ring
  // balanced: nchunk = ceil(r span / max span) chunks of about equal r span
  const int smax = hs_imma_chunk_span(l), rtot = (int)(diag.back().right - diag[0].right) + 1;
  const int nch = (rtot + smax - 1) / smax, span = (rtot + nch - 1) / nch;
  const int first_keyed = diag[0].shift == 0 ? 1 : 0;
  HsDiagTable tab{(int)diag.size(), 0, d_r, fkeys, (size_t)l * 2 * (l + 1) * N, first_keyed, 1, masks, 0, nullptr};
  size_t i = 0;
  while (i < diag.size()) {
    HsImmaChunk ch{};
    ch.r_lo = (int)diag[i].right;
    ch.r_hi = ch.r_lo;
    while (i < diag.size() && diag[i].right - ch.r_lo < span) {
      ch.r_hi = (int)diag[i].right;
      ch.keyed += diag[i].shift != 0;
      ++ch.ndiag;
      ++i;
    }
    // steps per 4-position group: ceil((span J + 31) / 32) + 1 (hs_imma.cu)
    ch.ns = ((ch.r_hi - ch.r_lo + 1) * J + 62) / 32 + 1;
    CK(cudaMalloc((void**)&ch.wt, hs_imma_tile_words(c, l, ch) * 8));
    launch_hs_imma_tiles(c, l, tab, imma_pmod, d_rdiag, ch, ch.wt);
    imma.push_back(ch);
  }
  CK(cudaStreamSynchronize(c.stream));
  imma_built = true;
}

// the tcgen05 A tables: chunks of kept diagonals whose r span fits the
// window ring (hs_tc_chunk_span), balanced like the mma.sync chunks
bool HsPlan::ensure_tc(Context& c) {
  if (tc_built) return true;
  if (tc_unfit) return false;
  const int l = level, N = c.N(), np = c.P->np();
  {  // the A tables are as large again as the fused keys: build them only if they fit
    const int smax0 = hs_tc_chunk_span(l), rtot0 = (int)(diag.back().right - diag[0].right) + 1;
    const int nch0 = (rtot0 + smax0 - 1) / smax0, span0 = (rtot0 + nch0 - 1) / nch0;
    const size_t need_bytes = (size_t)nch0 * hs_tc_table_bytes(c, l, span0);
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    if (need_bytes + (total_b >> 3) > free_b) {  // keep 1/8 of the device for the working set
      tc_unfit = true;
      return false;
    }
  }
  ensure_imma_consts(c);  // rdiag
  std::vector<u64> ce((size_t)np * 8);
  for (int pi = 0; pi < np; ++pi) {
    const u64 q = c.P->q(pi);
    u128 w = ((u128)1 << 64) % q;  // R mod q
    for (int e = 0; e < 8; ++e) {
      ce[(size_t)pi * 8 + e] = (u64)w;
      w = (w << 8) % q;
    }
  }
  std::vector<u64> pr(l);
  for (int t = 0; t < l; ++t) {
    const u64 q = c.P->q(t);
    pr[t] = (u64)(((u128)(c.P->q(c.L()) % q) << 64) % q);  // P R mod q_t
  }
  CK(cudaMalloc((void**)&tc_ce, ce.size() * 8));
  CK(cudaMemcpy(tc_ce, ce.data(), ce.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMalloc((void**)&tc_pR, pr.size() * 8));
  CK(cudaMemcpy(tc_pR, pr.data(), pr.size() * 8, cudaMemcpyHostToDevice));
  const int smax = hs_tc_chunk_span(l), rtot = (int)(diag.back().right - diag[0].right) + 1;
  const int nch = (rtot + smax - 1) / smax, span = (rtot + nch - 1) / nch;
  const int first_keyed = diag[0].shift == 0 ? 1 : 0;
  HsDiagTable tab{(int)diag.size(), 0, d_r, fkeys, (size_t)l * 2 * (l + 1) * N, first_keyed, 1, masks, 0, nullptr};
  size_t i = 0;
  while (i < diag.size()) {
    TcChunk ch{};
    ch.r_lo = (int)diag[i].right;
    ch.r_hi = ch.r_lo;
    while (i < diag.size() && diag[i].right - ch.r_lo < span) {
      ch.r_hi = (int)diag[i].right;
      ch.keyed += diag[i].shift != 0;
      ++ch.ndiag;
      ++i;
    }
    CK(cudaMalloc((void**)&ch.at, hs_tc_table_bytes(c, l, ch.r_hi - ch.r_lo + 1)));
    launch_hs_tc_tiles(c, l, tab, tc_pR, d_rdiag, ch.r_lo, ch.r_hi, ch.at);
    tc.push_back(ch);
  }
  CK(cudaStreamSynchronize(c.stream));
  tc_built = true;
  return true;
}

void HsPlan::accumulate(Context& c, const CtBatch& v, int i_lo, int i_hi, u64d* acc, u64d* cacc) {
  const int B = v.count, l = level, N = c.N();
  ensure_keys(c);
  for (int i = i_lo; i < i_hi; ++i) c.ks[KS_INNER] += diag[i].shift != 0 ? B : 0;
  if (use_imma(c, B, i_lo, i_hi) && hs_tc_enabled() && l <= kHsTcMaxLevel && ensure_tc(c)) {
    u64d* tmp = c.alloc((size_t)B * l * N);
    u64d* D = c.alloc((size_t)B * l * (l + 1) * N);
    ks_modup(c, v.d + (size_t)l * N, (long)v.stride(), B, l, nullptr, tmp, D);
    for (size_t ci = 0; ci < tc.size(); ++ci)
      launch_hs_tc(c, v.d, B, l, D, tc[ci].r_lo, tc[ci].r_hi, tc[ci].at, tc_ce, ci > 0, acc, tc[ci].keyed,
                   tc[ci].ndiag);
    launch_hs_cacc(c, v.d, masks, B, l, diag[0].right == 0 ? 1 : 0, cacc);
    c.free(tmp);
    c.free(D);
    return;
  }
  if (use_imma(c, B, i_lo, i_hi) && hs_imma_supported(c, level)) {
    ensure_imma(c);
    u64d* tmp = c.alloc((size_t)B * l * N);
    u64d* D = c.alloc((size_t)B * l * (l + 1) * N);
    ks_modup(c, v.d + (size_t)l * N, (long)v.stride(), B, l, nullptr, tmp, D);
    for (size_t ci = 0; ci < imma.size(); ++ci) launch_hs_imma(c, v.d, B, l, D, imma[ci], imma_ec, ci > 0, acc);
    launch_hs_cacc(c, v.d, masks, B, l, diag[0].right == 0 ? 1 : 0, cacc);
    c.free(tmp);
    c.free(D);
    return;
  }
  // the plan's chunks clipped to [i_lo, i_hi) (cached per range)
  const int* chunks = d_chunk;
  int nch = nchunk;
  if (i_lo != 0 || i_hi != (int)diag.size()) {
    auto key = std::make_pair(i_lo, i_hi);
    auto it = sub_chunks.find(key);
    if (it == sub_chunks.end()) {
      std::vector<int> sc{i_lo};
      for (int b : h_chunk)
        if (b > i_lo && b < i_hi) sc.push_back(b);
      if (i_hi > i_lo) sc.push_back(i_hi);
      int* d = nullptr;
      CK(cudaMalloc((void**)&d, sc.size() * sizeof(int)));
      CK(cudaMemcpy(d, sc.data(), sc.size() * sizeof(int), cudaMemcpyHostToDevice));
      it = sub_chunks.emplace(key, std::make_pair(d, (int)sc.size() - 1)).first;
    }
    chunks = it->second.first;
    nch = it->second.second;
  }
  u64d* tmp = c.alloc((size_t)B * l * N);
  u64d* D = c.alloc((size_t)B * l * (l + 1) * N);
  // (1) one ModUp of v.c1 for all diagonals (hoisting)
  ks_modup(c, v.d + (size_t)l * N, (long)v.stride(), B, l, nullptr, tmp, D);
  // (2) diagonal accumulation in the extended basis
  int keyed = 0;
  for (int i = i_lo; i < i_hi; ++i) keyed += diag[i].shift != 0;
  const int first_keyed = !diag.empty() && diag[0].shift == 0 ? 1 : 0;
  if (nch > 0 && i_hi > i_lo) {
    HsDiagTable tab{i_hi - i_lo, keyed, d_r, fkeys, (size_t)l * 2 * (l + 1) * N, first_keyed, i_lo == 0 ? 1 : 0,
                    masks, nch, chunks, unit_masks ? 1 : 0};
    launch_hs_diag(c, v.d, B, l, D, tab, acc, cacc);
  } else {
    CK(cudaMemsetAsync(acc, 0, (size_t)B * 2 * (l + 1) * N * 8, c.stream));
    CK(cudaMemsetAsync(cacc, 0, (size_t)B * 2 * l * N * 8, c.stream));
  }
  c.free(tmp);
  c.free(D);
}

void HsPlan::finish(Context& c, int B, double v_scale, u64d* acc, u64d* cacc, int nparts, CtBatch& out) {
  const int l = level, N = c.N(), S = c.S();
  if (nparts > 1) {  // sums of nparts reduced residues
    launch_reduce_rows(c, acc, (size_t)B * 2 * (l + 1) * N, l + 1, l);
    launch_reduce_rows(c, cacc, (size_t)B * 2 * l * N, l, -1);
  }
  u64d* tmpP = c.alloc((size_t)B * 2 * N);
  // (3) one ModDown of the sum (+ the Q-basis c-part) and (4) the rescale by
  // q_{l-1} (the masks were encoded at exactly that scale), fused into one
  // drop pass (ntt.cu §4.8; residues equal to ModDown followed by rescale)
  DropArgs d{};
  d.src = acc; d.src_b = 2L * (l + 1) * N; d.src_p = (long)(l + 1) * N; d.src_limbs = l + 1;
  d.dst = out.d; d.dst_b = (long)out.stride(); d.dst_p = (long)(l - 1) * N;
  d.pd = c.L(); d.nl = l - 1;
  d.add = cacc; d.add_b = 2L * l * N; d.add_p = (long)l * N; d.add_mask = 3; d.shifts = nullptr;
  d.fuse_rescale = 1;
  drop_last_limb(c, B, d, tmpP);
  out.scale = v_scale;
  // (5) log-depth fold, matvec.cpp:101-103: s += rot_left(s, m_eff * 2^t)
  // for t = folds-1..0 = sum of rot_left(s, m_eff u) over u < 2^folds, run
  // as hoisted rotation sums, one per group of <= 5 doublings (one ModUp of
  // s.c1, the 2^a - 1 key inner products on the rotated digits, one
  // ModDown) instead of `folds` serial key switches; metered as the
  // reference's folds (capi.cu)
  const std::vector<int> groups = fold_groups();
  if (fold.empty()) {
    int off = 0;
    for (int a : groups) {
      fold.push_back(std::make_unique<HsPlan>());
      fold.back()->build_rotsum(c, fold_rights(off, a), l - 1);
      off += a;
    }
  }
  for (auto& fp : fold) {
    const int lf = l - 1;
    u64d* facc = c.alloc((size_t)B * 2 * (lf + 1) * N);
    u64d* fcacc = c.alloc((size_t)B * 2 * lf * N);
    fp->accumulate(c, out, 0, (int)fp->diag.size(), facc, fcacc);
    CtBatch r{&c, B, lf, out.scale, c.alloc((size_t)B * 2 * lf * N)};
    DropArgs f{};
    f.src = facc; f.src_b = 2L * (lf + 1) * N; f.src_p = (long)(lf + 1) * N; f.src_limbs = lf + 1;
    f.dst = r.d; f.dst_b = (long)r.stride(); f.dst_p = (long)lf * N;
    f.pd = c.L(); f.nl = lf;
    f.add = fcacc; f.add_b = 2L * lf * N; f.add_p = (long)lf * N; f.add_mask = 3; f.shifts = nullptr;
    drop_last_limb(c, B, f, tmpP);
    CK(cudaMemcpyAsync(out.d, r.d, out.words() * 8, cudaMemcpyDeviceToDevice, c.stream));
    c.free(facc);
    c.free(fcacc);
    c.free(r.d);
  }
  c.free(tmpP);
}

void HsPlan::run(Context& c, const CtBatch& v, CtBatch& out) {
  const int B = v.count, l = level, N = c.N();
  u64d* acc = c.alloc((size_t)B * 2 * (l + 1) * N);
  u64d* cacc = c.alloc((size_t)B * 2 * l * N);
  accumulate(c, v, 0, (int)diag.size(), acc, cacc);
  finish(c, B, v.scale, acc, cacc, 1, out);
  c.free(acc);
  c.free(cacc);
}

}  // namespace hegpu
