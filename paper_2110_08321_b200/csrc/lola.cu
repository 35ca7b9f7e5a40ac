// lola.cu -- the LoLa comparators of the reference on the CKKS engine:
//   LolaPlan kind 0: lola_dense_matvec    proj/src/matvec.cpp:107-123
//   LolaPlan kind 1: lola_stacked_matvec  proj/src/matvec.cpp:125-166
// Each row product is one plaintext multiply (rows encoded at scale q_{l-1},
// rescaled), rotate_and_sum (proj/src/matvec.cpp:67-80) is log2(next_pow2 n)
// rotate-left + add steps batched over every product of the call, and the
// value-level clearing of the reference (masked_prefix(1) / keeping the
// segment starts) is a 0/1 mask multiply + rescale, so the decrypted slots
// equal the reference's slot vector (two levels consumed; the mask
// multiplies are free in the reference and are not metered).
#include <string>

#include "layers.hpp"

namespace hegpu {

namespace {

void need(bool ok, int code, const std::string& msg) {
  if (!ok) fail(code, msg);
}

int ceil_log2(int64_t x) {
  int b = 0;
  while ((int64_t{1} << b) < x) ++b;
  return b;
}

// out[c] = a[c / a_div] * p[c % p_mod]  (ciphertext x Montgomery plaintext)
__global__ void k_mul_plain_idx(PrimeTable pt, const u64d* __restrict__ a, int a_div, const u64d* __restrict__ p,
                                int p_mod, u64d* __restrict__ out, size_t total, int l, int N) {
  const size_t per = (size_t)2 * l * N, ln = (size_t)l * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const size_t c = i / per, r = i % per, lk = r % ln;
    const DevPrime pr = pt.p[lk / N];
    out[i] = mont_mul(a[(c / a_div) * per + r], p[(c % p_mod) * ln + lk], pr.q, pr.qneg_inv);
  }
}

void mul_plain_idx(Context& c, const u64d* a, int a_div, const u64d* p, int p_mod, u64d* out, int count, int l) {
  const size_t total = (size_t)count * 2 * l * c.N();
  unsigned g = (unsigned)((total + 255) / 256);
  if (g > 148 * 16) g = 148 * 16;
  LAUNCH_B(c, "k_mul_plain", 16.0 * total + 8.0 * (size_t)p_mod * l * c.N(),
           k_mul_plain_idx<<<g, 256, 0, c.stream>>>(c.primes, a, a_div, p, p_mod, out, total, l, c.N()));
}

// host slot vectors -> encoded Montgomery slot-order plaintext rows
u64d* encode_rows(Context& c, const std::vector<std::vector<double>>& rows, int level, double scale) {
  const int N = c.N(), S = c.S();
  std::vector<u64> wire(rows.size() * (size_t)level * N);
#pragma omp parallel for schedule(dynamic)
  for (long i = 0; i < (long)rows.size(); ++i)
    c.client->encode(rows[i].data(), S, scale, level, false, wire.data() + (size_t)i * level * N);
  u64d* d = nullptr;
  CK(cudaMalloc((void**)&d, wire.size() * 8));
  u64d* stage = c.alloc(wire.size());
  CK(cudaMemcpyAsync(stage, wire.data(), wire.size() * 8, cudaMemcpyHostToDevice, c.stream));
  launch_wire_to_slot(c, stage, d, rows.size() * level, 1, level, -1);
  c.free(stage);
  CK(cudaStreamSynchronize(c.stream));
  return d;
}

KeyRowMap one_key(Context& c, int left) {
  KeyRowMap km{};
  km.period = 1;
  km.shift[0] = left;
  km.key[0] = c.rot_key(left).data;
  return km;
}

}  // namespace

void LolaPlan::build(Context& c, int kind_, const double* A, int m_, int n_, int lvl) {
  ctx = &c;
  kind = kind_;
  m = m_;
  n = n_;
  level = lvl;
  const int S = c.S();
  // proj/src/matvec.cpp:35-41 (check_dims), :132-135
  need(m >= 1 && n >= 1, HEGPU_ERR_SHAPE, "lola: empty matrix");
  need(m <= S && n <= S, HEGPU_ERR_CAPACITY,
       "matrix " + std::to_string(m) + "x" + std::to_string(n) + " exceeds " + std::to_string(S) + " slots");
  need(level >= 3 && level <= c.L(), HEGPU_ERR_ARG, "lola: level must leave two primes (product + clearing rescale)");
  delta = 1;
  while (delta < n) delta <<= 1;
  folds = ceil_log2(delta);
  if (kind == 1) {
    need(delta <= S, HEGPU_ERR_CAPACITY,
         "stacked: padded width " + std::to_string(delta) + " exceeds " + std::to_string(S) + " slots");
    k = S / delta;
    batches = (m + k - 1) / k;
  } else {
    k = 1;
    batches = m;
  }
  // product plaintexts: dense row i packed at slots [0, n); stacked batch b
  // holds rows b k + j on [j delta, j delta + n)
  std::vector<std::vector<double>> prow(batches, std::vector<double>(S, 0.0));
  std::vector<std::vector<double>> clean(kind == 1 ? batches : 1, std::vector<double>(S, 0.0));
  for (int b = 0; b < batches; ++b)
    for (int j = 0; j < k; ++j) {
      const int row = b * k + j;
      if (row >= m) break;
      for (int x = 0; x < n; ++x) prow[b][(size_t)j * delta + x] = A[(size_t)row * n + x];
      if (kind == 1) clean[b][(size_t)j * delta] = 1.0;
    }
  if (kind == 0) clean[0][0] = 1.0;
  rows = encode_rows(c, prow, level, (double)c.P->q(level - 1));
  masks = encode_rows(c, clean, level - 1, (double)c.P->q(level - 2));
}

void LolaPlan::release() {
  if (ctx) cudaStreamSynchronize(ctx->stream);
  cudaFree(rows);
  cudaFree(masks);
  rows = masks = nullptr;
}

std::vector<int64_t> LolaPlan::right_rotations() const {
  const int S = ctx->S();
  std::vector<int64_t> r;
  if (kind == 1)
    for (int j = 1; j < k; ++j) r.push_back((int64_t)j * delta);
  for (int t = folds - 1; t >= 0; --t) r.push_back((S - (1 << t)) % S);  // rotate_left(1 << t)
  if (kind == 1)
    for (int b = 1; b < batches; ++b) r.push_back(b);
  return r;
}

int LolaPlan::out_count(int B) const { return kind == 0 ? B * m : B; }

int64_t LolaPlan::slot_of_row(int i) const {
  return kind == 0 ? 0 : (int64_t)(i % k) * delta + i / k;  // proj/src/matvec.cpp:158
}

void LolaPlan::run(Context& c, const CtBatch& v, CtBatch& out) {
  const int B = v.count, l = level, N = c.N(), S = c.S();
  const size_t ct1 = (size_t)2 * (l - 1) * N, ct2 = (size_t)2 * (l - 2) * N;
  const int P = B * batches;  // products (dense: rows, stacked: batches) per call
  // (1) the multiplicand: v, or the stacked copies sum_j rot_right(v, j delta)
  const u64d* src = v.d;
  u64d* stacked = nullptr;
  if (kind == 1 && k > 1) {
    stacked = c.alloc(v.words());
    u64d* r = c.alloc(v.words());
    CK(cudaMemcpyAsync(stacked, v.d, v.words() * 8, cudaMemcpyDeviceToDevice, c.stream));
    for (int j = 1; j < k; ++j) {
      eval_rotate(c, v.d, (long)v.stride(), B, l, one_key(c, S - j * delta), r, (long)v.stride());
      launch_add(c, stacked, r, stacked, B, l);
    }
    c.free(r);
    src = stacked;
  }
  // (2) products with the row plaintexts, rescaled to level l - 1
  CtBatch prod{&c, P, l, v.scale * (double)c.P->q(l - 1), c.alloc((size_t)P * 2 * l * N)};
  mul_plain_idx(c, src, batches, rows, batches, prod.d, P, l);
  CtBatch u{&c, P, l - 1, v.scale, c.alloc((size_t)P * ct1)};
  eval_rescale(c, prod, u);
  c.free(prod.d);
  if (stacked) c.free(stacked);
  // (3) rotate_and_sum(delta, 1): s += rot_left(s, 2^t), t = folds-1 .. 0
  if (folds > 0) {
    u64d* r = c.alloc((size_t)P * ct1);
    for (int t = folds - 1; t >= 0; --t) {
      eval_rotate(c, u.d, (long)ct1, P, l - 1, one_key(c, 1 << t), r, (long)ct1);
      launch_add(c, u.d, r, u.d, P, l - 1);
    }
    c.free(r);
  }
  // (4) value-level clearing as a 0/1 mask multiply + rescale -> level l - 2
  CtBatch w{&c, P, l - 1, v.scale * (double)c.P->q(l - 2), c.alloc((size_t)P * ct1)};
  mul_plain_idx(c, u.d, 1, masks, kind == 1 ? batches : 1, w.d, P, l - 1);
  c.free(u.d);
  if (kind == 0) {
    eval_rescale(c, w, out);  // out[b m + i]
    out.scale = v.scale;
    c.free(w.d);
    return;
  }
  CtBatch y{&c, P, l - 2, v.scale, c.alloc((size_t)P * ct2)};
  eval_rescale(c, w, y);
  c.free(w.d);
  // (5) res = batch_0 + sum_b rot_right(batch_b, b)
  for (int b0 = 0; b0 < B; ++b0)
    CK(cudaMemcpyAsync(out.d + (size_t)b0 * ct2, y.d + (size_t)b0 * batches * ct2, ct2 * 8,
                       cudaMemcpyDeviceToDevice, c.stream));
  if (batches > 1) {
    u64d* r = c.alloc((size_t)B * ct2);
    for (int b = 1; b < batches; ++b) {
      eval_rotate(c, y.d + (size_t)b * ct2, (long)(batches * ct2), B, l - 2, one_key(c, S - b), r, (long)ct2);
      launch_add(c, out.d, r, out.d, B, l - 2);
    }
    c.free(r);
  }
  out.scale = v.scale;
  c.free(y.d);
}

}  // namespace hegpu
