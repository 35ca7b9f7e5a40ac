// hegpu.hpp -- header-only C++ facade over the hegpu C-ABI that restores the
// reference's `hesim::` value-semantics API (RAII handles, exceptions,
// argument order `op(inputs..., ctx)`), so hesim call sites port by changing
// the namespace:
//
//   hesim (reference)                                   hegpu (this facade)
//   SlotVector pack(values, N, Kind::Ciphertext)         Ciphertext encrypt(values, level, nonce, ctx)
//   rotate_right(v, r, ctx)  slotvec.cpp:42-57          rotate_right(v, r, ctx)
//   rotate_left(v, r, ctx)   slotvec.cpp:59-66          rotate_left(v, r, ctx)
//   add(a, b, ctx)           slotvec.cpp:97-102         add(a, b, ctx) / add(a, pt, ctx)
//   mul(a, pt, ctx)          slotvec.cpp:104-109        mul(a, pt, ctx)
//   square_layer(v, ctx)     convlower.cpp:141-143      square_layer(v, ctx)   (+ relin + rescale)
//   merge_maps(maps, w, ctx) convlower.cpp:145-160      merge_maps(maps, c, w, ctx)
//   conv_packed_forward(taps, filters, shape, ctx)      conv_packed_forward(taps, filters, ctx)
//   hs_matvec(A, v, ctx)     matvec.cpp:82-105          hs_matvec(HsPlan(A, level, ctx), v, ctx)
//   MeterContext / OpTally   meter.hpp:12-70            Context::tally(), Context::stages()
//   CapacityError / ShapeError / LayoutError / IoError  same names; std::out_of_range for RANGE
//
// Ciphertexts are batches (count >= 1) living in device memory; every op
// allocates a fresh result (inputs are never mutated).
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "hegpu.h"

namespace hegpu {

struct CapacityError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ShapeError : std::runtime_error { using std::runtime_error::runtime_error; };
struct LayoutError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct KeyError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void throw_status(int rc, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (rc) {
    case HEGPU_OK: return;
    case HEGPU_ERR_CAPACITY: throw CapacityError(m);
    case HEGPU_ERR_SHAPE: throw ShapeError(m);
    case HEGPU_ERR_LAYOUT: throw LayoutError(m);
    case HEGPU_ERR_RANGE: throw std::out_of_range(m);
    case HEGPU_ERR_IO: throw IoError(m);
    case HEGPU_ERR_KEY: throw KeyError(m);
    case HEGPU_ERR_CUDA:
    case HEGPU_ERR_NCCL: throw DeviceError(m);
    default: throw std::invalid_argument(m);
  }
}

// proj/include/hesim/meter.hpp:12-31
struct OpTally {
  int64_t add_pc = 0, add_cc = 0, mul_pc = 0, mul_cc = 0, rot = 0;
  int64_t total() const { return add_pc + add_cc + mul_pc + mul_cc + rot; }
  friend bool operator==(const OpTally& a, const OpTally& b) {
    return a.add_pc == b.add_pc && a.add_cc == b.add_cc && a.mul_pc == b.mul_pc && a.mul_cc == b.mul_cc &&
           a.rot == b.rot;
  }
};

class Context {
 public:
  Context(int log_n, const std::vector<int>& q_bits, int p_bits, uint64_t seed, int device = 0) {
    hegpu_params p{};
    p.log_n = log_n;
    p.n_q = (int)q_bits.size();
    for (size_t i = 0; i < q_bits.size() && i < HEGPU_MAX_Q; ++i) p.q_bits[i] = q_bits[i];
    p.p_bits = p_bits;
    p.seed = seed;
    throw_status(hegpu_ctx_create(&p, device, &h_), hegpu_last_error(nullptr));
    hegpu_ctx_info(h_, &n_, &slots_, &l_, nullptr);
  }
  ~Context() { hegpu_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;

  hegpu_ctx* get() const { return h_; }
  int n() const { return n_; }
  int slots() const { return slots_; }
  int levels() const { return l_; }
  void check(int rc) const { throw_status(rc, hegpu_last_error(h_)); }

  // MeterContext::begin_stage / tally / stages (meter.hpp:40-70)
  void begin_stage(const std::string& label) { check(hegpu_begin_stage(h_, label.c_str())); }
  OpTally tally() const {
    int64_t t[5];
    check(hegpu_total_tally(h_, t));
    return OpTally{t[0], t[1], t[2], t[3], t[4]};
  }
  std::vector<std::pair<std::string, OpTally>> stages() const {
    std::vector<std::pair<std::string, OpTally>> out;
    char buf[128];
    int64_t t[5];
    for (int i = 0; i < hegpu_num_stages(h_); ++i) {
      check(hegpu_stage_tally(h_, i, buf, sizeof buf, t));
      out.emplace_back(buf, OpTally{t[0], t[1], t[2], t[3], t[4]});
    }
    return out;
  }
  void reset_meter() { check(hegpu_reset_meter(h_)); }
  void gen_rotation_keys(const std::vector<int64_t>& right_rots) {
    check(hegpu_gen_rotation_keys(h_, right_rots.data(), (int)right_rots.size()));
  }
  void gen_relin_key() { check(hegpu_gen_relin_key(h_)); }

  // client helpers (wire format, include/hegpu.h)
  std::vector<uint64_t> encode(const std::vector<double>& z, double scale, int level, bool with_p = false) const {
    std::vector<uint64_t> out((size_t)(level + (with_p ? 1 : 0)) * n_);
    check(hegpu_encode(h_, z.data(), (int)z.size(), scale, level, with_p, out.data()));
    return out;
  }
  std::vector<double> decode(const std::vector<uint64_t>& pt, int level, double scale) const {
    std::vector<double> out(slots_);
    check(hegpu_decode(h_, pt.data(), level, scale, out.data()));
    return out;
  }

 private:
  hegpu_ctx* h_ = nullptr;
  int n_ = 0, slots_ = 0, l_ = 0;
};

class Ciphertext {
 public:
  Ciphertext(Context& c, int count, int level) : c_(&c), count_(count), level_(level) {
    c.check(hegpu_ct_create(c.get(), count, level, &h_));
  }
  ~Ciphertext() { hegpu_ct_destroy(h_); }
  Ciphertext(Ciphertext&& o) noexcept : c_(o.c_), h_(o.h_), count_(o.count_), level_(o.level_) { o.h_ = nullptr; }
  Ciphertext& operator=(Ciphertext&& o) noexcept {
    std::swap(h_, o.h_);
    c_ = o.c_;
    count_ = o.count_;
    level_ = o.level_;
    return *this;
  }
  Ciphertext(const Ciphertext&) = delete;
  Ciphertext& operator=(const Ciphertext&) = delete;

  hegpu_ct* get() const { return h_; }
  Context& ctx() const { return *c_; }
  int count() const { return count_; }
  int level() const { return level_; }
  double scale() const {
    double s = 0;
    hegpu_ct_info(h_, nullptr, nullptr, &s);
    return s;
  }
  size_t words() const { return (size_t)count_ * 2 * level_ * c_->n(); }
  void upload(const std::vector<uint64_t>& wire, double scale) {
    c_->check(hegpu_ct_upload(h_, wire.data(), wire.size(), scale));
  }
  std::vector<uint64_t> download() const {
    std::vector<uint64_t> out(words());
    c_->check(hegpu_ct_download(h_, out.data(), out.size()));
    return out;
  }
  // decrypt + decode ciphertext i of the batch (client side)
  std::vector<double> decrypt(int i = 0) const {
    const std::vector<uint64_t> all = download();
    const size_t per = (size_t)2 * level_ * c_->n();
    std::vector<uint64_t> pt((size_t)level_ * c_->n());
    c_->check(hegpu_decrypt(c_->get(), all.data() + per * i, level_, pt.data()));
    return c_->decode(pt, level_, scale());
  }

 private:
  Context* c_;
  hegpu_ct* h_ = nullptr;
  int count_, level_;
};

class Plaintext {
 public:
  Plaintext(Context& c, const std::vector<double>& z, double scale, int level, bool with_p = false)
      : c_(&c), level_(level) {
    c.check(hegpu_pt_create(c.get(), 1, level, with_p, &h_));
    const std::vector<uint64_t> w = c.encode(z, scale, level, with_p);
    c.check(hegpu_pt_upload(h_, w.data(), w.size(), scale));
  }
  ~Plaintext() { hegpu_pt_destroy(h_); }
  Plaintext(const Plaintext&) = delete;
  Plaintext& operator=(const Plaintext&) = delete;
  hegpu_pt* get() const { return h_; }
  int level() const { return level_; }

 private:
  Context* c_;
  hegpu_pt* h_ = nullptr;
  int level_;
};

// pack(values, N, Kind::Ciphertext) -- client-side encode + encrypt
inline Ciphertext encrypt(const std::vector<double>& values, int level, uint64_t nonce, Context& ctx,
                          double scale = 1099511627776.0 /* 2^40 */) {
  const std::vector<uint64_t> pt = ctx.encode(values, scale, level);
  std::vector<uint64_t> ct((size_t)2 * level * ctx.n());
  ctx.check(hegpu_encrypt(ctx.get(), pt.data(), level, nonce, ct.data()));
  Ciphertext out(ctx, 1, level);
  out.upload(ct, scale);
  return out;
}

inline Ciphertext add(const Ciphertext& a, const Ciphertext& b, Context& ctx) {
  Ciphertext out(ctx, a.count(), a.level());
  ctx.check(hegpu_add(ctx.get(), a.get(), b.get(), out.get()));
  return out;
}
inline Ciphertext add(const Ciphertext& a, const Plaintext& p, Context& ctx) {
  Ciphertext out(ctx, a.count(), a.level());
  ctx.check(hegpu_add_plain(ctx.get(), a.get(), p.get(), out.get()));
  return out;
}
inline Ciphertext mul(const Ciphertext& a, const Plaintext& p, Context& ctx) {
  Ciphertext out(ctx, a.count(), a.level());
  ctx.check(hegpu_mul_plain(ctx.get(), a.get(), p.get(), out.get()));
  return out;
}
inline Ciphertext rescale(const Ciphertext& a, Context& ctx) {
  Ciphertext out(ctx, a.count(), a.level() - 1);
  ctx.check(hegpu_rescale(ctx.get(), a.get(), out.get()));
  return out;
}
inline Ciphertext rotate_right(const Ciphertext& v, int64_t r, Context& ctx) {
  Ciphertext out(ctx, v.count(), v.level());
  ctx.check(hegpu_rotate_right(ctx.get(), v.get(), r, out.get()));
  return out;
}
inline Ciphertext rotate_left(const Ciphertext& v, int64_t r, Context& ctx) {
  Ciphertext out(ctx, v.count(), v.level());
  ctx.check(hegpu_rotate_left(ctx.get(), v.get(), r, out.get()));
  return out;
}
inline Ciphertext square_layer(const Ciphertext& v, Context& ctx) {
  Ciphertext out(ctx, v.count(), v.level() - 1);
  ctx.check(hegpu_square(ctx.get(), v.get(), out.get()));
  return out;
}
inline Ciphertext merge_maps(const Ciphertext& maps, int c, int64_t w, Context& ctx) {
  Ciphertext out(ctx, maps.count() / c, maps.level());
  ctx.check(hegpu_merge_maps(ctx.get(), maps.get(), c, w, out.get()));
  return out;
}

// FilterBank (proj/include/hesim/refmodel.hpp:24-33): weights [c_out][c_in][k][k]
struct FilterBank {
  int c_out = 0, c_in = 0, k = 0;
  std::vector<double> weights, bias;
};
inline Ciphertext conv_packed_forward(const Ciphertext& taps, const FilterBank& f, int w_used, Context& ctx) {
  const int ntaps = f.c_in * f.k * f.k;
  Ciphertext out(ctx, taps.count() / ntaps * f.c_out, taps.level() - 1);
  ctx.check(hegpu_conv_packed_forward(ctx.get(), taps.get(), ntaps, f.weights.data(), f.c_out,
                                      f.bias.empty() ? nullptr : f.bias.data(), w_used, out.get()));
  return out;
}

// extract_diagonals + encoding, once per matrix (matvec.cpp:45-65)
class HsPlan {
 public:
  HsPlan(const std::vector<double>& A_row_major, int m, int n, int level, Context& ctx, bool skip_zero = true)
      : level_(level) {
    ctx.check(hegpu_hs_plan_create(ctx.get(), A_row_major.data(), m, n, level, skip_zero, &h_));
  }
  ~HsPlan() { hegpu_hs_plan_destroy(h_); }
  HsPlan(const HsPlan&) = delete;
  HsPlan& operator=(const HsPlan&) = delete;
  hegpu_hs_plan* get() const { return h_; }
  int level() const { return level_; }
  std::vector<int64_t> rotations() const {
    std::vector<int64_t> r(hegpu_hs_plan_rotations(h_, nullptr, 0));
    hegpu_hs_plan_rotations(h_, r.data(), (int)r.size());
    return r;
  }

 private:
  hegpu_hs_plan* h_ = nullptr;
  int level_;
};
inline Ciphertext hs_matvec(const HsPlan& plan, const Ciphertext& v, Context& ctx) {
  Ciphertext out(ctx, v.count(), v.level() - 1);
  ctx.check(hegpu_hs_matvec(ctx.get(), plan.get(), v.get(), out.get()));
  return out;
}

// ---- model / weights / input files (proj/include/hesim/modelio.hpp) --------
class ModelSpec {
 public:
  explicit ModelSpec(hegpu_model* h) : h_(h) {}
  ~ModelSpec() { hegpu_model_destroy(h_); }
  ModelSpec(const ModelSpec&) = delete;
  ModelSpec& operator=(const ModelSpec&) = delete;
  ModelSpec(ModelSpec&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  hegpu_model* get() const { return h_; }
  size_t weight_floats() const {
    size_t n = 0;
    hegpu_model_info(h_, nullptr, nullptr, nullptr, nullptr, &n);
    return n;
  }
  void check(int rc) const { throw_status(rc, hegpu_model_last_error(h_)); }

 private:
  hegpu_model* h_;
};

inline ModelSpec parse_model_json(const std::string& text) {
  hegpu_model* h = nullptr;
  throw_status(hegpu_model_parse(text.c_str(), &h), hegpu_model_last_error(nullptr));
  return ModelSpec(h);
}
inline ModelSpec resolve_model(const std::string& name_or_path) {
  hegpu_model* h = nullptr;
  throw_status(hegpu_model_load(name_or_path.c_str(), &h), hegpu_model_last_error(nullptr));
  return ModelSpec(h);
}
// flat float32-rounded weights in layer order (conv bank + bias, dense W + b)
inline std::vector<double> load_weights(const ModelSpec& m, const std::string& path) {
  std::vector<double> w(m.weight_floats());
  m.check(hegpu_model_load_weights(m.get(), path.c_str(), w.data(), w.size()));
  return w;
}
inline void save_weights(const ModelSpec& m, const std::vector<double>& w, const std::string& path) {
  m.check(hegpu_model_save_weights(m.get(), path.c_str(), w.data(), w.size()));
}
inline std::vector<double> load_input(const ModelSpec& m, const std::string& path) {
  int c = 0, d = 0;
  hegpu_model_info(m.get(), &c, &d, nullptr, nullptr, nullptr);
  std::vector<double> x((size_t)c * d * d);
  m.check(hegpu_model_load_input(m.get(), path.c_str(), x.data()));
  return x;
}


// ---- lower() / execute() (proj/include/hesim/netcompile.hpp:55-86) ---------
// The general stage driver: SubConv groups, grouped merges, the conv-pack
// repack, HS and LoLa-dense linear stages (include/hegpu.h, hegpu_prog_*).
enum class StageKind { ConvPack, Merge, Square, RepackConv, Linear };
struct Stage {
  StageKind kind;
  std::string label;
  int groups = 1;
  int policy = HEGPU_POLICY_HS;
};
struct OpReport {
  std::vector<std::pair<std::string, OpTally>> rows;
  OpTally total;
};
struct ExecResult {
  std::vector<double> logits;
  OpReport report;
};

// lower(model): the stage list alone (no device needed)
inline std::vector<Stage> lower(const ModelSpec& model) {
  char labels[64][64];
  int kinds[64], groups[64], pols[64];
  const int n = hegpu_model_lower(model.get(), 64, labels, kinds, groups, pols);
  if (n < 0) throw_status(-n, hegpu_prog_last_error(nullptr));
  std::vector<Stage> out;
  for (int i = 0; i < n && i < 64; ++i)
    out.push_back(Stage{static_cast<StageKind>(kinds[i]), labels[i], groups[i], pols[i]});
  return out;
}

// A lowered program bound to a context and its weights (keys, plans and
// plaintexts are prepared once; execute() evaluates one input).
class LoweredProgram {
 public:
  LoweredProgram(Context& ctx, const ModelSpec& model, const std::vector<double>& weights) : c_(&ctx) {
    throw_status(hegpu_prog_create(ctx.get(), model.get(), weights.data(), weights.size(), &h_),
                 hegpu_prog_last_error(nullptr));
    hegpu_prog_info(h_, &n_stages_, &input_cts_, &out_level_, &n_logits_);
  }
  ~LoweredProgram() { hegpu_prog_destroy(h_); }
  LoweredProgram(const LoweredProgram&) = delete;
  LoweredProgram& operator=(const LoweredProgram&) = delete;
  hegpu_prog* get() const { return h_; }
  Context& ctx() const { return *c_; }
  int input_cts() const { return input_cts_; }
  int out_level() const { return out_level_; }
  int n_logits() const { return n_logits_; }
  std::vector<Stage> stages() const {
    std::vector<Stage> out;
    for (int i = 0; i < n_stages_; ++i) {
      char label[64];
      int kind = 0, groups = 1, policy = 0;
      check(hegpu_prog_stage(h_, i, label, sizeof label, &kind, &groups, &policy));
      out.push_back(Stage{static_cast<StageKind>(kind), label, groups, policy});
    }
    return out;
  }
  void check(int rc) const { throw_status(rc, hegpu_prog_last_error(h_)); }

 private:
  Context* c_;
  hegpu_prog* h_ = nullptr;
  int n_stages_ = 0, input_cts_ = 0, out_level_ = 0, n_logits_ = 0;
};

// execute(program, weights, input, ctx) (netcompile.cpp:291-446): the client
// side (conv_pack / pack + encrypt, decrypt) is folded in here as in the
// simulator; `input` is [c][d][d] row-major.  The report is the context's
// per-stage tally of this run.
inline ExecResult execute(const LoweredProgram& prog, const std::vector<double>& input, uint64_t nonce = 0) {
  Context& ctx = prog.ctx();
  const int L = ctx.levels(), N = ctx.n();
  std::vector<uint64_t> in((size_t)prog.input_cts() * 2 * L * N);
  prog.check(hegpu_prog_encrypt_input(prog.get(), input.data(), nonce, in.data()));
  Ciphertext ci(ctx, prog.input_cts(), L), co(ctx, 1, prog.out_level());
  ci.upload(in, std::ldexp(1.0, 40));
  ctx.reset_meter();
  prog.check(hegpu_prog_run(prog.get(), ci.get(), co.get()));
  std::vector<uint64_t> out((size_t)2 * prog.out_level() * N);
  ctx.check(hegpu_ct_download(co.get(), out.data(), out.size()));
  ExecResult r;
  r.logits.resize(prog.n_logits());
  prog.check(hegpu_prog_decrypt_logits(prog.get(), out.data(), r.logits.data()));
  r.report.rows = ctx.stages();
  r.report.total = ctx.tally();
  return r;
}

}  // namespace hegpu
