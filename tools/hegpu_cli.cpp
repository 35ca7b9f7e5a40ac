// hegpu_cli -- the reference's command-line front end (proj/tools/hesim.cpp:
// run / count / sweep / verify, exit codes 0 ok, 1 I/O, 2 capacity/shape,
// 3 verification failure) over the encrypted B200 path.
//
//   hegpu_cli run   --model M [--weights W] [--input X] [--report R] [--seed S]
//   hegpu_cli count --model M [...]
//   hegpu_cli sweep [--n-min 16 --n-max 4096 --m-min 4 --m-max 512 --n-slots 4096,16384] [--measure]
//   hegpu_cli verify [--seed 1] [--cases 20] [--corrupt-kernel]
//
// M is a model JSON (path or name under $HECNN_MODEL_DIR) or a builtin name
// (cryptonets-hs, me, ce).  CKKS parameters follow the model: N = 2 n_slots,
// Q = {60, 40 x (1 + 2 dense stages)}, P = 60 bits.  Without --weights /
// --input the weights and input are drawn like the reference's
// random_weights / random_input (mt19937_64, N(0,1), the same scalings).
// Built by paper_2110_08321_b200/build.py next to libhegpu.so.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include <unistd.h>

#include "hegpu.h"

namespace {

constexpr int kExitOk = 0, kExitIo = 1, kExitCapacity = 2, kExitVerify = 3;

struct Fail {
  int code;
  std::string msg;
};

void fail_rc(int rc, const char* msg) {
  throw Fail{rc == HEGPU_ERR_IO ? kExitIo : kExitCapacity, msg && *msg ? msg : "hegpu error"};
}
// the message getter runs only after the call (argument order is unspecified)
#define check(call, msg)            \
  do {                              \
    const int rc_ = (call);         \
    if (rc_) fail_rc(rc_, (msg));   \
  } while (0)

// builtin layer lists (proj/src/netcompile.cpp:567-628), as model files
const std::map<std::string, std::string>& builtins() {
  static const std::map<std::string, std::string> b = {
      {"cryptonets-hs",
       R"({"name": "cryptonets-hs", "input": [1, 29, 29], "n_slots": 8192, "layers": [
        {"kind": "conv", "k": 5, "s": 2, "out_channels": 5, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 2, "s": 2}, {"kind": "conv", "k": 5, "s": 1, "out_channels": 50, "label": "Conv2"},
        {"kind": "avgpool", "k": 2, "s": 2}, {"kind": "flatten"}, {"kind": "dense", "units": 100, "label": "Dense1"},
        {"kind": "square"}, {"kind": "dense", "units": 10, "label": "Dense2"}]})"},
      {"me",
       R"({"name": "me", "input": [1, 30, 30], "n_slots": 8192, "layers": [
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 5, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 3, "s": 2}, {"kind": "conv", "k": 3, "s": 1, "out_channels": 50, "label": "Conv2"},
        {"kind": "avgpool", "k": 3, "s": 2}, {"kind": "flatten"}, {"kind": "dense", "units": 32, "label": "Dense1"},
        {"kind": "square"}, {"kind": "dense", "units": 10, "label": "Dense2"}]})"},
      {"ce",
       R"({"name": "ce", "input": [3, 32, 32], "n_slots": 16384, "layers": [
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 18, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool1"},
        {"kind": "subconv", "k": 3, "s": 1, "out_channels": 15, "groups": 3, "label": "Conv2"},
        {"kind": "conv", "k": 1, "s": 1, "out_channels": 64, "policy": "convpack", "label": "Conv3"},
        {"kind": "square"}, {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool2"},
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 64}, {"kind": "flatten"},
        {"kind": "dense", "units": 256, "label": "Dense1"}, {"kind": "square"},
        {"kind": "dense", "units": 10, "label": "Dense2"}]})"},
      // ce's layer list scaled to fit N = 4096 (ce itself declares n_slots = 16384, i.e. N = 2^15,
      // above the device NTT's 2^14): the same ten stages, three channel groups, the 1x1 repack conv
      {"ce-mini",
       R"({"name": "ce-mini", "input": [3, 16, 16], "n_slots": 2048, "layers": [
        {"kind": "conv", "k": 3, "s": 1, "out_channels": 6, "label": "Conv1"}, {"kind": "square"},
        {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool1"},
        {"kind": "subconv", "k": 3, "s": 1, "out_channels": 6, "groups": 3, "label": "Conv2"},
        {"kind": "conv", "k": 1, "s": 1, "out_channels": 8, "policy": "convpack", "label": "Conv3"},
        {"kind": "square"}, {"kind": "avgpool", "k": 2, "s": 2, "label": "Pool2"},
        {"kind": "conv", "k": 2, "s": 1, "out_channels": 12}, {"kind": "flatten"},
        {"kind": "dense", "units": 16, "label": "Dense1"}, {"kind": "square"},
        {"kind": "dense", "units": 10, "label": "Dense2"}]})"}};
  return b;
}

struct Model {
  hegpu_model* h = nullptr;
  int in_c = 0, in_d = 0, n_slots = 0, n_layers = 0;
  size_t nw = 0;
  std::string name;
  ~Model() { hegpu_model_destroy(h); }
  struct L {
    int kind, k, s, out, groups, policy;
  };
  std::vector<L> layers;
};

void load_model(const std::string& arg, Model& m) {
  const auto& b = builtins();
  const auto it = b.find(arg);
  const int rc = it != b.end() ? hegpu_model_parse(it->second.c_str(), &m.h) : hegpu_model_load(arg.c_str(), &m.h);
  check(rc, hegpu_model_last_error(nullptr));
  hegpu_model_info(m.h, &m.in_c, &m.in_d, &m.n_slots, &m.n_layers, &m.nw);
  m.name = it != b.end() ? arg : arg;
  for (int i = 0; i < m.n_layers; ++i) {
    Model::L l{};
    hegpu_model_layer(m.h, i, &l.kind, &l.k, &l.s, &l.out, &l.groups, &l.policy);
    m.layers.push_back(l);
  }
}

// (channels, side) entering each layer
std::pair<int, int> shape_before(const Model& m, int idx) {
  int c = m.in_c, d = m.in_d;
  for (int i = 0; i < idx; ++i) {
    const auto& l = m.layers[i];
    if (l.kind == HEGPU_LAYER_CONV || l.kind == HEGPU_LAYER_SUBCONV) {
      c = l.out;
      d = (d - l.k) / l.s + 1;
    } else if (l.kind == HEGPU_LAYER_AVGPOOL) {
      d = (d - l.k) / l.s + 1;
    } else if (l.kind == HEGPU_LAYER_DENSE) {
      c = l.out;
      d = 1;
    }
  }
  return {c, d};
}

// random_weights / random_input (proj/src/netcompile.cpp:515-565): the same
// engine, distributions and scalings, flattened in the weights-file order
std::vector<double> random_weights(const Model& m, uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  std::vector<double> w;
  auto filters = [&](int c_out, int c_in, int k) {
    const double scale = 1.0 / std::sqrt((double)(c_in * k * k));
    for (int i = 0; i < c_out * c_in * k * k; ++i) w.push_back(dist(rng) * scale);
    for (int i = 0; i < c_out; ++i) w.push_back(dist(rng) * 0.1);
  };
  for (int i = 0; i < m.n_layers; ++i) {
    const auto& l = m.layers[i];
    const auto s = shape_before(m, i);
    if (l.kind == HEGPU_LAYER_CONV) {
      filters(l.out, s.first, l.k);
    } else if (l.kind == HEGPU_LAYER_SUBCONV) {
      for (int g = 0; g < l.groups; ++g) filters(l.out / l.groups, s.first / l.groups, l.k);
    } else if (l.kind == HEGPU_LAYER_DENSE) {
      const int n = s.first * s.second * s.second;
      const double scale = 1.0 / std::sqrt((double)n);
      for (int r = 0; r < l.out * n; ++r) w.push_back(dist(rng) * scale);
      for (int r = 0; r < l.out; ++r) w.push_back(dist(rng) * 0.1);
    }
  }
  return w;
}

std::vector<double> random_input(const Model& m, uint64_t seed) {
  std::mt19937_64 rng(seed ^ 0x9e3779b97f4a7c15ull);
  std::normal_distribution<double> dist(0.0, 1.0);
  std::vector<double> x((size_t)m.in_c * m.in_d * m.in_d);
  for (auto& v : x) v = dist(rng);
  return x;
}

// FP64 forward pass of the layer list (proj/src/refmodel.cpp, netcompile.cpp:448-503)
std::vector<double> ref_forward(const Model& m, const std::vector<double>& w, const std::vector<double>& x) {
  std::vector<double> t = x;
  int c = m.in_c, d = m.in_d;
  size_t o = 0;
  for (const auto& l : m.layers) {
    if (l.kind == HEGPU_LAYER_CONV) {
      const int dout = (d - l.k) / l.s + 1;
      std::vector<double> y((size_t)l.out * dout * dout);
      const double* W = w.data() + o;
      const double* b = W + (size_t)l.out * c * l.k * l.k;
      for (int co = 0; co < l.out; ++co)
        for (int oy = 0; oy < dout; ++oy)
          for (int ox = 0; ox < dout; ++ox) {
            double acc = b[co];
            for (int ci = 0; ci < c; ++ci)
              for (int ky = 0; ky < l.k; ++ky)
                for (int kx = 0; kx < l.k; ++kx)
                  acc += W[((size_t)(co * c + ci) * l.k + ky) * l.k + kx] *
                         t[((size_t)ci * d + oy * l.s + ky) * d + ox * l.s + kx];
            y[((size_t)co * dout + oy) * dout + ox] = acc;
          }
      o += (size_t)l.out * c * l.k * l.k + l.out;
      t.swap(y);
      c = l.out;
      d = dout;
    } else if (l.kind == HEGPU_LAYER_AVGPOOL) {
      const int dout = (d - l.k) / l.s + 1;
      std::vector<double> y((size_t)c * dout * dout);
      const double scale = 1.0 / (double)(l.k * l.k);
      for (int ci = 0; ci < c; ++ci)
        for (int oy = 0; oy < dout; ++oy)
          for (int ox = 0; ox < dout; ++ox) {
            double acc = 0.0;
            for (int ky = 0; ky < l.k; ++ky)
              for (int kx = 0; kx < l.k; ++kx) acc += t[((size_t)ci * d + oy * l.s + ky) * d + ox * l.s + kx];
            y[((size_t)ci * dout + oy) * dout + ox] = acc * scale;
          }
      t.swap(y);
      d = dout;
    } else if (l.kind == HEGPU_LAYER_SQUARE) {
      for (auto& v : t) v *= v;
    } else if (l.kind == HEGPU_LAYER_DENSE) {
      const int n = c * d * d;
      const double* W = w.data() + o;
      const double* b = W + (size_t)l.out * n;
      std::vector<double> y(l.out);
      for (int r = 0; r < l.out; ++r) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += W[(size_t)r * n + j] * t[j];
        y[r] = acc + b[r];
      }
      o += (size_t)l.out * n + l.out;
      t.swap(y);
      c = l.out;
      d = 1;
    } else if (l.kind == HEGPU_LAYER_SUBCONV) {  // per channel group (netcompile.cpp:460-479)
      const int G = l.groups, pi = c / G, po = l.out / G, dout = (d - l.k) / l.s + 1;
      std::vector<double> y((size_t)l.out * dout * dout);
      for (int g = 0; g < G; ++g) {
        const double* W = w.data() + o;
        const double* b = W + (size_t)po * pi * l.k * l.k;
        for (int co = 0; co < po; ++co)
          for (int oy = 0; oy < dout; ++oy)
            for (int ox = 0; ox < dout; ++ox) {
              double acc = b[co];
              for (int ci = 0; ci < pi; ++ci)
                for (int ky = 0; ky < l.k; ++ky)
                  for (int kx = 0; kx < l.k; ++kx)
                    acc += W[((size_t)(co * pi + ci) * l.k + ky) * l.k + kx] *
                           t[((size_t)(g * pi + ci) * d + oy * l.s + ky) * d + ox * l.s + kx];
              y[((size_t)(g * po + co) * dout + oy) * dout + ox] = acc;
            }
        o += (size_t)po * pi * l.k * l.k + po;
      }
      t.swap(y);
      c = l.out;
      d = dout;
    }
  }
  return t;
}

struct Args {
  std::string cmd, model, weights, input, report, out, methods = "hs,lola-dense,lola-stacked";
  std::string policy;   // run / count: ModelSpec::default_policy (hesim.cpp:43-48)
  int model_slots = 0;  // run / count: --n-slots override of the model's slot count
  uint64_t seed = 0;
  bool seed_set = false, measure = false;
  bool worked = false;  // sweep --worked-example (hesim.cpp:152-165)
  bool corrupt_kernel = false;  // verify's negative control (hesim.cpp:212,237,334-337)
  int cases = 20, n_min = 16, n_max = 4096, m_min = 4, m_max = 512;
  std::vector<int> slots = {4096, 16384};
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) throw Fail{kExitCapacity, "usage: hegpu_cli run|count|sweep|verify [options]"};
  a.cmd = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) throw Fail{kExitCapacity, "missing value for " + k};
      return argv[++i];
    };
    if (k == "--model") a.model = val();
    else if (k == "--weights") a.weights = val();
    else if (k == "--input") a.input = val();
    else if (k == "--report") a.report = val();
    else if (k == "--out") a.out = val();
    else if (k == "--seed") a.seed = std::stoull(val()), a.seed_set = true;
    else if (k == "--cases") a.cases = std::stoi(val());
    else if (k == "--n-min") a.n_min = std::stoi(val());
    else if (k == "--n-max") a.n_max = std::stoi(val());
    else if (k == "--m-min") a.m_min = std::stoi(val());
    else if (k == "--m-max") a.m_max = std::stoi(val());
    else if (k == "--methods") a.methods = val();
    else if (k == "--measure") a.measure = true;
    else if (k == "--worked-example") a.worked = true;
    else if (k == "--corrupt-kernel") a.corrupt_kernel = true;
    else if (k == "--policy") a.policy = val();
    else if (k == "--n-slots") {
      a.slots.clear();
      std::stringstream ss(val());
      std::string tok;
      while (std::getline(ss, tok, ',')) a.slots.push_back(std::stoi(tok));
      if (a.slots.size() == 1) a.model_slots = a.slots[0];
    } else throw Fail{kExitCapacity, "unknown option " + k};
  }
  if (!a.seed_set && a.cmd == "verify") a.seed = 1;
  return a;
}

int log2i(int x) {
  int b = 0;
  while ((1 << b) < x) ++b;
  return b;
}

struct Ctx {
  hegpu_ctx* h = nullptr;
  explicit Ctx(int log_n, int n_q, uint64_t seed) {
    hegpu_params p{};
    p.log_n = log_n;
    p.n_q = n_q;
    // N = 2^15 (ce's n_slots = 16384) runs on the FP64 NTT: every prime below 2^45
    p.q_bits[0] = log_n > 14 ? 45 : 60;
    for (int i = 1; i < n_q; ++i) p.q_bits[i] = 40;
    p.p_bits = log_n > 14 ? 45 : 60;
    p.seed = seed;
    check(hegpu_ctx_create(&p, 0, &h), hegpu_last_error(nullptr));
  }
  ~Ctx() { hegpu_ctx_destroy(h); }
  void ok(int rc) const {
    if (rc) fail_rc(rc, hegpu_last_error(h));
  }
};

struct Report {
  std::vector<std::pair<std::string, std::vector<int64_t>>> rows;
  std::vector<int64_t> total;
  std::string csv() const {  // OpReport::to_csv, netcompile.cpp:655-665
    std::ostringstream os;
    os << "layer,total,add_pc,add_cc,mul_pc,mul_cc,rot\n";
    auto line = [&os](const std::string& l, const std::vector<int64_t>& t) {
      os << l << "," << (t[0] + t[1] + t[2] + t[3] + t[4]) << "," << t[0] << "," << t[1] << "," << t[2] << ","
         << t[3] << "," << t[4] << "\n";
    };
    for (const auto& r : rows) line(r.first, r.second);
    line("Total", total);
    return os.str();
  }
};

struct RunResult {
  std::vector<double> logits, want;
  Report report;
};

void collect_report(const Ctx& ctx, Report& rep) {
  for (int i = 0; i < hegpu_num_stages(ctx.h); ++i) {
    char label[128];
    int64_t t[5];
    ctx.ok(hegpu_stage_tally(ctx.h, i, label, sizeof label, t));
    rep.rows.emplace_back(label, std::vector<int64_t>(t, t + 5));
  }
  int64_t t[5];
  ctx.ok(hegpu_total_tally(ctx.h, t));
  rep.total.assign(t, t + 5);
}

// models outside the conv -> (square, linear)* family (SubConv groups, the
// stand-alone conv-pack repack, LoLa-dense stages, a dense first layer): the
// general stage driver hegpu_prog (execute, netcompile.cpp:291-446)
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

RunResult run_program(const Model& m, const std::vector<double>& w, const std::vector<double>& x, uint64_t seed) {
  const double t0 = now_s();
  char labels[64][64];
  int kinds[64], groups[64], pols[64];
  const int ns = hegpu_model_lower(m.h, 64, labels, kinds, groups, pols);
  if (ns < 0) fail_rc(-ns, hegpu_prog_last_error(nullptr));
  int depth = 0;
  for (int i = 0; i < ns && i < 64; ++i)
    depth += kinds[i] == HEGPU_STAGE_MERGE ? 0 : (kinds[i] == HEGPU_STAGE_LINEAR && pols[i] == HEGPU_POLICY_LOLA_DENSE) ? 2 : 1;
  Ctx ctx(log2i(2 * m.n_slots), depth + 1, seed + 1);
  hegpu_prog* prog = nullptr;
  const int rc = hegpu_prog_create(ctx.h, m.h, w.data(), w.size(), &prog);
  if (rc) fail_rc(rc, hegpu_prog_last_error(nullptr));
  int n_in = 0, out_level = 0, n_logits = 0, n, slots, L;
  hegpu_prog_info(prog, nullptr, &n_in, &out_level, &n_logits);
  hegpu_ctx_info(ctx.h, &n, &slots, &L, nullptr);
  std::vector<uint64_t> in((size_t)n_in * 2 * L * n);
  auto pok = [&](int r) {
    if (r) fail_rc(r, hegpu_prog_last_error(prog));
  };
  const double t1 = now_s();
  pok(hegpu_prog_encrypt_input(prog, x.data(), seed, in.data()));
  hegpu_ct *di = nullptr, *out = nullptr;
  ctx.ok(hegpu_ct_create(ctx.h, n_in, L, &di));
  ctx.ok(hegpu_ct_upload(di, in.data(), in.size(), std::ldexp(1.0, 40)));
  ctx.ok(hegpu_ct_create(ctx.h, 1, out_level, &out));
  ctx.ok(hegpu_reset_meter(ctx.h));
  // first run: resolves the plans' fused key tables; the second run is the
  // steady-state evaluation time of one encrypted inference
  const double t2 = now_s();
  pok(hegpu_prog_run(prog, di, out));
  const double t3 = now_s();
  pok(hegpu_prog_run(prog, di, out));
  const double t4 = now_s();
  ctx.ok(hegpu_reset_meter(ctx.h));
  pok(hegpu_prog_run(prog, di, out));
  std::fprintf(stderr, "timing: setup (keys, plans) %.2f s, client encrypt %.2f s, first run %.3f s, evaluation %.1f ms\n",
               t1 - t0, t2 - t1, t3 - t2, (t4 - t3) * 1e3);
  std::vector<uint64_t> o((size_t)2 * out_level * n);
  ctx.ok(hegpu_ct_download(out, o.data(), o.size()));
  RunResult r;
  r.logits.resize(n_logits);
  pok(hegpu_prog_decrypt_logits(prog, o.data(), r.logits.data()));
  collect_report(ctx, r.report);
  hegpu_ct_destroy(di);
  hegpu_ct_destroy(out);
  hegpu_prog_destroy(prog);
  return r;
}

RunResult run_model(const Model& m, const std::vector<double>& w, const std::vector<double>& x, uint64_t seed,
                    const std::string& weights_path) {
  hegpu_net_spec spec{};
  if (hegpu_model_net_spec(m.h, &spec) != HEGPU_OK) return run_program(m, w, x, seed);
  Ctx ctx(log2i(2 * m.n_slots), 2 + 2 * spec.n_dense, seed + 1);
  // the net reads a weights file: write the (random) weights to a temp file
  std::string wpath = weights_path;
  if (wpath.empty()) {
    wpath = "/tmp/hegpu_cli_w_" + std::to_string(::getpid()) + ".bin";
    check(hegpu_model_save_weights(m.h, wpath.c_str(), w.data(), w.size()), hegpu_model_last_error(m.h));
  }
  hegpu_net* net = nullptr;
  const int rc = hegpu_net_create_from_model(ctx.h, m.h, wpath.c_str(), &net);
  if (weights_path.empty()) std::remove(wpath.c_str());
  if (rc) {
    const char* e = hegpu_model_last_error(m.h);
    throw Fail{rc == HEGPU_ERR_IO ? kExitIo : kExitCapacity,
               (e && *e) ? e : hegpu_last_error(ctx.h)};
  }
  const int ntaps = hegpu_net_tap_cts(net);  // tap ciphertexts per image (region-packed)
  int n, slots, L;
  hegpu_ctx_info(ctx.h, &n, &slots, &L, nullptr);
  const int out_level = L - 1 - 2 * spec.n_dense;
  std::vector<uint64_t> taps((size_t)ntaps * 2 * L * n);
  ctx.ok(hegpu_net_encrypt_image(net, x.data(), seed, taps.data()));
  hegpu_ct *dt = nullptr, *out = nullptr;
  ctx.ok(hegpu_ct_create(ctx.h, ntaps, L, &dt));
  ctx.ok(hegpu_ct_upload(dt, taps.data(), taps.size(), std::ldexp(1.0, 40)));
  ctx.ok(hegpu_ct_create(ctx.h, 1, out_level, &out));
  ctx.ok(hegpu_reset_meter(ctx.h));
  ctx.ok(hegpu_net_run(net, dt, out));
  std::vector<uint64_t> o((size_t)2 * out_level * n);
  ctx.ok(hegpu_ct_download(out, o.data(), o.size()));
  RunResult r;
  r.logits.resize(spec.dense_out[spec.n_dense - 1]);
  ctx.ok(hegpu_net_decrypt_logits(net, o.data(), r.logits.data()));
  collect_report(ctx, r.report);
  hegpu_ct_destroy(dt);
  hegpu_ct_destroy(out);
  hegpu_net_destroy(net);
  return r;
}

void inputs(const Args& a, const Model& m, std::vector<double>& w, std::vector<double>& x) {
  if (a.weights.empty()) {
    w = random_weights(m, a.seed);
  } else {
    w.resize(m.nw);
    check(hegpu_model_load_weights(m.h, a.weights.c_str(), w.data(), w.size()), hegpu_model_last_error(m.h));
  }
  if (a.input.empty()) {
    x = random_input(m, a.seed);
  } else {
    x.resize((size_t)m.in_c * m.in_d * m.in_d);
    check(hegpu_model_load_input(m.h, a.input.c_str(), x.data()), hegpu_model_last_error(m.h));
  }
}

void emit(const std::string& path, const std::string& text) {
  if (path.empty()) {
    std::fputs(text.c_str(), stdout);
    return;
  }
  std::ofstream o(path, std::ios::binary);
  if (!o) throw Fail{kExitIo, "cannot open " + path + " for writing"};
  o << text;
}

int cmd_run(const Args& a, bool table) {
  if (a.model.empty()) throw Fail{kExitCapacity, "--model is required"};
  Model m;
  load_model(a.model, m);
  if (!a.policy.empty()) {  // configured_model, hesim.cpp:43-48
    const int pol = a.policy == "hs" ? HEGPU_POLICY_HS : a.policy == "lola-dense" ? HEGPU_POLICY_LOLA_DENSE
                    : a.policy == "lola-stacked" ? HEGPU_POLICY_LOLA_STACKED : -1;
    if (pol < 0) throw Fail{kExitCapacity, "unknown policy " + a.policy};
    check(hegpu_model_set_default_policy(m.h, pol), "set_default_policy");
  }
  if (a.model_slots > 0) {
    check(hegpu_model_set_n_slots(m.h, a.model_slots), "set_n_slots");
    m.n_slots = a.model_slots;
  }
  std::vector<double> w, x;
  inputs(a, m, w, x);
  const RunResult r = run_model(m, w, x, a.seed, a.weights);
  if (!table) {
    for (size_t i = 0; i < r.logits.size(); ++i) std::printf("logit,%zu,%.9g\n", i, r.logits[i]);
    emit(a.report, r.report.csv());
    return kExitOk;
  }
  std::printf("model: %s\n", a.model.c_str());
  std::printf("%-16s %8s %8s %8s %8s %8s %8s\n", "Layer", "HOPs", "AddPC", "AddCC", "MulPC", "MulCC", "Rot");
  auto line = [](const std::string& l, const std::vector<int64_t>& t, bool dash) {
    auto c = [&](int64_t v) { return dash && v == 0 ? std::string("-") : std::to_string(v); };
    std::printf("%-16s %8s %8s %8s %8s %8s %8s\n", l.c_str(), std::to_string(t[0] + t[1] + t[2] + t[3] + t[4]).c_str(),
                c(t[0]).c_str(), c(t[1]).c_str(), c(t[2]).c_str(), c(t[3]).c_str(), c(t[4]).c_str());
  };
  for (const auto& row : r.report.rows) line(row.first, row.second, true);
  line("Total", r.report.total, false);
  if (!a.report.empty()) emit(a.report, r.report.csv());
  return kExitOk;
}

// predict_hs (proj/src/matvec.cpp:168-187): rotations, multiplications
std::pair<int64_t, int64_t> predict_hs(int64_t m, int64_t n, int64_t N) {
  auto clog2 = [](int64_t x) {
    int b = 0;
    while ((int64_t{1} << b) < x) ++b;
    return b;
  };
  const bool plain = N >= m + n - 1 && (m << clog2((m + n - 1 + m - 1) / m)) <= N;
  int64_t me = m;
  if (!plain) {
    me = 1;
    while (me < m) me <<= 1;
  }
  const int folds = plain ? clog2((m + n - 1 + m - 1) / m) : clog2(N / me);
  return {me - 1 + folds, me};
}

// predict_lola_dense / predict_lola_stacked (proj/src/matvec.cpp:189-211)
std::pair<int64_t, int64_t> predict_lola(bool stacked, int64_t m, int64_t n, int64_t N) {
  int lg = 0;
  while ((int64_t{1} << lg) < n) ++lg;
  if (!stacked) return {m * lg, m};
  const int64_t delta = int64_t{1} << lg;
  if (delta > N) throw Fail{kExitCapacity, "stacked: padded width exceeds slot count"};
  const int64_t k = N / delta, batches = (m + k - 1) / k;
  return {batches * (k + lg - 1) + batches - 1, batches};
}

// one kernel call on the GPU with a dense matrix of U[0.5, 1.5] entries
// (hesim.cpp:119-140): the context's metered rotations / multiplications
std::pair<int64_t, int64_t> measure_gpu(const std::string& method, int m, int n, int N, uint64_t seed) {
  const bool hs = method == "hs";
  const int level = hs ? 2 : 3;
  Ctx ctx(log2i(2 * N), level, seed + 7);
  std::mt19937_64 rng(seed ^ ((uint64_t)m << 32) ^ (uint64_t)n ^ ((uint64_t)N << 16));
  std::uniform_real_distribution<double> dist(0.5, 1.5);
  std::vector<double> A((size_t)m * n), xv(n);
  for (auto& v : A) v = dist(rng);
  for (auto& v : xv) v = dist(rng);
  hegpu_hs_plan* hp = nullptr;
  hegpu_lola_plan* lp = nullptr;
  std::vector<int64_t> rots(4 * (size_t)N + 64);
  int nr = 0, outs = 1;
  if (hs) {
    ctx.ok(hegpu_hs_plan_create(ctx.h, A.data(), m, n, level, 1, &hp));
    nr = hegpu_hs_plan_rotations(hp, rots.data(), (int)rots.size());
  } else {
    ctx.ok(hegpu_lola_plan_create(ctx.h, method == "lola-dense" ? HEGPU_LOLA_DENSE : HEGPU_LOLA_STACKED, A.data(), m,
                                  n, level, &lp));
    nr = hegpu_lola_plan_rotations(lp, rots.data(), (int)rots.size());
    ctx.ok(hegpu_lola_plan_info(lp, nullptr, nullptr, nullptr, nullptr, &outs));
  }
  ctx.ok(hegpu_gen_rotation_keys(ctx.h, rots.data(), nr));
  int nn, slots, L;
  hegpu_ctx_info(ctx.h, &nn, &slots, &L, nullptr);
  std::vector<uint64_t> pt((size_t)level * nn), ct((size_t)2 * level * nn);
  ctx.ok(hegpu_encode(ctx.h, xv.data(), n, std::ldexp(1.0, 40), level, 0, pt.data()));
  ctx.ok(hegpu_encrypt(ctx.h, pt.data(), level, 1, ct.data()));
  hegpu_ct *v = nullptr, *o = nullptr;
  ctx.ok(hegpu_ct_create(ctx.h, 1, level, &v));
  ctx.ok(hegpu_ct_upload(v, ct.data(), ct.size(), std::ldexp(1.0, 40)));
  ctx.ok(hegpu_ct_create(ctx.h, outs, hs ? level - 1 : level - 2, &o));
  ctx.ok(hegpu_reset_meter(ctx.h));
  if (hs) ctx.ok(hegpu_hs_matvec(ctx.h, hp, v, o));
  else ctx.ok(hegpu_lola_matvec(ctx.h, lp, v, o));
  int64_t t[5];
  ctx.ok(hegpu_total_tally(ctx.h, t));
  hegpu_ct_destroy(v);
  hegpu_ct_destroy(o);
  if (hp) hegpu_hs_plan_destroy(hp);
  if (lp) hegpu_lola_plan_destroy(lp);
  return {t[4], t[2]};
}

// cmd_sweep (proj/tools/hesim.cpp:142-208): predicted (and with --measure,
// GPU-metered) rotations / multiplications per method, n, m, N
int cmd_sweep(const Args& a) {
  std::vector<std::string> methods;
  {
    std::stringstream ss(a.methods);
    std::string m;
    while (std::getline(ss, m, ','))
      if (!m.empty()) methods.push_back(m);
  }
  for (const auto& m : methods)
    if (m != "hs" && m != "lola-dense" && m != "lola-stacked") throw Fail{kExitCapacity, "--methods: unknown method " + m};
  std::ostringstream os;
  if (a.worked) {  // the m = 64, n = 4096, N = 16384 example of section 3.2 (matvec.hpp:74-83)
    const int m = 64, n = 4096, N = 16384;
    os << "method,n,m,N,rotations,multiplications\n";
    const auto hs = predict_hs(m, n, N), dn = predict_lola(false, m, n, N), st = predict_lola(true, m, n, N);
    os << "hs," << n << "," << m << "," << N << "," << hs.first << "," << hs.second << "\n";
    os << "lola-dense," << n << "," << m << "," << N << "," << dn.first << "," << dn.second << "\n";
    os << "lola-stacked," << n << "," << m << "," << N << "," << st.first << "," << st.second << "\n";
    os << "# prose reference: hs rotations 77, lola-stacked rotations 1023, lola-stacked multiplications 64\n";
    emit(a.out, os.str());
    return kExitOk;
  }
  os << "method,n,m,N,rotations,multiplications";
  if (a.measure) os << ",measured_rotations,measured_multiplications";
  os << "\n";
  for (const std::string& method : methods)
    for (int n = a.n_min; n <= a.n_max; n *= 2)
      for (int m = a.m_min; m <= a.m_max; m *= 2)
        for (int N : a.slots) {
          if (n > N || m > N) continue;
          const auto p = method == "hs" ? predict_hs(m, n, N) : predict_lola(method == "lola-stacked", m, n, N);
          os << method << "," << n << "," << m << "," << N << "," << p.first << "," << p.second;
          if (a.measure && log2i(2 * N) > 15) {
            os << ",,";  // ring degree 2N above the device NTT's 2^15
          } else if (a.measure) {
            const auto g = measure_gpu(method, m, n, N, a.seed);
            os << "," << g.first << "," << g.second;
          }
          os << "\n";
        }
  emit(a.out, os.str());
  return kExitOk;
}

// randomized suites (hesim.cpp:219-284) on the encrypted path: HS kernel
// vs A x, and the lowered encrypted builtins vs the FP64 forward pass; the
// tolerances are CKKS's (relative 1e-5 for one HS, 1e-3 on logits)
int cmd_verify(const Args& a) {
  std::mt19937_64 rng(a.seed);
  std::uniform_real_distribution<double> dist(-1.0, 1.0);
  double max_err = 0.0;
  bool ok = true;
  {
    Ctx ctx(13, 2, a.seed + 11);
    int n_, S, L;
    hegpu_ctx_info(ctx.h, &n_, &S, &L, nullptr);
    for (int c = 0; c < a.cases; ++c) {
      const int m = 1 + (int)(rng() % 48), n = 1 + (int)(rng() % 200);
      std::vector<double> A((size_t)m * n), xv(n);
      for (auto& v : A) v = dist(rng);
      for (auto& v : xv) v = dist(rng);
      hegpu_hs_plan* plan = nullptr;
      ctx.ok(hegpu_hs_plan_create(ctx.h, A.data(), m, n, 2, 1, &plan));
      std::vector<int64_t> rots(S + 64);
      ctx.ok(hegpu_gen_rotation_keys(ctx.h, rots.data(), hegpu_hs_plan_rotations(plan, rots.data(), (int)rots.size())));
      std::vector<uint64_t> pt((size_t)2 * n_), ct((size_t)4 * n_), o((size_t)2 * n_), dp((size_t)n_);
      ctx.ok(hegpu_encode(ctx.h, xv.data(), n, std::ldexp(1.0, 40), 2, 0, pt.data()));
      ctx.ok(hegpu_encrypt(ctx.h, pt.data(), 2, (uint64_t)c, ct.data()));
      hegpu_ct *v = nullptr, *out = nullptr;
      ctx.ok(hegpu_ct_create(ctx.h, 1, 2, &v));
      ctx.ok(hegpu_ct_upload(v, ct.data(), ct.size(), std::ldexp(1.0, 40)));
      ctx.ok(hegpu_ct_create(ctx.h, 1, 1, &out));
      ctx.ok(hegpu_hs_matvec(ctx.h, plan, v, out));
      ctx.ok(hegpu_ct_download(out, o.data(), o.size()));
      ctx.ok(hegpu_decrypt(ctx.h, o.data(), 1, dp.data()));
      std::vector<double> y(S);
      ctx.ok(hegpu_decode(ctx.h, dp.data(), 1, std::ldexp(1.0, 40), y.data()));
      for (int r = 0; r < m; ++r) {
        double want = 0.0;
        for (int j = 0; j < n; ++j) want += A[(size_t)r * n + j] * xv[j];
        if (a.corrupt_kernel && r == 0) want += 1e-3;  // negative control: perturbed expectation
        max_err = std::max(max_err, std::fabs(y[r] - want) / std::max(1.0, std::fabs(want)));
      }
      hegpu_ct_destroy(v);
      hegpu_ct_destroy(out);
      hegpu_hs_plan_destroy(plan);
    }
    if (max_err >= 1e-5) ok = false;
    std::printf("kernel-vs-oracle: %d cases, max relative error %.3g\n", a.cases, max_err);
  }
  double e2e = 0.0;
  for (const char* name : {"cryptonets-hs", "me", "ce-mini"}) {  // ce itself: tests/run_ce.py (58 GB of keys)
    Model m;
    load_model(name, m);
    const int draws = std::max(1, std::min(a.cases, 3));
    for (int d = 0; d < draws; ++d) {
      const uint64_t seed = a.seed * 1000 + d;
      const auto w = random_weights(m, seed);
      const auto x = random_input(m, seed);
      const RunResult r = run_model(m, w, x, seed, "");
      const auto want = ref_forward(m, w, x);
      for (size_t i = 0; i < want.size(); ++i)
        e2e = std::max(e2e, std::fabs(r.logits[i] - want[i]) / std::max(1.0, std::fabs(want[i])));
    }
    std::printf("end-to-end %s: %d draws, max relative error %.3g\n", name, draws, e2e);
  }
  std::printf("end-to-end ce: not part of verify (N = 2^15 with ~1200 rotation keys; see tests/run_ce.py); ce-mini runs its stages\n");
  if (e2e >= 1e-3) ok = false;
  std::printf("max observed error: %.3g\n", std::max(max_err, e2e));
  std::printf("%s\n", ok ? "verify: PASS" : "verify: FAIL");
  return ok ? kExitOk : kExitVerify;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    const Args a = parse(argc, argv);
    if (a.cmd == "run") return cmd_run(a, false);
    if (a.cmd == "count") return cmd_run(a, true);
    if (a.cmd == "sweep") return cmd_sweep(a);
    if (a.cmd == "verify") return cmd_verify(a);
    throw Fail{kExitCapacity, "unknown command " + a.cmd};
  } catch (const Fail& f) {
    std::fprintf(stderr, "error: %s\n", f.msg.c_str());
    return f.code;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitCapacity;
  }
}
