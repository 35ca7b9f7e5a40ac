// modelio.cpp -- model / weights / input files, the
// identical-input channel between the oracle, the GPU path and the reference:
//   model JSON  {"name", "input": [c, d, d], "n_slots", "layers": [{"kind",
//               "k", "s", "out_channels" | "units", "groups", "policy",
//               "label"}]}, unknown keys rejected (proj/src/modelio.cpp:106-147)
//   weights     little-endian float32 in layer order: conv [c_out][c_in][k][k]
//               then [c_out]; dense [m][n] then [m] (:169-202)
//   input       [c][d][d] little-endian float32 (:231-248)
// Errors are HEGPU_ERR_IO (hesim::IoError).  The JSON reader is a small
// recursive-descent parser for exactly what these files contain.
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <utility>
#include <vector>

#include "core.hpp"
#include "hegpu.h"
#include "lower.hpp"

using namespace hegpu;

namespace {

// ------------------------------------------------------------------ JSON
struct JVal {
  enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
  bool b = false;
  double num = 0;
  std::string str;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& key) const {
    for (const auto& kv : obj)
      if (kv.first == key) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const std::string& t;
  size_t i = 0;
  [[noreturn]] void err(const std::string& what) const {
    fail(HEGPU_ERR_IO, "model JSON parse error at offset " + std::to_string(i) + ": " + what);
  }
  void ws() {
    while (i < t.size() && (t[i] == ' ' || t[i] == '\n' || t[i] == '\r' || t[i] == '\t')) ++i;
  }
  bool lit(const char* s) {
    const size_t n = std::strlen(s);
    if (t.compare(i, n, s) == 0) {
      i += n;
      return true;
    }
    return false;
  }
  std::string string() {
    if (t[i] != '"') err("expected a string");
    ++i;
    std::string out;
    while (i < t.size() && t[i] != '"') {
      char c = t[i++];
      if (c == '\\') {
        if (i >= t.size()) err("bad escape");
        const char e = t[i++];
        switch (e) {
          case '"': case '\\': case '/': out += e; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'n': out += '\n'; break;
          case 'r': out += '\r'; break;
          case 't': out += '\t'; break;
          case 'u': {
            if (i + 4 > t.size()) err("bad \\u escape");
            const unsigned cp = (unsigned)std::strtoul(t.substr(i, 4).c_str(), nullptr, 16);
            i += 4;
            if (cp < 0x80) out += (char)cp;  // names and labels are ASCII
            else err("non-ASCII \\u escape");
            break;
          }
          default: err("bad escape");
        }
      } else {
        out += c;
      }
    }
    if (i >= t.size()) err("unterminated string");
    ++i;
    return out;
  }
  JVal value() {
    ws();
    if (i >= t.size()) err("unexpected end of input");
    JVal v;
    const char c = t[i];
    if (c == '{') {
      v.kind = JVal::Obj;
      ++i;
      ws();
      if (t[i] == '}') {
        ++i;
        return v;
      }
      for (;;) {
        ws();
        std::string key = string();
        ws();
        if (t[i] != ':') err("expected ':'");
        ++i;
        v.obj.emplace_back(std::move(key), value());
        ws();
        if (t[i] == ',') { ++i; continue; }
        if (t[i] == '}') { ++i; break; }
        err("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.kind = JVal::Arr;
      ++i;
      ws();
      if (t[i] == ']') {
        ++i;
        return v;
      }
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (t[i] == ',') { ++i; continue; }
        if (t[i] == ']') { ++i; break; }
        err("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.kind = JVal::Str;
      v.str = string();
    } else if (lit("true")) {
      v.kind = JVal::Bool;
      v.b = true;
    } else if (lit("false")) {
      v.kind = JVal::Bool;
    } else if (lit("null")) {
      v.kind = JVal::Null;
    } else {
      const char* p = t.c_str() + i;
      char* end = nullptr;
      v.num = std::strtod(p, &end);
      if (end == p) err("unexpected character");
      v.kind = JVal::Num;
      i += (size_t)(end - p);
    }
    return v;
  }
};

[[noreturn]] void io(const std::string& msg) { fail(HEGPU_ERR_IO, msg); }

void reject_unknown(const JVal& o, std::initializer_list<const char*> allowed, const std::string& where) {
  for (const auto& kv : o.obj) {
    bool ok = false;
    for (const char* a : allowed) ok = ok || kv.first == a;
    if (!ok) io("unknown field \"" + kv.first + "\" in " + where);
  }
}

const JVal& at(const JVal& o, const char* key) {
  const JVal* v = o.get(key);
  if (!v) io(std::string("model JSON: missing field \"") + key + "\"");
  return *v;
}

int as_int(const JVal& v, const char* what) {
  if (v.kind != JVal::Num || v.num != std::floor(v.num)) io(std::string("model JSON: ") + what + " must be an integer");
  return (int)v.num;
}

std::string as_str(const JVal& v, const char* what) {
  if (v.kind != JVal::Str) io(std::string("model JSON: ") + what + " must be a string");
  return v.str;
}

int parse_kind(const std::string& s) {
  if (s == "conv") return HEGPU_LAYER_CONV;
  if (s == "subconv") return HEGPU_LAYER_SUBCONV;
  if (s == "avgpool") return HEGPU_LAYER_AVGPOOL;
  if (s == "square") return HEGPU_LAYER_SQUARE;
  if (s == "flatten") return HEGPU_LAYER_FLATTEN;
  if (s == "dense") return HEGPU_LAYER_DENSE;
  io("unknown layer kind \"" + s + "\"");
}

int parse_policy(const std::string& s) {
  if (s == "convpack") return HEGPU_POLICY_CONVPACK;
  if (s == "hs") return HEGPU_POLICY_HS;
  if (s == "lola-dense") return HEGPU_POLICY_LOLA_DENSE;
  if (s == "lola-stacked") return HEGPU_POLICY_LOLA_STACKED;
  io("unknown kernel policy \"" + s + "\"");
}

std::string read_file(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) io("cannot open " + path);
  std::ostringstream os;
  os << in.rdbuf();
  return os.str();
}

bool exists(const std::string& p) {
  struct stat st;
  return ::stat(p.c_str(), &st) == 0;
}

}  // namespace


namespace {

std::unique_ptr<hegpu_model> parse_model(const std::string& text) {
  JParser p{text};
  const JVal doc = p.value();
  p.ws();
  if (p.i != text.size()) p.err("trailing characters");
  if (doc.kind != JVal::Obj) io("model JSON: top level must be an object");
  reject_unknown(doc, {"name", "input", "n_slots", "layers"}, "model");
  auto m = std::make_unique<hegpu_model>();
  m->name = as_str(at(doc, "name"), "name");
  const JVal& input = at(doc, "input");
  if (input.kind != JVal::Arr || input.arr.size() != 3 || as_int(input.arr[1], "input") != as_int(input.arr[2], "input"))
    io("input must be [channels, d, d]");
  m->in_c = as_int(input.arr[0], "input");
  m->in_d = as_int(input.arr[1], "input");
  m->n_slots = as_int(at(doc, "n_slots"), "n_slots");
  const JVal& layers = at(doc, "layers");
  if (layers.kind != JVal::Arr) io("model JSON: layers must be an array");
  for (const JVal& jl : layers.arr) {
    if (jl.kind != JVal::Obj) io("model JSON: a layer must be an object");
    reject_unknown(jl, {"kind", "k", "s", "out_channels", "units", "groups", "policy", "label"}, "layer");
    ModelLayer l;
    l.kind = parse_kind(as_str(at(jl, "kind"), "kind"));
    if (const JVal* v = jl.get("k")) l.k = as_int(*v, "k");
    if (const JVal* v = jl.get("s")) l.s = as_int(*v, "s");
    if (const JVal* v = jl.get("out_channels")) l.out = as_int(*v, "out_channels");
    if (const JVal* v = jl.get("units")) l.out = as_int(*v, "units");
    if (const JVal* v = jl.get("groups")) l.groups = as_int(*v, "groups");
    if (const JVal* v = jl.get("policy")) l.policy = parse_policy(as_str(*v, "policy"));
    if (const JVal* v = jl.get("label")) l.label = as_str(*v, "label");
    m->layers.push_back(std::move(l));
  }
  return m;
}

std::vector<double> read_f32(std::ifstream& in, size_t count, const std::string& path) {
  std::vector<float> raw(count);
  in.read(reinterpret_cast<char*>(raw.data()), (std::streamsize)(count * sizeof(float)));
  if ((size_t)in.gcount() != count * sizeof(float)) io(path + ": truncated float32 stream");
  return {raw.begin(), raw.end()};
}

void expect_end(std::ifstream& in, const std::string& path, const char* what) {
  char extra;
  if (in.read(&extra, 1)) io(path + ": trailing bytes after expected " + what);
}

template <typename F>
int guarded_model(hegpu_model* m, F&& f) {
  try {
    f();
    return HEGPU_OK;
  } catch (const Error& e) {
    if (m) m->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (m) m->last_error = e.what();
    return HEGPU_ERR_IO;
  }
}

thread_local std::string g_model_error;

}  // namespace

extern "C" int hegpu_model_parse(const char* json, hegpu_model** out) {
  if (!json || !out) return HEGPU_ERR_ARG;
  *out = nullptr;
  try {
    *out = parse_model(json).release();
    return HEGPU_OK;
  } catch (const Error& e) {
    g_model_error = e.what();
    return e.code;
  }
}

extern "C" int hegpu_model_load(const char* name_or_path, hegpu_model** out) {
  if (!name_or_path || !out) return HEGPU_ERR_ARG;
  *out = nullptr;
  try {
    const std::string name = name_or_path;
    std::string path;
    if (exists(name)) {
      path = name;
    } else if (const char* dir = std::getenv("HECNN_MODEL_DIR")) {
      for (const std::string& cand : {std::string(dir) + "/" + name, std::string(dir) + "/" + name + ".json"})
        if (path.empty() && exists(cand)) path = cand;
    }
    if (path.empty())
      io("model \"" + name + "\" is neither a file nor found under $HECNN_MODEL_DIR (the reference's builtins "
         "use AvgPool/SubConv stages outside this path)");
    *out = parse_model(read_file(path)).release();
    return HEGPU_OK;
  } catch (const Error& e) {
    g_model_error = e.what();
    return e.code;
  }
}

extern "C" const char* hegpu_model_last_error(const hegpu_model* m) {
  return m ? m->last_error.c_str() : g_model_error.c_str();
}

extern "C" void hegpu_model_destroy(hegpu_model* m) { delete m; }

extern "C" int hegpu_model_info(const hegpu_model* m, int* in_c, int* in_d, int* n_slots, int* n_layers,
                                size_t* weight_floats) {
  if (!m) return HEGPU_ERR_ARG;
  if (in_c) *in_c = m->in_c;
  if (in_d) *in_d = m->in_d;
  if (n_slots) *n_slots = m->n_slots;
  if (n_layers) *n_layers = (int)m->layers.size();
  if (weight_floats) *weight_floats = m->weight_count();
  return HEGPU_OK;
}

extern "C" int hegpu_model_set_default_policy(hegpu_model* m, int policy) {
  if (!m || policy < HEGPU_POLICY_HS || policy > HEGPU_POLICY_LOLA_STACKED) return HEGPU_ERR_ARG;
  m->default_policy = policy;
  return HEGPU_OK;
}

extern "C" int hegpu_model_set_n_slots(hegpu_model* m, int n_slots) {
  if (!m || n_slots < 1) return HEGPU_ERR_ARG;
  m->n_slots = n_slots;
  return HEGPU_OK;
}

extern "C" int hegpu_model_layer(const hegpu_model* m, int i, int* kind, int* k, int* s, int* out, int* groups,
                                 int* policy) {
  if (!m || i < 0 || i >= (int)m->layers.size()) return HEGPU_ERR_RANGE;
  const ModelLayer& l = m->layers[i];
  if (kind) *kind = l.kind;
  if (k) *k = l.k;
  if (s) *s = l.s;
  if (out) *out = l.out;
  if (groups) *groups = l.groups;
  if (policy) *policy = l.policy;
  return HEGPU_OK;
}

extern "C" int hegpu_model_load_weights(hegpu_model* m, const char* path, double* out, size_t count) {
  if (!m || !path || !out) return HEGPU_ERR_ARG;
  return guarded_model(m, [&] {
    const size_t n = m->weight_count();
    if (count != n) fail(HEGPU_ERR_SHAPE, "weights: the model needs " + std::to_string(n) + " values");
    std::ifstream in(path, std::ios::binary);
    if (!in) io(std::string("cannot open ") + path);
    const auto v = read_f32(in, n, path);
    expect_end(in, path, "weights");
    std::copy(v.begin(), v.end(), out);
  });
}

extern "C" int hegpu_model_save_weights(hegpu_model* m, const char* path, const double* w, size_t count) {
  if (!m || !path || !w) return HEGPU_ERR_ARG;
  return guarded_model(m, [&] {
    if (count != m->weight_count()) fail(HEGPU_ERR_SHAPE, "weights: wrong value count");
    std::ofstream o(path, std::ios::binary);
    if (!o) io(std::string("cannot open ") + path + " for writing");
    for (size_t i = 0; i < count; ++i) {
      const float f = (float)w[i];
      o.write(reinterpret_cast<const char*>(&f), sizeof f);
    }
  });
}

extern "C" int hegpu_model_load_input(hegpu_model* m, const char* path, double* out) {
  if (!m || !path || !out) return HEGPU_ERR_ARG;
  return guarded_model(m, [&] {
    std::ifstream in(path, std::ios::binary);
    if (!in) io(std::string("cannot open ") + path);
    const auto v = read_f32(in, (size_t)m->in_c * m->in_d * m->in_d, path);
    expect_end(in, path, "input");
    std::copy(v.begin(), v.end(), out);
  });
}

extern "C" int hegpu_model_save_input(hegpu_model* m, const char* path, const double* x) {
  if (!m || !path || !x) return HEGPU_ERR_ARG;
  return guarded_model(m, [&] {
    std::ofstream o(path, std::ios::binary);
    if (!o) io(std::string("cannot open ") + path + " for writing");
    for (size_t i = 0; i < (size_t)m->in_c * m->in_d * m->in_d; ++i) {
      const float f = (float)x[i];
      o.write(reinterpret_cast<const char*>(&f), sizeof f);
    }
  });
}

namespace {

hegpu_net_spec spec_of(const Lowered& lw) {
  hegpu_net_spec s{};
  s.in_c = lw.in_c;
  s.in_d = lw.in_d;
  s.k = lw.k;
  s.stride = lw.stride;
  s.c_out = lw.c_out;
  s.n_dense = (int)lw.dense.size();
  for (int i = 0; i < s.n_dense; ++i) s.dense_out[i] = lw.dense[i].rows;
  return s;
}

}  // namespace

extern "C" int hegpu_model_net_spec(const hegpu_model* m, hegpu_net_spec* spec) {
  if (!m || !spec) return HEGPU_ERR_ARG;
  try {
    *spec = spec_of(lower_model(*m, nullptr, 0));
    return HEGPU_OK;
  } catch (const Error& e) {
    g_model_error = e.what();
    return e.code;
  }
}

extern "C" int hegpu_model_compose(hegpu_model* m, const double* weights, size_t count, int stage, double* M,
                                   double* b, int* rows, int* cols) {
  if (!m || !weights) return HEGPU_ERR_ARG;
  return guarded_model(m, [&] {
    const Lowered lw = lower_model(*m, weights, count);
    if (stage < 0 || stage >= (int)lw.dense.size()) fail(HEGPU_ERR_RANGE, "model_compose: no such linear stage");
    const LoweredDense& d = lw.dense[stage];
    if (rows) *rows = d.rows;
    if (cols) *cols = d.cols;
    if (M) std::copy(d.M.begin(), d.M.end(), M);
    if (b) std::copy(d.b.begin(), d.b.end(), b);
  });
}

extern "C" int hegpu_net_create_from_model(hegpu_ctx* ctx, hegpu_model* m, const char* weights_path,
                                           hegpu_net** out) {
  if (!ctx || !m || !weights_path || !out) return HEGPU_ERR_ARG;
  std::vector<double> w(m->weight_count());
  int rc = hegpu_model_load_weights(m, weights_path, w.data(), w.size());
  if (rc) return rc;
  Lowered lw;
  rc = guarded_model(m, [&] { lw = lower_model(*m, w.data(), w.size()); });
  if (rc) return rc;
  const hegpu_net_spec s = spec_of(lw);
  const double* dw[4] = {nullptr, nullptr, nullptr, nullptr};
  const double* db[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<std::string> labels;
  for (int i = 0; i < s.n_dense; ++i) {
    dw[i] = lw.dense[i].M.data();
    db[i] = lw.dense[i].b.data();
    labels.push_back(lw.dense[i].label);
  }
  rc = hegpu_net_create(ctx, &s, lw.conv_w.data(), lw.conv_b.data(), dw, db, out);
  if (rc == HEGPU_OK) net_set_labels(*out, lw.conv_label, labels);
  return rc;
}
