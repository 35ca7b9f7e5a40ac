// program.cpp -- the reference's general stage driver on the CKKS engine:
// lower() (proj/src/netcompile.cpp:106-213) + execute() (:291-446) for every
// stage kind -- ConvPack, Merge into channel groups, Square, RepackConv and
// grouped Linear runs (SubConv) under the HS or LoLa-dense policy -- written
// as host C++ over the C-ABI operators (include/hegpu.h), the way the
// reference's execute() calls its free functions: each stage runs under
// hegpu_begin_stage(label) and the operators meter themselves, so the HOP
// report is the reference's by construction.
//
// Level / scale schedule: input at the top level, scale 2^40;
// ConvPack, RepackConv and Linear(HS) multiply by plaintexts at scale
// q_{l-1} and rescale (scale unchanged, one prime); Square: s^2 / q_{l-1};
// Linear(LoLa-dense): two primes.  masked_prefix (netcompile.cpp:424) is
// elided as in net.cu: every consumer's plaintexts are zero beyond the valid
// prefix (HS masks, LoLa rows, the RepackConv's masked constants).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "core.hpp"
#include "hegpu.h"
#include "lower.hpp"

using namespace hegpu;

namespace {

struct CtH {  // RAII ciphertext handle
  hegpu_ct* p = nullptr;
  CtH() = default;
  explicit CtH(hegpu_ct* q) : p(q) {}
  CtH(const CtH&) = delete;
  CtH& operator=(const CtH&) = delete;
  CtH(CtH&& o) noexcept : p(o.p) { o.p = nullptr; }
  CtH& operator=(CtH&& o) noexcept {
    if (this != &o) {
      hegpu_ct_destroy(p);
      p = o.p;
      o.p = nullptr;
    }
    return *this;
  }
  ~CtH() { hegpu_ct_destroy(p); }
};

struct StagePlan {
  int level_in = 0, level_out = 0, n_in = 0, n_out = 0;
  double scale_in = 0, scale_out = 0;
  ProgShape shape_in, shape_out;
  bool maps_in = false;
  // ConvPack
  hegpu_conv_plan* conv = nullptr;
  // RepackConv: the masked-constant conv over every map (hegpu_masked_conv)
  hegpu_masked_conv* repack = nullptr;
  // Linear, per group
  std::vector<hegpu_hs_plan*> hs;
  std::vector<hegpu_lola_plan*> lola;
  std::vector<hegpu_pt*> bias;
  int rows = 0;
};

}  // namespace

struct hegpu_prog {
  hegpu_ctx* h = nullptr;
  ModelDesc model;
  std::vector<ProgStage> stages;
  std::vector<StagePlan> plans;
  int N = 0, S = 0, top = 0, input_cts = 1, out_level = 0, n_logits = 0;
  double in_scale = 0, out_scale = 0;
  bool conv_first = false;
  std::string last_error;
  ~hegpu_prog() {
    for (auto& p : plans) {
      hegpu_conv_plan_destroy(p.conv);
      hegpu_masked_conv_destroy(p.repack);
      for (auto* x : p.hs) hegpu_hs_plan_destroy(x);
      for (auto* x : p.lola) hegpu_lola_plan_destroy(x);
      for (auto* x : p.bias) hegpu_pt_destroy(x);
    }
  }
};

namespace {

// C-ABI status -> exception carrying the context's message
void ok(hegpu_ctx* h, int rc, const char* what) {
  if (rc == HEGPU_OK) return;
  const char* e = hegpu_last_error(h);
  fail(rc, std::string(what) + ": " + (e ? e : ""));
}

CtH make_ct(hegpu_ctx* h, int count, int level) {
  hegpu_ct* p = nullptr;
  ok(h, hegpu_ct_create(h, count, level, &p), "ct_create");
  return CtH(p);
}

// pack(values on slots [0, len), n_slots, Plaintext) encoded at `scale`, uploaded
hegpu_pt* make_pt(hegpu_ctx* h, const double* z, int len, double scale, int level, int N) {
  std::vector<uint64_t> wire((size_t)level * N);
  ok(h, hegpu_encode(h, z, len, scale, level, 0, wire.data()), "encode");
  hegpu_pt* p = nullptr;
  ok(h, hegpu_pt_create(h, 1, level, 0, &p), "pt_create");
  const int rc = hegpu_pt_upload(p, wire.data(), wire.size(), scale);
  if (rc != HEGPU_OK) {
    hegpu_pt_destroy(p);
    ok(h, rc, "pt_upload");
  }
  return p;
}

template <typename F>
int guarded_prog(hegpu_prog* p, F&& f) {
  try {
    f();
    return HEGPU_OK;
  } catch (const Error& e) {
    if (p) p->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (p) p->last_error = e.what();
    return HEGPU_ERR_ARG;
  }
}

thread_local std::string g_prog_error;

void build(hegpu_prog& P, const double* w, size_t count) {
  hegpu_ctx* h = P.h;
  const ModelDesc& m = P.model;
  int n = 0, S = 0, nq = 0;
  ok(h, hegpu_ctx_info(h, &n, &S, &nq, nullptr), "ctx_info");
  P.N = n;
  P.S = S;
  P.top = nq;
  if (m.n_slots != S)
    fail(HEGPU_ERR_SHAPE, "model n_slots = " + std::to_string(m.n_slots) + " but the context has " +
                              std::to_string(S) + " slots");
  if (count != m.weight_count())
    fail(HEGPU_ERR_SHAPE, "weights: the model needs " + std::to_string(m.weight_count()) + " values");
  P.stages = lower_program(m);
  // primes consumed
  int depth = 0;
  for (const auto& st : P.stages) {
    if (st.kind == HEGPU_STAGE_LINEAR) {
      if (st.policy == HEGPU_POLICY_LOLA_STACKED)
        fail(HEGPU_ERR_SHAPE, st.label + ": the LoLa-stacked policy de-interleaves on cleartext values in the "
                                         "reference (netcompile.cpp:409-417); not an encrypted stage");
      if (st.policy == HEGPU_POLICY_CONVPACK) fail(HEGPU_ERR_SHAPE, st.label + ": ConvPack is not a matrix-vector kernel");
      depth += st.policy == HEGPU_POLICY_LOLA_DENSE ? 2 : 1;
    } else if (st.kind != HEGPU_STAGE_MERGE) {
      depth += 1;
    }
  }
  if (P.top < depth + 1)
    fail(HEGPU_ERR_CAPACITY, "program: the Q chain has " + std::to_string(P.top) + " primes, the stages consume " +
                                 std::to_string(depth) + " and the output needs one");
  std::vector<uint64_t> primes(nq + 4);  // Q chain, then P
  ok(h, hegpu_ctx_info(h, nullptr, nullptr, nullptr, primes.data()), "ctx_info");
  const std::vector<size_t> off = weight_offsets(m);
  std::vector<int64_t> rots;
  bool any_square = false;
  int l = P.top, ncts = 1;
  double scale = std::ldexp(1.0, 40);
  P.in_scale = scale;
  ProgShape shape{m.in_c, m.in_d, false, 0};
  bool maps = false;
  P.conv_first = !P.stages.empty() && P.stages[0].kind == HEGPU_STAGE_CONVPACK;
  if (!P.conv_first && shape.size() > S)
    fail(HEGPU_ERR_CAPACITY, "input of " + std::to_string(shape.size()) + " values exceeds n_slots");
  P.plans.resize(P.stages.size());
  for (size_t si = 0; si < P.stages.size(); ++si) {
    const ProgStage& st = P.stages[si];
    StagePlan& pl = P.plans[si];
    pl.level_in = l;
    pl.scale_in = scale;
    pl.shape_in = shape;
    pl.maps_in = maps;
    pl.n_in = ncts;
    switch (st.kind) {
      case HEGPU_STAGE_CONVPACK: {
        const ModelLayer& ly = m.layers[st.layer_idx[0]];
        const ProgShape next = prog_apply_layer(shape, ly, st.label);
        const int ntaps = ly.k * ly.k * shape.c, w_used = next.d * next.d;
        const double* W = w + off[st.layer_idx[0]];
        ok(h, hegpu_conv_plan_create(h, ntaps, W, ly.out, W + (size_t)ly.out * ntaps, w_used, l, scale, &pl.conv),
           st.label.c_str());
        P.input_cts = ntaps;
        ncts = ly.out;
        --l;
        maps = true;
        shape = next;
        break;
      }
      case HEGPU_STAGE_MERGE: {
        const int G = st.groups, per = shape.c / G;
        const int64_t wd = (int64_t)shape.d * shape.d;
        if ((int64_t)per * wd > S)
          fail(HEGPU_ERR_CAPACITY, st.label + ": group footprint " + std::to_string(per * wd) + " > n_slots = " +
                                       std::to_string(S));
        for (int j = 1; j < per; ++j) rots.push_back(j * wd % S);
        ncts = G;
        maps = false;
        break;
      }
      case HEGPU_STAGE_SQUARE:
        any_square = true;
        scale = scale * scale / (double)primes[l - 1];
        --l;
        break;
      case HEGPU_STAGE_REPACKCONV: {
        const ModelLayer& ly = m.layers[st.layer_idx[0]];
        if (ly.k != 1)
          fail(HEGPU_ERR_SHAPE, st.label + ": only 1x1 convolutions support the packed rotation lowering");
        const int c_in = shape.c, wd = shape.d * shape.d, c_out = ly.out;
        if (!maps) {
          const int per = c_in / ncts;
          for (int j = 1; j < per; ++j) rots.push_back((S - (int64_t)j * wd % S) % S);  // rotate_left(j w)
        }
        const double* W = w + off[st.layer_idx[0]];
        ok(h, hegpu_masked_conv_create(h, c_in, W, c_out, W + (size_t)c_out * c_in, wd, l, scale, &pl.repack),
           st.label.c_str());
        shape = prog_apply_layer(shape, ly, st.label);
        ncts = c_out;
        --l;
        maps = true;
        break;
      }
      case HEGPU_STAGE_LINEAR: {
        const int G = st.groups;
        if (ncts != G)
          fail(HEGPU_ERR_LAYOUT, st.label + ": expected " + std::to_string(G) + " input ciphertexts, have " +
                                     std::to_string(ncts));
        const int lo = st.policy == HEGPU_POLICY_LOLA_DENSE ? l - 2 : l - 1;
        for (int g = 0; g < G; ++g) {
          const GroupAffine a = compose_group(m, w, st.layer_idx, g, G, shape);
          pl.rows = a.rows;
          int rc;
          if (st.policy == HEGPU_POLICY_HS) {
            hegpu_hs_plan* hp = nullptr;
            rc = hegpu_hs_plan_create(h, a.M.data(), a.rows, a.cols, l, 1, &hp);
            if (rc != HEGPU_OK) fail(rc, st.label + ": " + hegpu_last_error(h));
            pl.hs.push_back(hp);
            const int nr = hegpu_hs_plan_rotations(hp, nullptr, 0);
            std::vector<int64_t> r(nr > 0 ? nr : 0);
            if (nr > 0) hegpu_hs_plan_rotations(hp, r.data(), nr);
            rots.insert(rots.end(), r.begin(), r.end());
          } else {
            hegpu_lola_plan* lp = nullptr;
            rc = hegpu_lola_plan_create(h, HEGPU_LOLA_DENSE, a.M.data(), a.rows, a.cols, l, &lp);
            if (rc != HEGPU_OK) fail(rc, st.label + ": " + hegpu_last_error(h));
            pl.lola.push_back(lp);
            const int nr = hegpu_lola_plan_rotations(lp, nullptr, 0);
            std::vector<int64_t> r(nr > 0 ? nr : 0);
            if (nr > 0) hegpu_lola_plan_rotations(lp, r.data(), nr);
            rots.insert(rots.end(), r.begin(), r.end());
            for (int j = 1; j < a.rows; ++j) rots.push_back(j);  // merge_maps(rows, 1)
          }
          pl.bias.push_back(make_pt(h, a.b.data(), a.rows, scale, lo, P.N));
        }
        for (int r : st.layer_idx) shape = prog_apply_layer(shape, m.layers[r], st.label);
        l = lo;
        maps = false;
        break;
      }
      default:
        fail(HEGPU_ERR_ARG, "program: unknown stage kind");
    }
    pl.level_out = l;
    pl.scale_out = scale;
    pl.shape_out = shape;
    pl.n_out = ncts;
  }
  if (ncts != 1) fail(HEGPU_ERR_LAYOUT, "program must end in a single output ciphertext");
  P.out_level = l;
  P.out_scale = scale;
  P.n_logits = shape.size();
  std::vector<int64_t> nz;
  for (int64_t r : rots)
    if (r % S) nz.push_back(r % S);
  if (!nz.empty()) ok(h, hegpu_gen_rotation_keys(h, nz.data(), (int)nz.size()), "gen_rotation_keys");
  if (any_square) ok(h, hegpu_gen_relin_key(h), "gen_relin_key");
}

// One pass over a batch of B images.  Layouts of the intermediate batch:
// ConvPack leaves maps image-major [b][map]; every other stage keeps its
// ciphertexts UNIT-MAJOR [unit][b] (unit = channel group after a Merge /
// Linear stage, map after a RepackConv), so the B ciphertexts a stage
// operator works on are contiguous and run as one batched C-ABI call (the
// grouped HS stages take the tensor-core kernel from B = 8 on).
void run(hegpu_prog& P, hegpu_ct* input, hegpu_ct* out) {
  hegpu_ctx* h = P.h;
  int cnt = 0, lvl = 0;
  ok(h, hegpu_ct_info(input, &cnt, &lvl, nullptr), "ct_info");
  if (cnt < P.input_cts || cnt % P.input_cts != 0 || lvl != P.top)
    fail(HEGPU_ERR_SHAPE, "prog_run: input must be B x " + std::to_string(P.input_cts) +
                              " ciphertexts at the top level");
  const int B = cnt / P.input_cts;
  ok(h, hegpu_ct_info(out, &cnt, &lvl, nullptr), "ct_info");
  if (cnt != B || lvl != P.out_level) fail(HEGPU_ERR_SHAPE, "prog_run: the output handle must hold B ciphertexts at the output level");
  ok(h, hegpu_ct_set_scale(input, P.in_scale), "ct_set_scale");
  CtH cur;              // owned intermediate batch (empty while the state is the caller's input)
  hegpu_ct* x = input;  // current state: pl.n_in units x B ciphertexts at pl.level_in
  bool image_major = true;  // [b][unit] (the input taps, ConvPack's maps) vs [unit][b]
  auto sub = [&](hegpu_ct* src, int first, int count) {
    hegpu_ct* v = nullptr;
    ok(h, hegpu_ct_view(src, first, count, &v), "ct_view");
    return CtH(v);
  };
  // HEGPU_PROG_TIMING=1: synchronise after every stage and print its wall time (diagnostics)
  static const bool timing = [] {
    const char* e = std::getenv("HEGPU_PROG_TIMING");
    return e && e[0] == '1';
  }();
  auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  for (size_t si = 0; si < P.stages.size(); ++si) {
    const ProgStage& st = P.stages[si];
    const StagePlan& pl = P.plans[si];
    ok(h, hegpu_begin_stage(h, st.label.c_str()), "begin_stage");
    const double t_stage = timing ? (hegpu_sync(h), now()) : 0.0;
    CtH nxt;
    bool nxt_image_major = false;
    switch (st.kind) {
      case HEGPU_STAGE_CONVPACK: {
        nxt = make_ct(h, B * pl.n_out, pl.level_out);
        ok(h, hegpu_conv_plan_run(h, pl.conv, x, nxt.p), st.label.c_str());
        nxt_image_major = true;
        break;
      }
      case HEGPU_STAGE_MERGE: {
        // per group: its maps of every image gathered image-major [b][j]
        // (one strided copy per image), then ONE batched merge_maps over the
        // B images into the group's B contiguous outputs
        const int G = st.groups, C = pl.shape_in.c, per = C / G;
        const int64_t wd = (int64_t)pl.shape_in.d * pl.shape_in.d;
        nxt = make_ct(h, G * B, pl.level_out);
        // at most ~256 maps per merge call (its ModUp digits are (per - 1) l (l + 1) limbs per image)
        const int bc = std::max(1, std::min(B, 256 / std::max(1, per)));
        CtH gather = make_ct(h, bc * per, pl.level_in);
        for (int g = 0; g < G; ++g)
          for (int b0 = 0; b0 < B; b0 += bc) {
            const int nb = std::min(bc, B - b0);
            for (int b = b0; b < b0 + nb; ++b) {
              if (image_major)  // [b][c] -> maps g*per .. of image b
                ok(h, hegpu_ct_gather(gather.p, (b - b0) * per, x, b * C + g * per, 1, per), "ct_gather");
              else              // [c][b] -> the same maps, stride B
                ok(h, hegpu_ct_gather(gather.p, (b - b0) * per, x, g * per * B + b, B, per), "ct_gather");
            }
            ok(h, hegpu_ct_set_scale(gather.p, pl.scale_in), "ct_set_scale");
            CtH gv = sub(gather.p, 0, nb * per), og = sub(nxt.p, g * B + b0, nb);
            ok(h, hegpu_merge_maps(h, gv.p, per, wd, og.p), st.label.c_str());
          }
        break;
      }
      case HEGPU_STAGE_SQUARE: {
        nxt = make_ct(h, B * pl.n_in, pl.level_out);
        ok(h, hegpu_square(h, x, nxt.p), st.label.c_str());
        nxt_image_major = image_major;
        break;
      }
      case HEGPU_STAGE_REPACKCONV: {
        const int c_in = pl.shape_in.c, c_out = pl.n_out, l = pl.level_in;
        const int64_t wd = (int64_t)pl.shape_in.d * pl.shape_in.d;
        // taps, tap-major [t][b]: the maps themselves, or rotate_left(group
        // ct, j w) (netcompile.cpp:366-373; one batched rotation per (g, j))
        CtH rot;
        hegpu_ct* taps = x;
        if (pl.maps_in && image_major) {  // ConvPack maps [b][t] -> [t][b]
          rot = make_ct(h, c_in * B, l);
          for (int b = 0; b < B; ++b)
            for (int t = 0; t < c_in; ++t) {
              CtH src = sub(x, b * c_in + t, 1), dst = sub(rot.p, t * B + b, 1);
              ok(h, hegpu_ct_copy(dst.p, src.p), "ct_copy");
            }
          taps = rot.p;
        } else if (!pl.maps_in) {
          const int G = pl.n_in, per = c_in / G;
          rot = make_ct(h, c_in * B, l);
          for (int g = 0; g < G; ++g) {
            CtH sg = sub(x, g * B, B);
            for (int j = 0; j < per; ++j) {
              CtH dst = sub(rot.p, (g * per + j) * B, B);
              ok(h, hegpu_rotate_left(h, sg.p, (int64_t)j * wd % P.S, dst.p), st.label.c_str());
            }
          }
          taps = rot.p;
        }
        // the masked-constant MAC over every map, the masked bias and the
        // rescale in one operator (maps map-major [co][b])
        ok(h, hegpu_ct_set_scale(taps, pl.scale_in), "ct_set_scale");
        nxt = make_ct(h, c_out * B, pl.level_out);
        ok(h, hegpu_masked_conv_run(h, pl.repack, taps, nxt.p), st.label.c_str());
        break;
      }
      case HEGPU_STAGE_LINEAR: {
        const int G = st.groups;
        nxt = make_ct(h, G * B, pl.level_out);
        for (int g = 0; g < G; ++g) {
          CtH ig = sub(x, g * B, B), og = sub(nxt.p, g * B, B);
          ok(h, hegpu_ct_set_scale(ig.p, pl.scale_in), "ct_set_scale");
          if (st.policy == HEGPU_POLICY_HS) {
            ok(h, hegpu_hs_matvec(h, pl.hs[g], ig.p, og.p), st.label.c_str());
          } else {  // lola_dense_matvec rows [b][row], then merge_maps(rows, 1) (netcompile.cpp:402-405)
            CtH rows = make_ct(h, B * pl.rows, pl.level_out);
            ok(h, hegpu_lola_matvec(h, pl.lola[g], ig.p, rows.p), st.label.c_str());
            ok(h, hegpu_merge_maps(h, rows.p, pl.rows, 1, og.p), st.label.c_str());
          }
          ok(h, hegpu_add_plain(h, og.p, pl.bias[g], og.p), st.label.c_str());  // netcompile.cpp:423
        }
        break;
      }
    }
    ok(h, hegpu_ct_set_scale(nxt.p, pl.scale_out), "ct_set_scale");
    if (timing) {
      hegpu_sync(h);
      std::fprintf(stderr, "prog stage %-14s B=%d  %.3f ms\n", st.label.c_str(), B, (now() - t_stage) * 1e3);
    }
    cur = std::move(nxt);
    x = cur.p;
    image_major = nxt_image_major;
  }
  ok(h, hegpu_ct_copy(out, x), "ct_copy");
  ok(h, hegpu_sync(h), "sync");
}

}  // namespace

extern "C" int hegpu_prog_create(hegpu_ctx* ctx, const hegpu_model* model, const double* weights, size_t count,
                                 hegpu_prog** out) {
  if (!ctx || !model || !weights || !out) return HEGPU_ERR_ARG;
  *out = nullptr;
  auto p = std::make_unique<hegpu_prog>();
  p->h = ctx;
  p->model = *model;
  try {
    build(*p, weights, count);
  } catch (const Error& e) {
    g_prog_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_prog_error = e.what();
    return HEGPU_ERR_ARG;
  }
  *out = p.release();
  return HEGPU_OK;
}

extern "C" const char* hegpu_prog_last_error(const hegpu_prog* p) {
  return p ? p->last_error.c_str() : g_prog_error.c_str();
}

extern "C" void hegpu_prog_destroy(hegpu_prog* p) { delete p; }

extern "C" int hegpu_prog_info(const hegpu_prog* p, int* n_stages, int* input_cts, int* out_level, int* n_logits) {
  if (!p) return HEGPU_ERR_ARG;
  if (n_stages) *n_stages = (int)p->stages.size();
  if (input_cts) *input_cts = p->input_cts;
  if (out_level) *out_level = p->out_level;
  if (n_logits) *n_logits = p->n_logits;
  return HEGPU_OK;
}

static void copy_label(const std::string& s, char* dst, int len) {
  if (!dst || len <= 0) return;
  std::strncpy(dst, s.c_str(), (size_t)len - 1);
  dst[len - 1] = 0;
}

extern "C" int hegpu_prog_stage(const hegpu_prog* p, int i, char* label, int label_len, int* kind, int* groups,
                                int* policy) {
  if (!p || i < 0 || i >= (int)p->stages.size()) return HEGPU_ERR_RANGE;
  const ProgStage& st = p->stages[i];
  copy_label(st.label, label, label_len);
  if (kind) *kind = st.kind;
  if (groups) *groups = st.groups;
  if (policy) *policy = st.policy;
  return HEGPU_OK;
}

extern "C" int hegpu_model_lower(const hegpu_model* model, int cap, char (*labels)[64], int* kinds, int* groups,
                                 int* policies) {
  if (!model) return -HEGPU_ERR_ARG;
  try {
    const std::vector<ProgStage> st = lower_program(*model);
    for (int i = 0; i < (int)st.size() && i < cap; ++i) {
      if (labels) copy_label(st[i].label, labels[i], 64);
      if (kinds) kinds[i] = st[i].kind;
      if (groups) groups[i] = st[i].groups;
      if (policies) policies[i] = st[i].policy;
    }
    return (int)st.size();
  } catch (const Error& e) {
    g_prog_error = e.what();
    return -e.code;
  }
}

extern "C" int hegpu_prog_encrypt_input(hegpu_prog* p, const double* image, uint64_t nonce, uint64_t* cts_out) {
  if (!p || !image || !cts_out) return HEGPU_ERR_ARG;
  return guarded_prog(p, [&] {
    hegpu_ctx* h = p->h;
    const ModelDesc& m = p->model;
    const int L = p->top, N = p->N;
    std::vector<uint64_t> pt((size_t)L * N);
    if (!p->conv_first) {  // the flattened input as one dense ciphertext (netcompile.cpp:309-319)
      ok(h, hegpu_encode(h, image, m.in_c * m.in_d * m.in_d, p->in_scale, L, 0, pt.data()), "encode");
      ok(h, hegpu_encrypt(h, pt.data(), L, nonce, cts_out), "encrypt");
      return;
    }
    // conv_pack (convlower.cpp:9-37): tap t = (ci k + ky) k + kx, slot oy d_out + ox
    const ModelLayer& ly = m.layers[0];
    const int k = ly.k, s = ly.s, d = (m.in_d - k) / s + 1, w = d * d;
    std::vector<double> win(w);
    for (int ci = 0; ci < m.in_c; ++ci)
      for (int ky = 0; ky < k; ++ky)
        for (int kx = 0; kx < k; ++kx) {
          const int t = (ci * k + ky) * k + kx;
          for (int oy = 0; oy < d; ++oy)
            for (int ox = 0; ox < d; ++ox)
              win[oy * d + ox] = image[((size_t)ci * m.in_d + oy * s + ky) * m.in_d + ox * s + kx];
          ok(h, hegpu_encode(h, win.data(), w, p->in_scale, L, 0, pt.data()), "encode");
          ok(h, hegpu_encrypt(h, pt.data(), L, nonce * (uint64_t)p->input_cts + (uint64_t)t,
                              cts_out + (size_t)t * 2 * L * N),
             "encrypt");
        }
  });
}

extern "C" int hegpu_prog_run(hegpu_prog* p, hegpu_ct* input, hegpu_ct* out) {
  if (!p || !input || !out) return HEGPU_ERR_ARG;
  return guarded_prog(p, [&] { run(*p, input, out); });
}

extern "C" int hegpu_prog_decrypt_logits(hegpu_prog* p, const uint64_t* out_ct, double* logits) {
  if (!p || !out_ct || !logits) return HEGPU_ERR_ARG;
  return guarded_prog(p, [&] {
    hegpu_ctx* h = p->h;
    const int lo = p->out_level;
    std::vector<uint64_t> pt((size_t)lo * p->N);
    std::vector<double> slots(p->S);
    ok(h, hegpu_decrypt(h, out_ct, lo, pt.data()), "decrypt");
    ok(h, hegpu_decode(h, pt.data(), lo, p->out_scale, slots.data()), "decode");
    std::memcpy(logits, slots.data(), sizeof(double) * p->n_logits);
  });
}

extern "C" double hegpu_prog_output_scale(const hegpu_prog* p) { return p ? p->out_scale : 0.0; }
