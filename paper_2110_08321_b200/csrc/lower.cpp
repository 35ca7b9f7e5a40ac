// lower.cpp -- lower() + compose_run for model files (SURVEY.md §8f next #2,
// proj/src/netcompile.cpp:106-278): a first conv-pack layer, then alternating
// Square stages and maximal LINEAR RUNS (conv / avgpool / flatten / dense
// layers) whose affine maps are composed on the host into one matrix + bias
// and executed as one Halevi-Shoup layer.  So the reference's builtin shapes
// (conv, square, avgpool, conv, avgpool, flatten, dense, square, dense) run on
// the same GPU net as the configs' conv, square, dense, square, dense.
// Outside this family (SubConv groups, a stand-alone conv-pack repack, LoLa
// policies) the model is rejected with HEGPU_ERR_SHAPE.
//
// Composition is dense FP64 in the reference's row orders:
//   conv_to_matrix  convlower.cpp:76-102   row (co, oy, ox), col (ci, y, x)
//   conv_bias_vector convlower.cpp:104-113
//   pool_to_matrix  convlower.cpp:115-139
//   fold            netcompile.cpp:234-244 (M <- L M, b <- L b + b_L)
#include <string>
#include <vector>

#include "core.hpp"
#include "hegpu.h"
#include "lower.hpp"

namespace hegpu {

namespace {

struct Affine {  // rows x cols, row-major
  int rows = 0, cols = 0;
  std::vector<double> M, b;
};

// apply a linear layer y = L x + c (given as a row -> (col, coeff) list and c)
// to the affine map so far
template <class RowTerms>
void fold(Affine& a, int out_rows, RowTerms&& terms, const std::vector<double>& c) {
  if (a.M.empty()) {  // shapes only
    a.rows = out_rows;
    return;
  }
  Affine n;
  n.rows = out_rows;
  n.cols = a.cols;
  n.M.assign((size_t)out_rows * a.cols, 0.0);
  n.b.assign(out_rows, 0.0);
  for (int r = 0; r < out_rows; ++r) {
    double* dst = n.M.data() + (size_t)r * a.cols;
    double bb = c.empty() ? 0.0 : c[r];
    terms(r, [&](int col, double coef) {
      const double* src = a.M.data() + (size_t)col * a.cols;
      for (int j = 0; j < a.cols; ++j) dst[j] += coef * src[j];
      bb += coef * a.b[col];
    });
    n.b[r] = bb;
  }
  a = std::move(n);
}

}  // namespace

std::pair<int, int> ModelDesc::shape_before(size_t idx) const {
  int c = in_c, d = in_d;
  for (size_t i = 0; i < idx && i < layers.size(); ++i) {
    const ModelLayer& l = layers[i];
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

size_t ModelDesc::weight_count() const {
  size_t n = 0;
  for (size_t i = 0; i < layers.size(); ++i) {
    const ModelLayer& l = layers[i];
    const auto s = shape_before(i);
    if (l.kind == HEGPU_LAYER_CONV) {
      n += (size_t)l.out * s.first * l.k * l.k + l.out;
    } else if (l.kind == HEGPU_LAYER_SUBCONV) {
      n += (size_t)l.groups * ((size_t)(l.out / l.groups) * (s.first / l.groups) * l.k * l.k + l.out / l.groups);
    } else if (l.kind == HEGPU_LAYER_DENSE) {
      n += (size_t)l.out * s.first * s.second * s.second + l.out;
    }
  }
  return n;
}

Lowered lower_model(const ModelDesc& m, const double* w, size_t wcount) {
  auto bad = [&](const std::string& why) {
    fail(HEGPU_ERR_SHAPE, "model \"" + m.name + "\" is outside the GPU path (" + why + ")");
  };
  const auto& L = m.layers;
  if (m.default_policy != HEGPU_POLICY_HS) bad("a non-HS default policy (the general driver runs it)");
  if (L.empty() || L[0].kind != HEGPU_LAYER_CONV) bad("the first layer must be a conv-pack conv");
  if (L[0].groups != 1 || (L[0].policy != -1 && L[0].policy != HEGPU_POLICY_CONVPACK))
    bad("the first conv must be a plain conv-pack layer");
  Lowered out;
  out.in_c = m.in_c;
  out.in_d = m.in_d;
  out.k = L[0].k;
  out.stride = L[0].s;
  out.c_out = L[0].out;
  out.conv_label = L[0].label.empty() ? "Conv1" : L[0].label;
  // weight stream offsets per layer (conv bank + bias, dense W + b)
  std::vector<size_t> off(L.size(), 0);
  {
    size_t o = 0;
    for (size_t i = 0; i < L.size(); ++i) {
      off[i] = o;
      const auto s = m.shape_before(i);
      if (L[i].kind == HEGPU_LAYER_CONV) o += (size_t)L[i].out * s.first * L[i].k * L[i].k + L[i].out;
      else if (L[i].kind == HEGPU_LAYER_SUBCONV) bad("SubConv groups (next #2, grouped merges)");
      else if (L[i].kind == HEGPU_LAYER_DENSE) o += (size_t)L[i].out * s.first * s.second * s.second + L[i].out;
    }
    if (w && o != wcount) fail(HEGPU_ERR_SHAPE, "weights: the model needs " + std::to_string(o) + " values");
  }
  if (w) {
    out.conv_w.assign(w + off[0], w + off[0] + (size_t)out.c_out * m.in_c * out.k * out.k);
    out.conv_b.assign(w + off[0] + out.conv_w.size(), w + off[0] + out.conv_w.size() + out.c_out);
  }
  size_t i = 1;
  int linear_n = 0;
  while (i < L.size()) {
    if (L[i].kind != HEGPU_LAYER_SQUARE) bad("layer " + std::to_string(i) + " must be a square");
    ++i;
    if (i >= L.size()) bad("a square must be followed by a linear run");
    // maximal linear run starting at i (netcompile.cpp:182-193)
    std::pair<int, int> shape = m.shape_before(i);
    Affine a;
    a.rows = a.cols = shape.first * shape.second * shape.second;
    if (w) {
      a.M.assign((size_t)a.rows * a.cols, 0.0);
      for (int r = 0; r < a.rows; ++r) a.M[(size_t)r * a.cols + r] = 1.0;
      a.b.assign(a.rows, 0.0);
    }
    std::string label;
    size_t j = i;
    for (; j < L.size() && L[j].kind != HEGPU_LAYER_SQUARE; ++j) {
      const ModelLayer& l = L[j];
      if (!l.label.empty()) label += (label.empty() ? "" : "-") + l.label;
      const int c = shape.first, d = shape.second;
      if (l.kind == HEGPU_LAYER_CONV) {
        if (l.policy == HEGPU_POLICY_CONVPACK) bad("a stand-alone conv-pack repack (RepackConv)");
        if (l.groups != 1) bad("grouped conv");
        const int k = l.k, s = l.s, co_n = l.out, dout = (d - k) / s + 1;
        if (k > d) bad("conv window larger than its input");
        const double* W = w ? w + off[j] : nullptr;
        std::vector<double> cb;
        if (W) {
          const double* bias = W + (size_t)co_n * c * k * k;
          cb.resize((size_t)co_n * dout * dout);
          for (int co = 0; co < co_n; ++co)
            for (int p = 0; p < dout * dout; ++p) cb[(size_t)co * dout * dout + p] = bias[co];
        }
        fold(a, co_n * dout * dout, [&](int r, auto&& emit) {
          const int co = r / (dout * dout), oy = (r / dout) % dout, ox = r % dout;
          for (int ci = 0; ci < c; ++ci)
            for (int ky = 0; ky < k; ++ky)
              for (int kx = 0; kx < k; ++kx)
                emit((ci * d + oy * s + ky) * d + ox * s + kx, W[((size_t)(co * c + ci) * k + ky) * k + kx]);
        }, cb);
        shape = {co_n, dout};
      } else if (l.kind == HEGPU_LAYER_AVGPOOL) {
        const int k = l.k, s = l.s, dout = (d - k) / s + 1;
        if (k > d) bad("pool window larger than its input");
        const double scale = 1.0 / (double)(k * k);
        fold(a, c * dout * dout, [&](int r, auto&& emit) {
          const int ci = r / (dout * dout), oy = (r / dout) % dout, ox = r % dout;
          for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx) emit((ci * d + oy * s + ky) * d + ox * s + kx, scale);
        }, {});
        shape = {c, dout};
      } else if (l.kind == HEGPU_LAYER_FLATTEN) {
        // layout unchanged
      } else if (l.kind == HEGPU_LAYER_DENSE) {
        if (l.policy != -1 && l.policy != HEGPU_POLICY_HS) bad("dense layers use the HS policy (LoLa is next #3)");
        const int n = c * d * d, mo = l.out;
        const double* W = w ? w + off[j] : nullptr;
        std::vector<double> db;
        if (W) db.assign(W + (size_t)mo * n, W + (size_t)mo * n + mo);
        fold(a, mo, [&](int r, auto&& emit) {
          for (int col = 0; col < n; ++col) emit(col, W[(size_t)r * n + col]);
        }, db);
        shape = {mo, 1};
      } else {
        bad("layer kind " + std::to_string(l.kind) + " inside a linear run");
      }
    }
    if (j == i) bad("empty linear run");
    if ((int)out.dense.size() >= 4) bad("at most 4 linear stages");
    ++linear_n;
    out.dense.push_back({label.empty() ? "Linear" + std::to_string(linear_n) : label, a.rows, a.cols, a.M, a.b});
    i = j;
  }
  if (out.dense.empty()) bad("no linear stage after the conv");
  return out;
}


// ------------------------------------------------ the general lowering -----
namespace {

bool is_linear_kind(int k) {
  return k == HEGPU_LAYER_CONV || k == HEGPU_LAYER_SUBCONV || k == HEGPU_LAYER_AVGPOOL ||
         k == HEGPU_LAYER_FLATTEN || k == HEGPU_LAYER_DENSE;
}
bool is_standalone_convpack(const ModelLayer& l) {  // netcompile.cpp:21-24
  return l.kind == HEGPU_LAYER_CONV && l.policy == HEGPU_POLICY_CONVPACK;
}

// netcompile.cpp:71-91
int lookahead_groups(const ModelDesc& m, size_t from) {
  const auto& L = m.layers;
  for (size_t j = from; j < L.size(); ++j) {
    if (L[j].kind == HEGPU_LAYER_SQUARE) continue;
    if (is_standalone_convpack(L[j])) return 1;
    if (L[j].kind == HEGPU_LAYER_SUBCONV) return L[j].groups;
    if (is_linear_kind(L[j].kind)) {
      for (size_t r = j; r < L.size() && is_linear_kind(L[r].kind) && !is_standalone_convpack(L[r]); ++r)
        if (L[r].kind == HEGPU_LAYER_SUBCONV) return L[r].groups;
      return 1;
    }
  }
  return 1;
}

}  // namespace

ProgShape prog_apply_layer(const ProgShape& s, const ModelLayer& l, const std::string& where) {
  ProgShape o = s;
  switch (l.kind) {
    case HEGPU_LAYER_CONV:
    case HEGPU_LAYER_SUBCONV:
      if (s.flat) fail(HEGPU_ERR_SHAPE, where + ": convolution after flatten");
      if (l.kind == HEGPU_LAYER_SUBCONV && (l.groups < 1 || s.c % l.groups != 0 || l.out % l.groups != 0))
        fail(HEGPU_ERR_SHAPE, where + ": channels not divisible into " + std::to_string(l.groups) + " groups");
      if (l.k < 1 || l.s < 1 || l.k > s.d) fail(HEGPU_ERR_SHAPE, where + ": window larger than its input");
      o.c = l.out;
      o.d = (s.d - l.k) / l.s + 1;
      break;
    case HEGPU_LAYER_AVGPOOL:
      if (s.flat) fail(HEGPU_ERR_SHAPE, where + ": pooling after flatten");
      if (l.k < 1 || l.s < 1 || l.k > s.d) fail(HEGPU_ERR_SHAPE, where + ": window larger than its input");
      o.d = (s.d - l.k) / l.s + 1;
      break;
    case HEGPU_LAYER_FLATTEN:
      o.flat = true;
      o.flat_len = s.size();
      break;
    case HEGPU_LAYER_DENSE:
      o.flat = true;
      o.flat_len = l.out;
      break;
    default:
      break;
  }
  return o;
}

std::vector<ProgStage> lower_program(const ModelDesc& m) {
  const auto& L = m.layers;
  const int N = m.n_slots;
  if (L.empty()) fail(HEGPU_ERR_SHAPE, "model has no layers");
  if (N <= 0 || (N & (N - 1))) fail(HEGPU_ERR_SHAPE, "n_slots must be a power of two");
  std::vector<ProgStage> out;
  ProgShape shape{m.in_c, m.in_d, false, 0};
  size_t idx = 0;
  int flat_n = 0, square_n = 0, linear_n = 0;
  bool maps_layout = false;
  if (L[0].kind == HEGPU_LAYER_CONV && (L[0].policy == -1 || L[0].policy == HEGPU_POLICY_CONVPACK)) {
    ProgStage st;
    st.kind = HEGPU_STAGE_CONVPACK;
    st.label = L[0].label.empty() ? "Conv1" : L[0].label;
    st.layer_idx = {0};
    const ProgShape next = prog_apply_layer(shape, L[0], st.label);
    if ((int64_t)next.d * next.d > N)
      fail(HEGPU_ERR_CAPACITY, st.label + ": d_out^2 = " + std::to_string(next.d * next.d) + " > n_slots = " +
                                   std::to_string(N));
    out.push_back(st);
    shape = next;
    maps_layout = true;
    idx = 1;
  }
  while (idx < L.size()) {
    const ModelLayer& l = L[idx];
    if (l.kind == HEGPU_LAYER_SQUARE) {
      if (maps_layout) {
        ProgStage mg;
        mg.kind = HEGPU_STAGE_MERGE;
        mg.label = "Flat" + std::to_string(++flat_n);
        mg.groups = lookahead_groups(m, idx + 1);
        if (shape.c % mg.groups != 0)
          fail(HEGPU_ERR_SHAPE, mg.label + ": " + std::to_string(shape.c) + " maps not divisible into " +
                                    std::to_string(mg.groups) + " groups");
        if ((int64_t)(shape.c / mg.groups) * shape.d * shape.d > N)
          fail(HEGPU_ERR_CAPACITY, mg.label + ": group footprint " +
                                       std::to_string((shape.c / mg.groups) * shape.d * shape.d) + " > n_slots = " +
                                       std::to_string(N));
        out.push_back(mg);
        maps_layout = false;
      }
      ProgStage sq;
      sq.kind = HEGPU_STAGE_SQUARE;
      sq.label = "Square" + std::to_string(++square_n);
      sq.layer_idx = {(int)idx};
      out.push_back(sq);
      ++idx;
      continue;
    }
    if (!is_linear_kind(l.kind)) fail(HEGPU_ERR_SHAPE, "unsupported layer kind at index " + std::to_string(idx));
    if (is_standalone_convpack(l)) {
      ProgStage st;
      st.kind = HEGPU_STAGE_REPACKCONV;
      st.label = l.label.empty() ? "Conv" + std::to_string(idx) : l.label;
      st.layer_idx = {(int)idx};
      out.push_back(st);
      shape = prog_apply_layer(shape, l, st.label);
      maps_layout = true;
      ++idx;
      continue;
    }
    ProgStage st;  // maximal fused linear run
    st.kind = HEGPU_STAGE_LINEAR;
    st.policy = m.default_policy;  // netcompile.cpp:178
    size_t j = idx;
    for (; j < L.size() && is_linear_kind(L[j].kind) && !is_standalone_convpack(L[j]); ++j) {
      st.layer_idx.push_back((int)j);
      if (L[j].kind == HEGPU_LAYER_SUBCONV) st.groups = L[j].groups;
      if (L[j].policy != -1) st.policy = L[j].policy;
      if (!L[j].label.empty()) st.label += (st.label.empty() ? "" : "-") + L[j].label;
    }
    ++linear_n;
    if (st.label.empty()) st.label = "Linear" + std::to_string(linear_n);
    if (st.groups > 1 && st.policy != HEGPU_POLICY_HS)
      fail(HEGPU_ERR_SHAPE, st.label + ": grouped stages require the HS kernel");
    if (maps_layout) {
      ProgStage mg;
      mg.kind = HEGPU_STAGE_MERGE;
      mg.label = "Flat" + std::to_string(++flat_n);
      mg.groups = st.groups;
      out.push_back(mg);
      maps_layout = false;
    }
    ProgShape run_shape = shape;
    for (int r : st.layer_idx) run_shape = prog_apply_layer(run_shape, L[r], st.label);
    const int mm = run_shape.size(), nn = shape.size();
    if (mm > N || nn > N)
      fail(HEGPU_ERR_CAPACITY, st.label + ": fused " + std::to_string(mm) + "x" + std::to_string(nn) +
                                   " exceeds n_slots = " + std::to_string(N));
    out.push_back(st);
    shape = run_shape;
    idx = j;
  }
  return out;
}

std::vector<size_t> weight_offsets(const ModelDesc& m) {
  std::vector<size_t> off(m.layers.size(), 0);
  size_t o = 0;
  for (size_t i = 0; i < m.layers.size(); ++i) {
    off[i] = o;
    const ModelLayer& l = m.layers[i];
    const auto s = m.shape_before(i);
    if (l.kind == HEGPU_LAYER_CONV) o += (size_t)l.out * s.first * l.k * l.k + l.out;
    else if (l.kind == HEGPU_LAYER_SUBCONV)
      o += (size_t)l.groups * ((size_t)(l.out / l.groups) * (s.first / l.groups) * l.k * l.k + l.out / l.groups);
    else if (l.kind == HEGPU_LAYER_DENSE) o += (size_t)l.out * s.first * s.second * s.second + l.out;
  }
  return off;
}

GroupAffine compose_group(const ModelDesc& m, const double* w, const std::vector<int>& idxs, int group,
                          int n_groups, ProgShape shape) {
  if (!w) fail(HEGPU_ERR_ARG, "compose_group: no weights");
  const std::vector<size_t> off = weight_offsets(m);
  int c = shape.c / n_groups, d = shape.d;
  const int n0 = shape.flat ? shape.flat_len : c * d * d;
  Affine a;
  a.rows = a.cols = n0;
  a.M.assign((size_t)n0 * n0, 0.0);
  for (int r = 0; r < n0; ++r) a.M[(size_t)r * n0 + r] = 1.0;
  a.b.assign(n0, 0.0);
  bool any = false;
  for (int li : idxs) {
    const ModelLayer& l = m.layers[li];
    if (l.kind == HEGPU_LAYER_CONV || l.kind == HEGPU_LAYER_SUBCONV) {
      const bool sub = l.kind == HEGPU_LAYER_SUBCONV;
      if (!sub && n_groups != 1) fail(HEGPU_ERR_SHAPE, "a plain conv inside a grouped linear run");
      if (sub && l.groups != n_groups) fail(HEGPU_ERR_SHAPE, "SubConv group count differs from the stage's");
      const int k = l.k, s = l.s, co_n = sub ? l.out / l.groups : l.out, dout = (d - k) / s + 1;
      const size_t bank = (size_t)co_n * c * k * k + co_n;
      const double* W = w + off[li] + (sub ? (size_t)group * bank : 0);
      const double* bias = W + (size_t)co_n * c * k * k;
      std::vector<double> cb((size_t)co_n * dout * dout);
      for (int co = 0; co < co_n; ++co)
        for (int p = 0; p < dout * dout; ++p) cb[(size_t)co * dout * dout + p] = bias[co];
      const int cc = c, dd = d;
      fold(a, co_n * dout * dout, [&](int r, auto&& emit) {
        const int co = r / (dout * dout), oy = (r / dout) % dout, ox = r % dout;
        for (int ci = 0; ci < cc; ++ci)
          for (int ky = 0; ky < k; ++ky)
            for (int kx = 0; kx < k; ++kx)
              emit((ci * dd + oy * s + ky) * dd + ox * s + kx, W[((size_t)(co * cc + ci) * k + ky) * k + kx]);
      }, cb);
      c = co_n;
      d = dout;
      any = true;
    } else if (l.kind == HEGPU_LAYER_AVGPOOL) {
      const int k = l.k, s = l.s, dout = (d - k) / s + 1;
      const double scale = 1.0 / (double)(k * k);
      const int dd = d;
      fold(a, c * dout * dout, [&](int r, auto&& emit) {
        const int ci = r / (dout * dout), oy = (r / dout) % dout, ox = r % dout;
        for (int ky = 0; ky < k; ++ky)
          for (int kx = 0; kx < k; ++kx) emit((ci * dd + oy * s + ky) * dd + ox * s + kx, scale);
      }, {});
      d = dout;
      any = true;
    } else if (l.kind == HEGPU_LAYER_FLATTEN) {
      // layout unchanged
    } else if (l.kind == HEGPU_LAYER_DENSE) {
      const int n = a.rows, mo = l.out;
      const double* W = w + off[li];
      std::vector<double> db(W + (size_t)mo * n, W + (size_t)mo * n + mo);
      fold(a, mo, [&](int r, auto&& emit) {
        for (int col = 0; col < n; ++col) emit(col, W[(size_t)r * n + col]);
      }, db);
      c = mo;
      d = 1;
      any = true;
    } else {
      fail(HEGPU_ERR_SHAPE, "non-linear layer inside a fused run");
    }
  }
  if (!any) fail(HEGPU_ERR_SHAPE, "empty linear run");
  GroupAffine g;
  g.rows = a.rows;
  g.cols = a.cols;
  g.M = std::move(a.M);
  g.b = std::move(a.b);
  return g;
}

}  // namespace hegpu
