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

}  // namespace hegpu
