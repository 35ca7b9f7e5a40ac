// lower.hpp -- host-side model description and its lowering to the GPU net
// (lower.cpp, modelio.cpp).
#pragma once
#include <cstddef>
#include <string>
#include <utility>
#include <vector>

struct hegpu_net;

namespace hegpu {

struct ModelLayer {
  int kind = 0, k = 0, s = 1, out = 0, groups = 1, policy = -1;  // HEGPU_LAYER_* / HEGPU_POLICY_* (-1 none)
  std::string label;
};

struct ModelDesc {
  std::string name;
  int in_c = 0, in_d = 0, n_slots = 0;
  std::vector<ModelLayer> layers;
  std::pair<int, int> shape_before(size_t idx) const;  // (channels, side) entering layer idx
  size_t weight_count() const;                         // float32 values in the weights stream
};

struct LoweredDense {
  std::string label;
  int rows = 0, cols = 0;
  std::vector<double> M, b;  // rows x cols row-major, rows
};

struct Lowered {
  int in_c = 0, in_d = 0, k = 0, stride = 1, c_out = 0;
  std::string conv_label;
  std::vector<double> conv_w, conv_b;
  std::vector<LoweredDense> dense;  // one per Square + linear run
};

// w: the flat weights stream (wcount values) or nullptr for shapes only
Lowered lower_model(const ModelDesc& m, const double* w, size_t wcount);

// stage labels of a net built from a model (net.cu)
void net_set_labels(hegpu_net* net, const std::string& conv, const std::vector<std::string>& dense);

}  // namespace hegpu
