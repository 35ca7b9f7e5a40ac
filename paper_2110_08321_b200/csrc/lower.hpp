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
  int default_policy = 1;  // HEGPU_POLICY_HS: linear stages without a per-layer policy (netcompile.hpp:33-35)
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

// ---- the general lowering (program.cpp): every stage kind of the
// reference's lower() (proj/src/netcompile.cpp:106-213) ----------------------
struct ProgShape {  // ShapeState, netcompile.cpp:26-32
  int c = 0, d = 0;
  bool flat = false;
  int flat_len = 0;
  int size() const { return flat ? flat_len : c * d * d; }
};
ProgShape prog_apply_layer(const ProgShape& s, const ModelLayer& l, const std::string& where);

struct ProgStage {  // Stage, netcompile.hpp:57-63
  int kind = 0;  // HEGPU_STAGE_*
  std::string label;
  std::vector<int> layer_idx;
  int groups = 1;
  int policy = 1;  // HEGPU_POLICY_HS
};
std::vector<ProgStage> lower_program(const ModelDesc& m);

// offset of every layer's values in the flat weights stream (modelio.cpp:169-202)
std::vector<size_t> weight_offsets(const ModelDesc& m);

struct GroupAffine {
  int rows = 0, cols = 0;
  std::vector<double> M, b;  // rows x cols row-major, rows
};
// compose_run (netcompile.cpp:225-278): the affine map of the linear run
// `idxs` restricted to channel group `group` of `n_groups`; `shape` is the
// run's (ungrouped) input shape
GroupAffine compose_group(const ModelDesc& m, const double* w, const std::vector<int>& idxs, int group,
                          int n_groups, ProgShape shape);

}  // namespace hegpu

// the C-ABI model handle (modelio.cpp parses it, program.cpp lowers it)
struct hegpu_model : hegpu::ModelDesc {
  std::string last_error;
};

namespace hegpu {

// stage labels of a net built from a model (net.cu)
void net_set_labels(hegpu_net* net, const std::string& conv, const std::vector<std::string>& dense);

}  // namespace hegpu
