// net.cu -- the stage driver: the reference's `execute` stage loop
// (proj/src/netcompile.cpp:291-446) for the hot-path model family
//   ConvPack "Conv1" -> Merge "Flat1" -> { Square "Square<i>", Linear(HS)
//   "Dense<i>" }*,
// i.e. the stage list lower() produces for Conv -> Square -> Dense -> ...
// (netcompile.cpp:106-213), run on a batch of B images in one pass.
//
// Level schedule: taps at level L; conv + rescale -> L-1;
// merge at L-1; every Square and every Dense consumes one prime.
// masked_prefix (netcompile.cpp:424) is elided: the next HS masks are zero
// beyond n (matvec.cpp:57-61) and logits are read from slots 0..m-1.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>

#include "handles.hpp"
#include "layers.hpp"
#include "lower.hpp"

using namespace hegpu;


struct hegpu_net {
  Context* c = nullptr;
  hegpu_net_spec spec{};
  int d_out = 0, w_used = 0, ntaps = 0, top = 0;
  // region packing of the fused first layer: `regions` taps share one tap
  // ciphertext (tap s in region s % regions of ciphertext s / regions), so
  // an image ships tap_cts = ceil(ntaps / regions) ciphertexts; after the
  // conv one hoisted rotation sum folds the regions onto region 0
  int regions = 1, tap_cts = 0;
  std::unique_ptr<HsPlan> region_sum;
  double tap_scale = 0, out_scale = 0;
  std::unique_ptr<ConvLayer> conv;
  // the conv weights as given (conv_w [c_out][ntaps], conv_b), kept for the
  // per-rank output-map slices of hegpu_net_run_split(layer = -1)
  std::vector<double> conv_w, conv_b;
  std::map<std::pair<int, int>, std::unique_ptr<ConvLayer>> conv_slices;
  std::vector<HsPlan> plans;
  std::vector<u64d*> bias;   // per dense layer, [level][N] Montgomery
  std::vector<double> bias_scale;
  // meter stage labels (execute's labels: ConvPack, Flat<i>, Square<i>, and
  // the linear runs' joined layer labels for nets built from model files)
  std::string conv_label = "Conv1";
  std::vector<std::string> dense_labels;
  // host-input pipeline (hegpu_net_run_host_compact): double-buffered
  // compact staging, a copy stream and its events
  uint8_t* stage[2] = {nullptr, nullptr};
  size_t stage_bytes = 0;
  int next_stage = 0;
  cudaStream_t copy = nullptr;
  cudaEvent_t freed[2] = {nullptr, nullptr};  // compute done reading stage[s]
  std::vector<cudaEvent_t> sub_events[2];     // per stage buffer, one per input sub-chunk
  // the compute side of a serving pass as a CUDA graph, per (buffers, shape,
  // staging buffer): one stream entry instead of ~900 launches, so the host
  // never blocks on a full launch queue and the next pass's uploads are
  // enqueued while this pass computes.  Replays re-apply the captured
  // metering.
  struct ServeGraph {
    const uint8_t* host;
    const uint64_t* out;
    int batch, chunk, cur, uses = 0;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<std::pair<std::string, std::array<int64_t, 5>>> meter;
    std::array<int64_t, 4> ks{};
    int64_t launches = 0;
  };
  std::vector<ServeGraph> serve_graphs;
  // hegpu_net_run on two streams: the batch's two halves (independent images)
  // enqueued on the engine stream and on `side`, so one half's partial last
  // wave and single-wave launches overlap the other half's kernels
  std::vector<cudaStream_t> side;
  std::vector<cudaEvent_t> join;
  cudaEvent_t fork = nullptr;
  // hegpu_net_run_split: dense layer `layer`'s HS accumulated over part
  // `part` of `nparts` diagonal ranges, partials combined by `reduce`
  struct Split {
    static constexpr int kNone = -1000;  // no split (HEGPU_SPLIT_* codes are >= -1 - n_dense)
    int layer = kNone, part = 0, nparts = 1;
    hegpu_reduce_fn reduce = nullptr;
    void* user = nullptr;
  } split;
  ~hegpu_net() {
    for (auto& p : plans) p.release();
    for (u64d* b : bias) cudaFree(b);
    for (int s = 0; s < 2; ++s) {
      if (stage[s]) cudaFree(stage[s]);
      if (freed[s]) cudaEventDestroy(freed[s]);
      for (cudaEvent_t e : sub_events[s]) cudaEventDestroy(e);
    }
    for (auto& g : serve_graphs) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      if (g.g) cudaGraphDestroy(g.g);
    }
    if (copy) cudaStreamDestroy(copy);
    for (cudaStream_t st : side) cudaStreamDestroy(st);
    for (cudaEvent_t ev : join) cudaEventDestroy(ev);
    if (fork) cudaEventDestroy(fork);
  }
};

namespace {

void need(bool ok, int code, const std::string& msg) {
  if (!ok) fail(code, msg);
}

template <typename F>
int guarded(Context* c, F&& f) {
  try {
    bind_device(c);
    f();
    return HEGPU_OK;
  } catch (const Error& e) {
    if (c) c->last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->last_error = e.what();
    return HEGPU_ERR_ARG;
  }
}

struct Scratch {
  Context& c;
  u64d* p;
  Scratch(Context& cc, size_t words) : c(cc), p(cc.alloc(words)) {}
  ~Scratch() { c.free(p); }
};

// Conv1: ConvPack (netcompile.cpp:321-331); maps [B][c_out] at top-1
void conv_meter(hegpu_net& net, int B) {
  Context& c = *net.c;
  const hegpu_net_spec& s = net.spec;
  c.meter.begin(net.conv_label);
  c.meter.bump(HEGPU_MUL_PC, (int64_t)B * net.ntaps * s.c_out);
  c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (net.ntaps - 1) * s.c_out);
  c.meter.bump(HEGPU_ADD_PC, (int64_t)B * s.c_out);
}

// out = sum_{r < regions} rot_left(x, r F): one ModUp, regions - 1 key inner
// products on the rotated digits, one ModDown (unit-mask HS plan)
void region_fold(hegpu_net& net, CtBatch& x) {
  if (net.regions <= 1) return;
  Context& c = *net.c;
  const int B = x.count, l = x.level, N = c.N();
  HsPlan& pl = *net.region_sum;
  u64d* acc = c.alloc((size_t)B * 2 * (l + 1) * N);
  u64d* cacc = c.alloc((size_t)B * 2 * l * N);
  u64d* tmpP = c.alloc((size_t)B * 2 * N);
  pl.accumulate(c, x, 0, (int)pl.diag.size(), acc, cacc);
  u64d* r = c.alloc((size_t)B * 2 * l * N);
  DropArgs f{};
  f.src = acc; f.src_b = 2L * (l + 1) * N; f.src_p = (long)(l + 1) * N; f.src_limbs = l + 1;
  f.dst = r; f.dst_b = 2L * l * N; f.dst_p = (long)l * N;
  f.pd = c.L(); f.nl = l;
  f.add = cacc; f.add_b = 2L * l * N; f.add_p = (long)l * N; f.add_mask = 3; f.shifts = nullptr;
  drop_last_limb(c, B, f, tmpP);
  CK(cudaMemcpyAsync(x.d, r, x.words() * 8, cudaMemcpyDeviceToDevice, c.stream));
  c.free(acc);
  c.free(cacc);
  c.free(tmpP);
  c.free(r);
}

void run_conv(hegpu_net& net, const CtBatch& taps, CtBatch& maps) {
  conv_meter(net, taps.count / net.tap_cts);
  net.conv->run(*net.c, taps, maps);
  region_fold(net, maps);
}

void run_after_conv(hegpu_net& net, const CtBatch& mb, CtBatch& out);
void run_dense(hegpu_net& net, CtBatch x, CtBatch& out, u64d* cur_p);
void run_first_split(hegpu_net& net, const CtBatch& taps, CtBatch& x);

void run_net_one(hegpu_net& net, const CtBatch& taps, CtBatch& out);

// HEGPU_NET_STREAMS=n (default 2): a batch of >= n * kMinPart images runs as
// n parts of independent images on n streams (fork / join events; inside a
// stream capture the side streams join the capture), so one part's partial
// last wave and its single-wave launches overlap the other parts' kernels.
// Measured on cfg 2 (64 images): 3.118 -> 2.996 ms per step with two parts;
// parts of 8 images (cfg 3 at batch 16) lose, hence the minimum.
constexpr int kMinPart = 32;
int net_streams() {
  static const int n = [] {
    const char* e = std::getenv("HEGPU_NET_STREAMS");
    return e ? std::max(1, std::min(8, atoi(e))) : 2;
  }();
  return n;
}
int net_min_part() {
  static const int n = [] {
    const char* e = std::getenv("HEGPU_NET_MINPART");
    return e ? std::max(1, atoi(e)) : kMinPart;
  }();
  return n;
}

void run_net(hegpu_net& net, const CtBatch& taps, CtBatch& out) {
  Context& c = *net.c;
  const int B = taps.count / net.tap_cts;
  const int parts = std::min(net_streams(), B / net_min_part());
  if (parts < 2 || net.split.layer != hegpu_net::Split::kNone || !c.ktimer_name.empty())
    return run_net_one(net, taps, out);
  while ((int)net.side.size() < parts - 1) {
    cudaStream_t st = nullptr;
    cudaEvent_t ev = nullptr;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    net.side.push_back(st);
    net.join.push_back(ev);
  }
  if (!net.fork) CK(cudaEventCreateWithFlags(&net.fork, cudaEventDisableTiming));
  cudaStream_t main = c.stream;
  CK(cudaEventRecord(net.fork, main));
  double scale = 0;
  for (int p = parts - 1; p >= 0; --p) {  // the side streams first, the engine stream last
    const int b0 = (int)((int64_t)B * p / parts), b1 = (int)((int64_t)B * (p + 1) / parts);
    CtBatch tp{&c, (b1 - b0) * net.tap_cts, taps.level, taps.scale, taps.d + (size_t)b0 * net.tap_cts * taps.stride()};
    CtBatch op{&c, b1 - b0, out.level, out.scale, out.d + (size_t)b0 * out.stride()};
    if (p > 0) {
      CK(cudaStreamWaitEvent(net.side[p - 1], net.fork, 0));
      c.stream = net.side[p - 1];
    } else {
      c.stream = main;
    }
    try {
      run_net_one(net, tp, op);
    } catch (...) {
      c.stream = main;
      throw;
    }
    if (p > 0) CK(cudaEventRecord(net.join[p - 1], net.side[p - 1]));
    scale = op.scale;
  }
  c.stream = main;
  for (int p = 1; p < parts; ++p) CK(cudaStreamWaitEvent(main, net.join[p - 1], 0));
  out.scale = scale;
}

void run_net_one(hegpu_net& net, const CtBatch& taps, CtBatch& out) {
  Context& c = *net.c;
  const int B = taps.count / net.tap_cts;
  const int sl = net.split.layer;
  if (sl != hegpu_net::Split::kNone && (sl == HEGPU_SPLIT_FIRST_LAYER || sl <= HEGPU_SPLIT_FIRST_AND_DENSE(0))) {
    Scratch cur(c, (size_t)B * 2 * (net.top - 1) * c.N());
    CtBatch x{&c, B, net.top - 1, 0, cur.p};
    run_first_split(net, taps, x);
    run_dense(net, x, out, cur.p);
    return;
  }
  const int mo = net.conv->out_per_image();
  Scratch maps(c, (size_t)B * mo * 2 * (net.top - 1) * c.N());
  CtBatch mb{&c, B * mo, net.top - 1, 0, maps.p};
  run_conv(net, taps, mb);
  run_after_conv(net, mb, out);
}

// config 3 across GPUs, the first layer: this rank's share
// lo .. hi-1 of the c_out output maps -- their conv-pack MAC + rescale and
// their merge rotations (map j rotated right by j d_out^2 into its slot
// range) -- accumulated as (extended-basis acc, Q-basis C); the caller's
// reduction sums every rank's share; every rank then reduces mod q and runs
// the one ModDown per image: the merged ciphertext, bit-identical to the
// single-GPU Conv1 + Flat1
void run_first_split(hegpu_net& net, const CtBatch& taps, CtBatch& x) {
  Context& c = *net.c;
  const hegpu_net_spec& s = net.spec;
  const auto& sp = net.split;
  const int B = x.count, N = c.N(), l = net.top - 1;
  const int lo = s.c_out * sp.part / sp.nparts, hi = s.c_out * (sp.part + 1) / sp.nparts, M = hi - lo;
  c.meter.begin(net.conv_label);
  c.meter.bump(HEGPU_MUL_PC, (int64_t)B * net.ntaps * M);
  c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (net.ntaps - 1) * M);
  c.meter.bump(HEGPU_ADD_PC, (int64_t)B * M);
  const size_t acc_w = (size_t)B * 2 * (l + 1) * N, c_w = (size_t)B * 2 * l * N;
  Scratch part(c, acc_w + c_w);
  u64d* acc = part.p;
  u64d* C = part.p + acc_w;
  if (M > 0) {
    auto key = std::make_pair(lo, hi);
    auto it = net.conv_slices.find(key);
    if (it == net.conv_slices.end()) {
      const double* w = net.conv_w.data() + (size_t)lo * net.ntaps;
      it = net.conv_slices
               .emplace(key, std::make_unique<ConvLayer>(c, net.ntaps, M, w, net.conv_b.data() + lo, net.w_used,
                                                         net.top, net.tap_scale))
               .first;
    }
    Scratch maps(c, (size_t)B * M * 2 * l * N);
    CtBatch mb{&c, B * M, l, 0, maps.p};
    it->second->run(c, taps, mb);
    c.meter.begin("Flat1");
    eval_merge_partial(c, mb, M, lo, net.w_used, acc, C);
    const int64_t rots = M - (lo == 0 ? 1 : 0);
    c.meter.bump(HEGPU_ROT, (int64_t)B * rots);
    c.meter.bump(HEGPU_ADD_CC, (int64_t)B * rots);
  } else {
    c.meter.begin("Flat1");
    CK(cudaMemsetAsync(part.p, 0, (acc_w + c_w) * 8, c.stream));
  }
  CK(cudaStreamSynchronize(c.stream));
  need(sp.reduce(part.p, acc_w + c_w, sp.user) == 0, HEGPU_ERR_CUDA,
       "net_run_split: the partial-sum reduction failed");
  if (sp.nparts > 1) {  // sums of nparts reduced residues
    launch_reduce_rows(c, acc, acc_w, l + 1, l);
    launch_reduce_rows(c, C, c_w, l, -1);
  }
  u64d* tmpP = c.alloc((size_t)B * 2 * N);
  DropArgs d{};
  d.src = acc; d.src_b = 2L * (l + 1) * N; d.src_p = (long)(l + 1) * N; d.src_limbs = l + 1;
  d.dst = x.d; d.dst_b = (long)x.stride(); d.dst_p = (long)l * N;
  d.pd = c.L(); d.nl = l;
  d.add = C; d.add_b = 2L * l * N; d.add_p = (long)l * N; d.add_mask = 3; d.shifts = nullptr;
  drop_last_limb(c, B, d, tmpP);
  c.free(tmpP);
  x.scale = taps.scale;
}

// Flat1 onwards, on the conv-layer maps
void run_after_conv(hegpu_net& net, const CtBatch& mb, CtBatch& out) {
  Context& c = *net.c;
  const hegpu_net_spec& s = net.spec;
  const int mo = net.conv->out_per_image(), B = mb.count / mo, N = c.N();
  const int l = mb.level;
  // Flat1: Merge (netcompile.cpp:332-347): c_out - 1 key-switched
  // rotations summed lazily with one ModDown per image (eval_merge).  With
  // the fused first layer the maps already sit at their merged offsets (one
  // ciphertext per image) and no key switch runs; the
  // stage meters the reference's HOPs either way
  c.meter.begin("Flat1");
  Scratch cur(c, (size_t)B * 2 * l * N);
  CtBatch x{&c, B, l, 0, cur.p};
  merge_maps(c, mb, mo, net.w_used, x);
  c.meter.bump(HEGPU_ROT, (int64_t)B * (s.c_out - 1));
  c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (s.c_out - 1));
  run_dense(net, x, out, cur.p);
}

// Square<i> / Dense<i> pairs on the merged ciphertexts x (level top - 1);
// cur_p is x's buffer, reused for the intermediate layer outputs
void run_dense(hegpu_net& net, CtBatch x, CtBatch& out, u64d* cur_p) {
  Context& c = *net.c;
  const hegpu_net_spec& s = net.spec;
  const int B = x.count, N = c.N();
  int l = x.level;
  struct { u64d* p; } cur{cur_p};
  Scratch nxt(c, (size_t)B * 2 * l * N);
  for (int i = 0; i < s.n_dense; ++i) {
    // Square<i> (netcompile.cpp:348-351)
    c.meter.begin("Square" + std::to_string(i + 1));
    CtBatch y{&c, B, l - 1, 0, nxt.p};
    square_layer(c, x, y);
    c.meter.bump(HEGPU_MUL_CC, B);
    --l;
    // Dense<i>: Linear / HS (netcompile.cpp:380-434)
    c.meter.begin(i < (int)net.dense_labels.size() ? net.dense_labels[i] : "Dense" + std::to_string(i + 1));
    HsPlan& pl = net.plans[i];
    const bool last = i + 1 == s.n_dense;
    CtBatch z{&c, B, l - 1, 0, last ? out.d : cur.p};
    const int64_t kept = (int64_t)pl.diag.size();
    int i_lo = 0, i_hi = (int)kept;
    const int sl = net.split.layer;
    const int split_dense = sl == hegpu_net::Split::kNone                 ? -1
                            : sl >= 0                                    ? sl
                            : sl <= HEGPU_SPLIT_FIRST_AND_DENSE(0)       ? -2 - sl
                                                                         : -1;
    if (split_dense == i) {
      // this rank's diagonal range; partial sums combined by the caller's
      // reduction (NCCL all-reduce), then one ModDown / rescale / folds
      const auto& sp = net.split;
      i_lo = (int)(kept * sp.part / sp.nparts);
      i_hi = (int)(kept * (sp.part + 1) / sp.nparts);
      const size_t words = pl.acc_words(B, N);
      Scratch acc(c, words);
      u64d* cacc = acc.p + (size_t)B * 2 * (l + 1) * N;
      pl.accumulate(c, y, i_lo, i_hi, acc.p, cacc);
      CK(cudaStreamSynchronize(c.stream));
      need(sp.reduce(acc.p, words, sp.user) == 0, HEGPU_ERR_CUDA, "net_run_split: the partial-sum reduction failed");
      pl.finish(c, B, y.scale, acc.p, cacc, sp.nparts, z);
    } else {
      pl.run(c, y, z);
    }
    int64_t rots = 0;
    for (int d = i_lo; d < i_hi; ++d) rots += pl.diag[d].right != 0;
    c.meter.bump(HEGPU_MUL_PC, B * (i_hi - i_lo));
    c.meter.bump(HEGPU_ROT, B * (rots + pl.folds));
    c.meter.bump(HEGPU_ADD_CC, B * ((i_lo == 0 && i_hi > 0 ? i_hi - i_lo - 1 : i_hi - i_lo) + pl.folds));
    // bias add(out, pack(b)) (netcompile.cpp:423)
    launch_add_plain(c, z.d, net.bias[i], 0, z.d, B, l - 1);
    c.meter.bump(HEGPU_ADD_PC, B);
    --l;
    x = z;
    if (last) out.scale = z.scale;
  }
}

}  // namespace

namespace hegpu {
void net_set_labels(hegpu_net* net, const std::string& conv, const std::vector<std::string>& dense) {
  net->conv_label = conv;
  net->dense_labels = dense;
}
}  // namespace hegpu

extern "C" int hegpu_net_create(hegpu_ctx* h, const hegpu_net_spec* spec, const double* conv_w,
                                const double* conv_b, const double* const* dense_w, const double* const* dense_b,
                                hegpu_net** out) {
  if (!h || !spec || !conv_w || !out || (spec->n_dense > 0 && (!dense_w || !dense_b))) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    const hegpu_net_spec& s = *spec;
    need(c.device >= 0 && c.stream, HEGPU_ERR_CUDA, "client-only context: the evaluator needs a CUDA device");
    need(s.n_dense >= 1 && s.n_dense <= 4, HEGPU_ERR_SHAPE, "net: 1..4 dense layers supported");
    need(s.first_layer == HEGPU_FIRST_LAYER_REFERENCE || s.first_layer == HEGPU_FIRST_LAYER_FUSED, HEGPU_ERR_ARG,
         "net: unknown first_layer");
    need(s.k >= 1 && s.stride >= 1 && s.k <= s.in_d, HEGPU_ERR_SHAPE, "net: window larger than input");
    auto net = std::make_unique<hegpu_net>();
    net->c = &c;
    net->spec = s;
    net->d_out = (s.in_d - s.k) / s.stride + 1;
    net->w_used = net->d_out * net->d_out;
    net->ntaps = s.k * s.k * s.in_c;
    net->top = c.L();
    const int S = c.S();
    // lower() capacity checks (netcompile.cpp:125-128, 147-152, 203-207)
    need(net->w_used <= S, HEGPU_ERR_CAPACITY,
         "Conv1: d_out^2 = " + std::to_string(net->w_used) + " > n_slots = " + std::to_string(S));
    need((int64_t)s.c_out * net->w_used <= S, HEGPU_ERR_CAPACITY,
         "Flat1: group footprint " + std::to_string(s.c_out * net->w_used) + " > n_slots = " + std::to_string(S));
    need(c.L() >= 2 + 2 * s.n_dense, HEGPU_ERR_CAPACITY, "net: Q chain too short for the level schedule");
    net->tap_scale = std::ldexp(1.0, 40);
    net->conv_w.assign(conv_w, conv_w + (size_t)s.c_out * net->ntaps);
    if (conv_b) net->conv_b.assign(conv_b, conv_b + s.c_out);
    else net->conv_b.assign(s.c_out, 0.0);
    net->conv = std::make_unique<ConvLayer>(c, net->ntaps, s.c_out, conv_w, conv_b, net->w_used, net->top,
                                            net->tap_scale);
    std::vector<int64_t> rots;
    const int F = s.c_out * net->w_used;
    if (s.first_layer == HEGPU_FIRST_LAYER_FUSED) {
      // Conv1 + Flat1 fused, taps packed `regions` per ciphertext
      net->regions = std::max(1, std::min(net->ntaps, S / F));
      net->conv->make_merged(c, conv_w, conv_b, net->w_used, net->tap_scale, net->regions);
    } else {
      // the reference's stages: conv_pack taps (one window per ciphertext),
      // conv_packed_forward + rescale -> c_out maps, merge_maps with the
      // right rotations j * d_out^2, j = 1 .. c_out - 1 (convlower.cpp:145-160)
      net->regions = 1;
      for (int j = 1; j < s.c_out; ++j) rots.push_back((int64_t)j * net->w_used % S);
    }
    net->tap_cts = (net->ntaps + net->regions - 1) / net->regions;
    if (net->regions > 1) {
      std::vector<int64_t> rr{0};
      for (int r = 1; r < net->regions; ++r) rr.push_back((S - (int64_t)r * F % S) % S);
      std::sort(rr.begin(), rr.end());
      net->region_sum = std::make_unique<HsPlan>();
      net->region_sum->build_rotsum(c, rr, net->top - 1);
      for (int64_t r : rr)
        if (r) rots.push_back(r);
    }
    double scale = net->tap_scale;  // after conv + rescale
    int l = net->top - 1;
    int n = s.c_out * net->w_used;
    net->plans.resize(s.n_dense);
    for (int i = 0; i < s.n_dense; ++i) {
      scale = scale * scale / (double)c.P->q(l - 1);  // square + rescale
      --l;
      const int m = s.dense_out[i];
      try {
        net->plans[i].build(c, dense_w[i], m, n, l, true);
      } catch (const Error& e) {
        fail(e.code, "Dense" + std::to_string(i + 1) + ": " + e.what());
      }
      for (int64_t r : net->plans[i].right_rotations()) rots.push_back(r);
      --l;  // HS rescale; bias at the same scale
      std::vector<double> bz(dense_b[i], dense_b[i] + m);
      std::vector<u64> wire((size_t)l * c.N());
      c.client->encode(bz.data(), m, scale, l, false, wire.data());
      u64d* d = nullptr;
      CK(cudaMalloc((void**)&d, wire.size() * 8));
      u64d* stage = c.alloc(wire.size());
      CK(cudaMemcpyAsync(stage, wire.data(), wire.size() * 8, cudaMemcpyHostToDevice, c.stream));
      launch_wire_to_slot(c, stage, d, (size_t)l, 1, l, -1);
      c.free(stage);
      net->bias.push_back(d);
      net->bias_scale.push_back(scale);
      n = m;
    }
    net->out_scale = scale;
    CK(cudaStreamSynchronize(c.stream));
    if (int rc = hegpu_gen_rotation_keys(h, rots.data(), (int)rots.size())) fail(rc, c.last_error);
    if (int rc = hegpu_gen_relin_key(h)) fail(rc, c.last_error);
    *out = net.release();
  });
}

extern "C" void hegpu_net_destroy(hegpu_net* net) {
  if (!net) return;
  try { bind_device(net->c); } catch (...) {}
  cudaStreamSynchronize(net->c->stream);
  delete net;
}

extern "C" int hegpu_net_run(hegpu_net* net, const hegpu_ct* taps, hegpu_ct* out) {
  if (!net || !taps || !out) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    need(taps->b.level == net->top && taps->b.count % net->tap_cts == 0, HEGPU_ERR_SHAPE,
         "net_run: taps must be B * tap_cts ciphertexts at the top level");
    const int B = taps->b.count / net->tap_cts;
    need(out->b.count == B && out->b.level == net->top - 1 - 2 * net->spec.n_dense, HEGPU_ERR_SHAPE,
         "net_run: bad output handle");
    CtBatch o = out->b;
    run_net(*net, taps->b, o);
    out->b.scale = o.scale;
  });
}

extern "C" int hegpu_net_run_split(hegpu_net* net, const hegpu_ct* taps, hegpu_ct* out, int layer, int part,
                                   int nparts, hegpu_reduce_fn reduce, void* user) {
  if (!net || !taps || !out || !reduce) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    need(layer > hegpu_net::Split::kNone, HEGPU_ERR_RANGE, "net_run_split: no such layer");
    const bool first = layer == HEGPU_SPLIT_FIRST_LAYER || layer <= HEGPU_SPLIT_FIRST_AND_DENSE(0);
    const int dense = layer >= 0 ? layer : layer <= HEGPU_SPLIT_FIRST_AND_DENSE(0) ? -2 - layer : -1;
    need(first || dense >= 0, HEGPU_ERR_RANGE, "net_run_split: no such layer");
    need(dense < net->spec.n_dense, HEGPU_ERR_RANGE, "net_run_split: no such dense layer");
    need(!first || net->spec.first_layer == HEGPU_FIRST_LAYER_REFERENCE, HEGPU_ERR_ARG,
         "net_run_split: the first-layer split needs the reference first layer (per-map conv + merge)");
    need(nparts >= 1 && nparts <= 8 && part >= 0 && part < nparts, HEGPU_ERR_RANGE, "net_run_split: bad part");
    need(taps->b.level == net->top && taps->b.count % net->tap_cts == 0, HEGPU_ERR_SHAPE,
         "net_run_split: taps must be B * tap_cts ciphertexts at the top level");
    const int B = taps->b.count / net->tap_cts;
    need(out->b.count == B && out->b.level == net->top - 1 - 2 * net->spec.n_dense, HEGPU_ERR_SHAPE,
         "net_run_split: bad output handle");
    net->split = {layer, part, nparts, reduce, user};
    CtBatch o = out->b;
    try {
      run_net(*net, taps->b, o);
    } catch (...) {
      net->split = {};
      throw;
    }
    net->split = {};
    out->b.scale = o.scale;
  });
}

extern "C" int hegpu_net_run_compact(hegpu_net* net, const void* dev_taps, int batch, hegpu_ct* out) {
  if (!net || !dev_taps || !out || batch < 1) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    need(out->b.count == batch && out->b.level == net->top - 1 - 2 * net->spec.n_dense, HEGPU_ERR_SHAPE,
         "net_run_compact: bad output handle");
    const int L = net->top, N = c.N();
    const int mo = net->conv->out_per_image();
    Scratch prod(c, (size_t)batch * mo * 2 * L * N);
    Scratch maps(c, (size_t)batch * mo * 2 * (L - 1) * N);
    CtBatch pb{&c, batch * mo, L, 0, prod.p};
    conv_meter(*net, batch);
    net->conv->mac_compact(c, static_cast<const uint8_t*>(dev_taps), batch, net->tap_scale, pb);
    CtBatch mb{&c, batch * mo, L - 1, 0, maps.p};
    eval_rescale(c, pb, mb);
    mb.scale = net->tap_scale;
    region_fold(*net, mb);
    CtBatch o = out->b;
    run_after_conv(*net, mb, o);
    out->b.scale = o.scale;
  });
}

extern "C" int hegpu_net_run_host(hegpu_net* net, const uint64_t* host_taps, int batch, uint64_t* host_out) {
  if (!net || !host_taps || !host_out || batch < 1) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    const int N = c.N(), L = net->top, lo = net->top - 1 - 2 * net->spec.n_dense;
    const size_t in_words = (size_t)batch * net->tap_cts * 2 * L * N;
    const size_t out_words = (size_t)batch * 2 * lo * N;
    Scratch stage(c, in_words);
    Scratch taps(c, in_words);
    CK(cudaMemcpyAsync(stage.p, host_taps, in_words * 8, cudaMemcpyHostToDevice, c.stream));
    launch_wire_to_slot(c, stage.p, taps.p, (size_t)batch * net->tap_cts * 2 * L, 0, L, -1);
    CtBatch tb{&c, batch * net->tap_cts, L, net->tap_scale, taps.p};
    Scratch o(c, out_words);
    CtBatch ob{&c, batch, lo, 0, o.p};
    run_net(*net, tb, ob);
    launch_slot_to_wire(c, o.p, stage.p, (size_t)batch * 2 * lo, 0, lo, -1);
    CK(cudaMemcpyAsync(host_out, stage.p, out_words * 8, cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
  });
}

extern "C" size_t hegpu_net_compact_image_bytes(const hegpu_net* net) {
  return net ? (size_t)net->tap_cts * net->c->client->compact_bytes(net->top) : 0;
}

#ifndef HEGPU_NET_SUBCHUNK
#define HEGPU_NET_SUBCHUNK 16  // images per upload sub-chunk (expand + conv MAC granularity)
#endif

namespace {

void serve_compute(hegpu_net& n, const uint8_t* stage, int cur, int batch, int chunk, uint64_t* host_out);

// enqueue one host-input pass (no host synchronisation): the staging buffer
// alternates between calls so call k+1's uploads overlap call k's compute
void enqueue_host_compact(hegpu_net& n, const uint8_t* host, int batch, int chunk, uint64_t* host_out) {
  Context& c = *n.c;
  const int N = c.N(), L = n.top, lo = n.top - 1 - 2 * n.spec.n_dense;
  // two-level pipeline: the copy stream streams every image's compact taps
  // in sub-chunks of c1 images; the compute stream expands + convolves each
  // sub-chunk as soon as it lands, and runs merge..Dense on chunks of c2.
  const int c2 = chunk > 0 ? std::min(chunk, batch) : std::min(batch, 32);
  const int c1 = std::min(c2, HEGPU_NET_SUBCHUNK);
  const size_t per_img = hegpu_net_compact_image_bytes(&n);
  const size_t out_words = (size_t)2 * lo * N;
  const size_t map_words = (size_t)2 * (L - 1) * N;
  if (n.stage_bytes < per_img * batch) {
    CK(cudaDeviceSynchronize());
    for (int s = 0; s < 2; ++s) {
      if (n.stage[s]) cudaFree(n.stage[s]);
      n.stage[s] = nullptr;
      CK(cudaMalloc((void**)&n.stage[s], per_img * batch));
    }
    n.stage_bytes = per_img * batch;
  }
  if (!n.copy) {
    CK(cudaStreamCreateWithFlags(&n.copy, cudaStreamNonBlocking));
    for (int s = 0; s < 2; ++s) CK(cudaEventCreateWithFlags(&n.freed[s], cudaEventDisableTiming));
  }
  const int cur = n.next_stage;
  n.next_stage ^= 1;
  uint8_t* stage = n.stage[cur];
  const int nsub = (batch + c1 - 1) / c1;
  auto& subs = n.sub_events[cur];
  while ((int)subs.size() < nsub) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    subs.push_back(e);
  }
  // this staging buffer is free once the call that used it last has expanded
  CK(cudaStreamWaitEvent(n.copy, n.freed[cur], 0));
  for (int j = 0; j < nsub; ++j) {
    const int b0 = j * c1, nb = std::min(c1, batch - b0);
#ifndef HEGPU_DIAG_NO_H2D  // diagnostics build only: compute path without the uploads
    CK(cudaMemcpyAsync(stage + (size_t)b0 * per_img, host + (size_t)b0 * per_img, per_img * nb,
                       cudaMemcpyHostToDevice, n.copy));
#endif
    CK(cudaEventRecord(subs[j], n.copy));
  }
  serve_compute(n, stage, cur, batch, chunk, host_out);
}

// compute side of one serving pass on the engine stream (captured into a
// CUDA graph from the second use of the same buffers on)
void compute_pass(hegpu_net& n, const uint8_t* stage, int cur, int batch, int chunk, uint64_t* host_out,
                  bool captured) {
  Context& c = *n.c;
  const int N = c.N(), L = n.top, lo = n.top - 1 - 2 * n.spec.n_dense;
  const int c2 = chunk > 0 ? std::min(chunk, batch) : std::min(batch, 32);
  const int c1 = std::min(c2, HEGPU_NET_SUBCHUNK);
  const size_t per_img = hegpu_net_compact_image_bytes(&n);
  const size_t out_words = (size_t)2 * lo * N;
  const size_t map_words = (size_t)2 * (L - 1) * N;
  const auto& subs = n.sub_events[cur];
  // each sub-chunk is multiply-accumulated straight from its compact bytes
  // as it lands; the conv rescale runs once per chunk (full-width NTT grids)
  const int mo = n.conv->out_per_image();
  Scratch prod(c, (size_t)c2 * mo * 2 * L * N);
  Scratch maps(c, (size_t)c2 * mo * map_words);
  Scratch o(c, (size_t)c2 * out_words);
  Scratch wire(c, (size_t)c2 * out_words);
  for (int m0 = 0; m0 < batch; m0 += c2) {
    const int nm = std::min(c2, batch - m0);
    CtBatch pb{&c, nm * mo, L, 0, prod.p};
    for (int b0 = m0; b0 < m0 + nm; b0 += c1) {
      const int nb = std::min(c1, m0 + nm - b0);
      CK(cudaStreamWaitEvent(c.stream, subs[b0 / c1], captured ? cudaEventWaitExternal : 0));
      CtBatch sb{&c, nb * mo, L, 0, prod.p + (size_t)(b0 - m0) * mo * 2 * L * N};
      n.conv->mac_compact(c, stage + (size_t)b0 * per_img, nb, n.tap_scale, sb);
      pb.scale = sb.scale;
    }
    if (m0 + nm >= batch) {  // last read of the staging buffer
      if (captured) CK(cudaEventRecordWithFlags(n.freed[cur], c.stream, cudaEventRecordExternal));
      else CK(cudaEventRecord(n.freed[cur], c.stream));
    }
    conv_meter(n, nm);
    CtBatch rb{&c, nm * mo, L - 1, 0, maps.p};
    eval_rescale(c, pb, rb);
    rb.scale = n.tap_scale;
    region_fold(n, rb);
    CtBatch mb{&c, nm * mo, L - 1, n.tap_scale, maps.p};
    CtBatch ob{&c, nm, lo, 0, o.p};
    run_after_conv(n, mb, ob);
    launch_slot_to_wire(c, o.p, wire.p, (size_t)nm * 2 * lo, 0, lo, -1);
    CK(cudaMemcpyAsync(host_out + (size_t)m0 * out_words, wire.p, (size_t)nm * out_words * 8,
                       cudaMemcpyDeviceToHost, c.stream));
  }
}

void serve_compute(hegpu_net& n, const uint8_t* stage, int cur, int batch, int chunk, uint64_t* host_out) {
  Context& c = *n.c;
  static const bool graphs = [] {
    const char* e = std::getenv("HEGPU_SERVE_GRAPHS");
    return !(e && e[0] == '0');
  }();
  if (!graphs) return compute_pass(n, stage, cur, batch, chunk, host_out, false);
  hegpu_net::ServeGraph* sg = nullptr;
  for (auto& g : n.serve_graphs)
    if (g.host == stage && g.out == host_out && g.batch == batch && g.chunk == chunk && g.cur == cur) sg = &g;
  if (!sg) {
    if (n.serve_graphs.size() >= 16) {  // bounded cache: drop the oldest
      auto& old = n.serve_graphs.front();
      CK(cudaStreamSynchronize(c.stream));
      if (old.exec) cudaGraphExecDestroy(old.exec);
      if (old.g) cudaGraphDestroy(old.g);
      n.serve_graphs.erase(n.serve_graphs.begin());
    }
    n.serve_graphs.push_back({stage, host_out, batch, chunk, cur});
    sg = &n.serve_graphs.back();
  }
  if (sg->exec) {
    for (const auto& st : sg->meter) {
      c.meter.begin(st.first);
      for (int f = 0; f < 5; ++f) c.meter.bump(f, st.second[f]);
    }
    c.launches += sg->launches;
    for (int k = 0; k < 4; ++k) c.ks[k] += sg->ks[k];
    CK(cudaGraphLaunch(sg->exec, c.stream));
    return;
  }
  if (sg->uses++ == 0) return compute_pass(n, stage, cur, batch, chunk, host_out, false);  // warm-up pass
  const auto before = c.meter.stages;
  const auto ks0 = c.ks;
  const int64_t l0 = c.launches;
  CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  try {
    compute_pass(n, stage, cur, batch, chunk, host_out, true);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c.stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CK(cudaStreamEndCapture(c.stream, &sg->g));
  CK(cudaGraphInstantiate(&sg->exec, sg->g, 0));
  for (const auto& st : c.meter.stages) {
    std::array<int64_t, 5> d = st.second;
    for (const auto& b : before)
      if (b.first == st.first)
        for (int f = 0; f < 5; ++f) d[f] -= b.second[f];
    sg->meter.emplace_back(st.first, d);
  }
  sg->launches = c.launches - l0;
  for (int k = 0; k < 4; ++k) sg->ks[k] = c.ks[k] - ks0[k];
  CK(cudaGraphLaunch(sg->exec, c.stream));
}

}  // namespace

extern "C" int hegpu_net_run_host_compact(hegpu_net* net, const uint8_t* host, int batch, int chunk,
                                          uint64_t* host_out) {
  if (!net || !host || !host_out || batch < 1) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    enqueue_host_compact(*net, host, batch, chunk, host_out);
    CK(cudaStreamSynchronize(c.stream));
  });
}

extern "C" int hegpu_net_submit_host_compact(hegpu_net* net, const uint8_t* host, int batch, int chunk,
                                             uint64_t* host_out) {
  if (!net || !host || !host_out || batch < 1) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] { enqueue_host_compact(*net, host, batch, chunk, host_out); });
}

extern "C" int hegpu_net_wait(hegpu_net* net) {
  if (!net) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] { CK(cudaStreamSynchronize(c.stream)); });
}

namespace {
// the client's input packing (conv_pack, convlower.cpp:9-37, tap t =
// (ci*k+ky)*k+kx, slot oy*d_out+ox) in the fused first layer's form: tap
// ciphertext g holds taps g*R .. g*R+R-1, tap s's window replicated at the
// c_out map offsets of its region s % R (R = net.regions)
template <class Emit>
void pack_image_taps(hegpu_net& net, const double* image, Emit&& emit) {
  Context& c = *net.c;
  const hegpu_net_spec& s = net.spec;
  const int d = net.d_out, w = net.w_used, L = net.top, R = net.regions;
  const int reps = net.conv->merged ? s.c_out : 1;
  const size_t F = (size_t)reps * w;
  std::vector<double> win((size_t)net.ntaps * w);
  for (int ci = 0; ci < s.in_c; ++ci)
    for (int ky = 0; ky < s.k; ++ky)
      for (int kx = 0; kx < s.k; ++kx) {
        const int t = (ci * s.k + ky) * s.k + kx;
        for (int oy = 0; oy < d; ++oy)
          for (int ox = 0; ox < d; ++ox)
            win[(size_t)t * w + oy * d + ox] =
                image[((size_t)ci * s.in_d + oy * s.stride + ky) * s.in_d + ox * s.stride + kx];
      }
  std::vector<double> z((size_t)R * F);
  std::vector<u64> pt((size_t)L * c.N());
  for (int g = 0; g < net.tap_cts; ++g) {
    std::fill(z.begin(), z.end(), 0.0);
    int used = 0;
    for (int r = 0; r < R && g * R + r < net.ntaps; ++r, ++used)
      for (int co = 0; co < reps; ++co)
        std::copy_n(win.data() + (size_t)(g * R + r) * w, w, z.data() + (size_t)r * F + (size_t)co * w);
    c.client->encode(z.data(), (int)((size_t)used * F), net.tap_scale, L, false, pt.data());
    emit(g, pt.data());
  }
}
}  // namespace

extern "C" int hegpu_net_encrypt_image_compact(hegpu_net* net, const double* image, uint64_t nonce,
                                               uint8_t* taps_out) {
  if (!net || !image || !taps_out) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    const int L = net->top;
    const size_t per = c.client->compact_bytes(L);
    // same packing + encode as hegpu_net_encrypt_image, same nonces: the
    // compact taps expand to exactly those ciphertexts
    pack_image_taps(*net, image, [&](int g, const u64* pt) {
      c.client->encrypt_compact(pt, L, nonce * (uint64_t)net->tap_cts + (uint64_t)g, taps_out + (size_t)g * per);
    });
  });
}

extern "C" int hegpu_net_encrypt_image(hegpu_net* net, const double* image, uint64_t nonce, uint64_t* taps_out) {
  if (!net || !image || !taps_out) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    const int N = c.N(), L = net->top;
    pack_image_taps(*net, image, [&](int g, const u64* pt) {
      c.client->encrypt(pt, L, nonce * (uint64_t)net->tap_cts + (uint64_t)g, taps_out + (size_t)g * 2 * L * N);
    });
  });
}

extern "C" int hegpu_net_tap_cts(const hegpu_net* net) { return net ? net->tap_cts : -1; }
extern "C" int hegpu_net_first_layer(const hegpu_net* net) { return net ? net->spec.first_layer : -1; }

extern "C" int hegpu_net_decrypt_logits(hegpu_net* net, const uint64_t* out_ct, double* logits) {
  if (!net || !out_ct || !logits) return HEGPU_ERR_ARG;
  Context& c = *net->c;
  return guarded(&c, [&] {
    const int N = c.N(), lo = net->top - 1 - 2 * net->spec.n_dense;
    std::vector<u64> pt((size_t)lo * N);
    std::vector<double> slots(c.S());
    c.client->decrypt(out_ct, lo, pt.data());
    c.client->decode(pt.data(), lo, net->out_scale, slots.data());
    std::memcpy(logits, slots.data(), sizeof(double) * net->spec.dense_out[net->spec.n_dense - 1]);
  });
}

extern "C" double hegpu_net_output_scale(const hegpu_net* net) { return net ? net->out_scale : 0.0; }
