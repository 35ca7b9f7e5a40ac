// capi.cu -- the C-ABI of include/hegpu.h: handles, metering, error
// translation, host<->device conversion and the evaluator / layer entry
// points.  No CPU fallback exists: every evaluator call runs CUDA kernels
// and fails with HEGPU_ERR_CUDA when no device is present.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "engine.hpp"
#include "handles.hpp"
#include "layers.hpp"

using namespace hegpu;


namespace hegpu {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(HEGPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void Meter::begin(const std::string& label) {
  for (size_t i = 0; i < stages.size(); ++i)
    if (stages[i].first == label) { cur = (int)i; return; }
  stages.emplace_back(label, std::array<int64_t, 5>{});
  cur = (int)stages.size() - 1;
}

void Meter::bump(int field, int64_t n) {
  total[field] += n;
  if (cur >= 0) stages[cur].second[field] += n;
}

u64d* Context::alloc(size_t words) {
  void* p = nullptr;
  if (!words) words = 1;
  CK(cudaMallocAsync(&p, words * 8, stream));
  return (u64d*)p;
}

void Context::free(u64d* p) {
  if (p) CK(cudaFreeAsync(p, stream));
}

const DeviceKey& Context::rot_key(int shift) {
  auto it = rot_keys.find(shift);
  if (it == rot_keys.end())
    fail(HEGPU_ERR_KEY, "no Galois key for a left rotation by " + std::to_string(shift) + " slots");
  return it->second;
}

}  // namespace hegpu

namespace {

thread_local std::string g_create_error;

template <typename F>
int guarded(Context* c, F&& f) {
  try {
    bind_device(c);
    f();
    return HEGPU_OK;
  } catch (const Error& e) {
    if (c) c->last_error = e.what();
    else g_create_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (c) c->last_error = e.what();
    else g_create_error = e.what();
    return HEGPU_ERR_ARG;
  }
}

void need(bool ok, int code, const std::string& msg) {
  if (!ok) fail(code, msg);
}

void need_gpu(const Context& c) {
  need(c.device >= 0 && c.stream, HEGPU_ERR_CUDA, "client-only context: the evaluator needs a CUDA device");
}

void upload_key(Context& c, const std::vector<u64>& wire, DeviceKey& k) {
  const size_t words = wire.size();
  u64d* stage = c.alloc(words);
  CK(cudaMemcpyAsync(stage, wire.data(), words * 8, cudaMemcpyHostToDevice, c.stream));
  if (!k.data) CK(cudaMalloc((void**)&k.data, words * 8));
  const int np = c.P->np();
  launch_wire_to_slot(c, stage, k.data, (size_t)c.L() * 2 * np, 1, np, c.L());
  launch_split31(c, k.data, words);  // keys are only ever multiply-accumulated
  c.free(stage);
  CK(cudaStreamSynchronize(c.stream));
}

}  // namespace

// ============================================================== context =====
extern "C" int hegpu_ctx_create(const hegpu_params* p, int device, hegpu_ctx** out) {
  if (!p || !out) return HEGPU_ERR_ARG;
  *out = nullptr;
  auto* h = new hegpu_ctx();
  Context& c = h->c;
  int rc = guarded(nullptr, [&] {
    c.hp = *p;
    c.P = std::make_unique<Params>(*p);
    need(c.P->np() <= HEGPU_MAX_PRIMES, HEGPU_ERR_ARG, "too many primes");
    need(c.P->n <= 32768, HEGPU_ERR_ARG, "ring degree above 2^15 is not supported by the smem NTT");
    c.client = std::make_unique<Client>(*c.P);
    c.device = device;
    if (device == HEGPU_CLIENT_ONLY) return;  // data-owner side: no device state
    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
      fail(HEGPU_ERR_CUDA, "no CUDA device: the hegpu evaluator has no CPU fallback");
    need(device >= 0 && device < n_dev, HEGPU_ERR_ARG, "bad device index");
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~0ull;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    const int np = c.P->np(), N = c.P->n;
    for (int i = 0; i < np; ++i) {
      const Prime& pr = c.P->primes[i];
      c.primes.p[i] = DevPrime{pr.q, pr.qneg_inv, pr.r_mod, pr.r2_mod, shoup_pre(1, pr.q)};
    }
    upload_twiddles(c);
    std::vector<u64> consts((size_t)2 * np + (size_t)2 * np * np);
    for (int i = 0; i < np; ++i) {
      const u64 q = c.P->q(i);
      consts[2 * i] = c.P->primes[i].ninv;
      consts[2 * i + 1] = shoup_pre(c.P->primes[i].ninv, q);
      for (int d = 0; d < np; ++d) {
        const u64 v = i == d ? 0 : inv_mod(c.P->q(d) % q, q);
        consts[2 * np + ((size_t)i * np + d) * 2] = v;
        consts[2 * np + ((size_t)i * np + d) * 2 + 1] = shoup_pre(v, q);
      }
    }
    CK(cudaMalloc((void**)&c.d_consts, consts.size() * 8));
    CK(cudaMemcpy(c.d_consts, consts.data(), consts.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMalloc((void**)&c.d_slot_src, (size_t)N * 4));
    CK(cudaMemcpy(c.d_slot_src, c.P->slot_src.data(), (size_t)N * 4, cudaMemcpyHostToDevice));
  });
  if (rc != HEGPU_OK) {
    delete h;
    return rc;
  }
  *out = h;
  return HEGPU_OK;
}

extern "C" void hegpu_ctx_destroy(hegpu_ctx* h) {
  if (!h) return;
  Context& c = h->c;
  try { bind_device(&c); } catch (...) {}
  if (c.stream) cudaStreamSynchronize(c.stream);
  for (auto& kv : c.rot_keys) cudaFree(kv.second.data);
  if (c.relin.data) cudaFree(c.relin.data);
  cudaFree(c.d_tw);
  cudaFree(c.d_twd);
  cudaFree(c.d_fpq);
  cudaFree(c.d_consts);
  cudaFree(c.d_slot_src);
  if (c.stream) cudaStreamDestroy(c.stream);
  delete h;
}

extern "C" const char* hegpu_last_error(const hegpu_ctx* h) {
  return h ? h->c.last_error.c_str() : g_create_error.c_str();
}

extern "C" int hegpu_ctx_info(const hegpu_ctx* h, int* n, int* slots, int* n_q, uint64_t* primes) {
  if (!h) return HEGPU_ERR_ARG;
  const Params& P = *h->c.P;
  if (n) *n = P.n;
  if (slots) *slots = P.slots;
  if (n_q) *n_q = P.L;
  if (primes)
    for (int i = 0; i < P.np(); ++i) primes[i] = P.q(i);
  return HEGPU_OK;
}

extern "C" int hegpu_sync(hegpu_ctx* h) {
  if (!h) return HEGPU_ERR_ARG;
  return guarded(&h->c, [&] { CK(cudaStreamSynchronize(h->c.stream)); });
}

extern "C" int64_t hegpu_kernel_launches(const hegpu_ctx* h) { return h ? h->c.launches : -1; }

extern "C" void* hegpu_stream(const hegpu_ctx* h) { return h ? (void*)h->c.stream : nullptr; }

struct hegpu_graph {
  Context* c;
  cudaGraph_t g;
  cudaGraphExec_t exec;
};

extern "C" int hegpu_capture_begin(hegpu_ctx* h) {
  if (!h) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    CK(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
  });
}

extern "C" int hegpu_capture_end(hegpu_ctx* h, hegpu_graph** out) {
  if (!h || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    cudaGraph_t g = nullptr;
    CK(cudaStreamEndCapture(c.stream, &g));
    cudaGraphExec_t exec = nullptr;
    CK(cudaGraphInstantiate(&exec, g, 0));
    *out = new hegpu_graph{&c, g, exec};
  });
}

extern "C" int hegpu_graph_launch(hegpu_graph* gr) {
  if (!gr) return HEGPU_ERR_ARG;
  Context& c = *gr->c;
  return guarded(&c, [&] { CK(cudaGraphLaunch(gr->exec, c.stream)); });
}

extern "C" void hegpu_graph_destroy(hegpu_graph* gr) {
  if (!gr) return;
  try { bind_device(gr->c); } catch (...) {}
  cudaStreamSynchronize(gr->c->stream);
  cudaGraphExecDestroy(gr->exec);
  cudaGraphDestroy(gr->g);
  delete gr;
}

extern "C" int hegpu_kernel_timer(hegpu_ctx* h, const char* name) {
  if (!h) return HEGPU_ERR_ARG;
  h->c.ktimer_name = name ? name : "";
  h->c.ktimer_used = 0;
  h->c.ktimer_bytes = 0;
  h->c.ktimer_ops = 0;
  return HEGPU_OK;
}

extern "C" int hegpu_kernel_timer_read(hegpu_ctx* h, double* total_ms, int64_t* launches, double* bytes) {
  return hegpu_kernel_timer_read_ops(h, total_ms, launches, bytes, nullptr);
}

extern "C" int hegpu_kernel_timer_read_ops(hegpu_ctx* h, double* total_ms, int64_t* launches, double* bytes,
                                           double* modmuls) {
  if (!h) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    CK(cudaStreamSynchronize(c.stream));
    double tot = 0;
    for (size_t i = 0; i < c.ktimer_used; ++i) {
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, c.ktimer_events[i].first, c.ktimer_events[i].second));
      tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = (int64_t)c.ktimer_used;
    if (bytes) *bytes = c.ktimer_bytes;
    if (modmuls) *modmuls = c.ktimer_ops;
    c.ktimer_used = 0;
    c.ktimer_bytes = 0;
    c.ktimer_ops = 0;
  });
}

extern "C" int hegpu_ct_export_device(hegpu_ct* t, void* dst, size_t nwords) {
  if (!t || !dst) return HEGPU_ERR_ARG;
  Context& c = *t->b.ctx;
  return guarded(&c, [&] {
    need(nwords == t->b.words(), HEGPU_ERR_SHAPE, "ct_export_device: word count mismatch");
    launch_slot_to_wire(c, t->b.d, (u64d*)dst, (size_t)t->b.count * 2 * t->b.level, 0, t->b.level, -1);
  });
}

// ============================================================== metering ====
extern "C" int hegpu_begin_stage(hegpu_ctx* h, const char* label) {
  if (!h || !label) return HEGPU_ERR_ARG;
  h->c.meter.begin(label);
  return HEGPU_OK;
}
extern "C" int hegpu_num_stages(const hegpu_ctx* h) { return h ? (int)h->c.meter.stages.size() : -1; }
extern "C" int hegpu_stage_tally(const hegpu_ctx* h, int idx, char* label, int len, int64_t t[5]) {
  if (!h || idx < 0 || idx >= (int)h->c.meter.stages.size()) return HEGPU_ERR_ARG;
  const auto& s = h->c.meter.stages[idx];
  if (label && len > 0) {
    std::strncpy(label, s.first.c_str(), (size_t)len - 1);
    label[len - 1] = 0;
  }
  if (t)
    for (int i = 0; i < 5; ++i) t[i] = s.second[i];
  return HEGPU_OK;
}
extern "C" int hegpu_total_tally(const hegpu_ctx* h, int64_t t[5]) {
  if (!h || !t) return HEGPU_ERR_ARG;
  for (int i = 0; i < 5; ++i) t[i] = h->c.meter.total[i];
  return HEGPU_OK;
}
extern "C" int hegpu_reset_meter(hegpu_ctx* h) {
  if (!h) return HEGPU_ERR_ARG;
  h->c.meter = Meter();
  h->c.ks = {};
  return HEGPU_OK;
}
extern "C" int hegpu_ks_counters(const hegpu_ctx* h, int64_t out[4]) {
  if (!h || !out) return HEGPU_ERR_ARG;
  for (int i = 0; i < 4; ++i) out[i] = h->c.ks[i];
  return HEGPU_OK;
}

// ============================================================== client ======
extern "C" int hegpu_encode(hegpu_ctx* h, const double* z, int len, double scale, int level, int with_p,
                            uint64_t* out) {
  if (!h || (!z && len) || !out) return HEGPU_ERR_ARG;
  return guarded(&h->c, [&] {
    need(level >= 1 && level <= h->c.L(), HEGPU_ERR_ARG, "encode: bad level");
    h->c.client->encode(z, len, scale, level, with_p != 0, out);
  });
}
extern "C" int hegpu_decode(hegpu_ctx* h, const uint64_t* pt, int level, double scale, double* slots) {
  if (!h || !pt || !slots) return HEGPU_ERR_ARG;
  return guarded(&h->c, [&] {
    need(level >= 1 && level <= h->c.L(), HEGPU_ERR_ARG, "decode: bad level");
    h->c.client->decode(pt, level, scale, slots);
  });
}
extern "C" int hegpu_encrypt(hegpu_ctx* h, const uint64_t* pt, int level, uint64_t nonce, uint64_t* ct) {
  if (!h || !pt || !ct) return HEGPU_ERR_ARG;
  return guarded(&h->c, [&] {
    need(level >= 1 && level <= h->c.L(), HEGPU_ERR_ARG, "encrypt: bad level");
    h->c.client->encrypt(pt, level, nonce, ct);
  });
}
extern "C" int hegpu_decrypt(hegpu_ctx* h, const uint64_t* ct, int level, uint64_t* pt) {
  if (!h || !pt || !ct) return HEGPU_ERR_ARG;
  return guarded(&h->c, [&] {
    need(level >= 1 && level <= h->c.L(), HEGPU_ERR_ARG, "decrypt: bad level");
    h->c.client->decrypt(ct, level, pt);
  });
}

extern "C" size_t hegpu_compact_bytes(const hegpu_ctx* h, int level) {
  if (!h || level < 1 || level > h->c.L()) return 0;
  return h->c.client->compact_bytes(level);
}

extern "C" int hegpu_encrypt_compact(hegpu_ctx* h, const uint64_t* pt, int level, uint64_t nonce, uint8_t* out) {
  if (!h || !pt || !out) return HEGPU_ERR_ARG;
  return guarded(&h->c, [&] {
    need(level >= 1 && level <= h->c.L(), HEGPU_ERR_ARG, "encrypt_compact: bad level");
    h->c.client->encrypt_compact(pt, level, nonce, out);
  });
}

extern "C" int hegpu_gen_rotation_keys(hegpu_ctx* h, const int64_t* rots, int n) {
  if (!h || (n && !rots)) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    const int S = c.S();
    std::vector<int> todo;
    for (int i = 0; i < n; ++i) {
      need(rots[i] >= 0 && rots[i] < S, HEGPU_ERR_RANGE, "rotation amount outside [0, S)");
      const int shift = (int)((S - rots[i] % S) % S);
      if (shift == 0 || c.rot_keys.count(shift)) continue;
      if (std::find(todo.begin(), todo.end(), shift) == todo.end()) todo.push_back(shift);
    }
    // host key generation is independent per Galois element: batches of keys
    // are generated on all host cores, then uploaded in order
    const size_t kw = c.client->key_words();
    const int batch = 32;
    std::vector<std::vector<u64>> wires(batch, std::vector<u64>(kw));
    for (size_t b0 = 0; b0 < todo.size(); b0 += batch) {
      const int nb = (int)std::min<size_t>(batch, todo.size() - b0);
#pragma omp parallel for schedule(dynamic)
      for (int i = 0; i < nb; ++i) c.client->gen_galois_key(c.P->galois_left(todo[b0 + i]), wires[i].data());
      for (int i = 0; i < nb; ++i) {
        DeviceKey& k = c.rot_keys[todo[b0 + i]];
        k.shift = todo[b0 + i];
        upload_key(c, wires[i], k);
      }
    }
  });
}

extern "C" int hegpu_gen_relin_key(hegpu_ctx* h) {
  if (!h) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    if (c.has_relin) return;
    std::vector<u64> wire(c.client->key_words());
    c.client->gen_relin_key(wire.data());
    upload_key(c, wire, c.relin);
    c.has_relin = true;
  });
}

extern "C" int hegpu_export_rotation_key(hegpu_ctx* h, int64_t r, uint64_t* out) {
  if (!h || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need(r > 0 && r < c.S(), HEGPU_ERR_RANGE, "rotation amount outside (0, S)");
    c.client->gen_galois_key(c.P->galois_right(r), out);
  });
}

extern "C" int hegpu_export_relin_key(hegpu_ctx* h, uint64_t* out) {
  if (!h || !out) return HEGPU_ERR_ARG;
  return guarded(&h->c, [&] { h->c.client->gen_relin_key(out); });
}

// ============================================================== handles =====
extern "C" int hegpu_ct_create(hegpu_ctx* h, int count, int level, hegpu_ct** out) {
  if (!h || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    need(count >= 1 && level >= 1 && level <= c.L(), HEGPU_ERR_ARG, "ct_create: bad count/level");
    // from the context's stream-ordered pool: handles that live for one
    // stage of a driver loop (hegpu_prog) cost no cudaMalloc / cudaFree
    auto* t = new hegpu_ct{CtBatch{&c, count, level, 1.0, nullptr}};
    try {
      t->b.d = c.alloc(t->b.words());
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

extern "C" void hegpu_ct_destroy(hegpu_ct* t) {
  if (!t) return;
  if (t->view) {
    delete t;
    return;
  }
  try {
    bind_device(t->b.ctx);
    t->b.ctx->free(t->b.d);  // stream-ordered: after everything enqueued so far
  } catch (...) {
  }
  delete t;
}

extern "C" int hegpu_ct_view(hegpu_ct* src, int first, int count, hegpu_ct** out) {
  if (!src || !out) return HEGPU_ERR_ARG;
  Context& c = *src->b.ctx;
  return guarded(&c, [&] {
    need(first >= 0 && count >= 1 && first + count <= src->b.count, HEGPU_ERR_RANGE,
         "ct_view: range outside the source batch");
    auto* t = new hegpu_ct{CtBatch{&c, count, src->b.level, src->b.scale, src->b.d + (size_t)first * src->b.stride()}};
    t->view = true;
    *out = t;
  });
}

extern "C" int hegpu_ct_copy(hegpu_ct* dst, const hegpu_ct* src) {
  if (!dst || !src) return HEGPU_ERR_ARG;
  Context& c = *src->b.ctx;
  return guarded(&c, [&] {
    need(dst->b.ctx == src->b.ctx, HEGPU_ERR_ARG, "ct_copy: handles from different contexts");
    need(dst->b.count == src->b.count && dst->b.level == src->b.level, HEGPU_ERR_SHAPE,
         "ct_copy: count/level mismatch");
    if (dst->b.d != src->b.d)
      CK(cudaMemcpyAsync(dst->b.d, src->b.d, src->b.words() * 8, cudaMemcpyDeviceToDevice, c.stream));
    dst->b.scale = src->b.scale;
  });
}

extern "C" int hegpu_ct_gather(hegpu_ct* dst, int dst_first, const hegpu_ct* src, int src_first, int src_stride,
                               int count) {
  if (!dst || !src) return HEGPU_ERR_ARG;
  Context& c = *src->b.ctx;
  return guarded(&c, [&] {
    need(dst->b.ctx == src->b.ctx, HEGPU_ERR_ARG, "ct_gather: handles from different contexts");
    need(dst->b.level == src->b.level, HEGPU_ERR_SHAPE, "ct_gather: level mismatch");
    need(count >= 1 && src_stride >= 1 && dst_first >= 0 && src_first >= 0 && dst_first + count <= dst->b.count &&
             src_first + (int64_t)(count - 1) * src_stride < src->b.count,
         HEGPU_ERR_RANGE, "ct_gather: range outside a batch");
    const size_t ct = src->b.stride() * 8;
    CK(cudaMemcpy2DAsync(dst->b.d + (size_t)dst_first * dst->b.stride(), ct,
                         src->b.d + (size_t)src_first * src->b.stride(), ct * (size_t)src_stride, ct, (size_t)count,
                         cudaMemcpyDeviceToDevice, c.stream));
  });
}

extern "C" int hegpu_ct_set_scale(hegpu_ct* t, double scale) {
  if (!t || !(scale > 0)) return HEGPU_ERR_ARG;
  t->b.scale = scale;
  return HEGPU_OK;
}

extern "C" int hegpu_ct_upload(hegpu_ct* t, const uint64_t* host, size_t nwords, double scale) {
  if (!t || !host) return HEGPU_ERR_ARG;
  Context& c = *t->b.ctx;
  return guarded(&c, [&] {
    need(nwords == t->b.words(), HEGPU_ERR_SHAPE, "ct_upload: word count mismatch");
    u64d* stage = c.alloc(nwords);
    CK(cudaMemcpyAsync(stage, host, nwords * 8, cudaMemcpyHostToDevice, c.stream));
    launch_wire_to_slot(c, stage, t->b.d, (size_t)t->b.count * 2 * t->b.level, 0, t->b.level, -1);
    c.free(stage);
    t->b.scale = scale;
    CK(cudaStreamSynchronize(c.stream));
  });
}

extern "C" int hegpu_ct_download(hegpu_ct* t, uint64_t* host, size_t nwords) {
  if (!t || !host) return HEGPU_ERR_ARG;
  Context& c = *t->b.ctx;
  return guarded(&c, [&] {
    need(nwords == t->b.words(), HEGPU_ERR_SHAPE, "ct_download: word count mismatch");
    u64d* stage = c.alloc(nwords);
    launch_slot_to_wire(c, t->b.d, stage, (size_t)t->b.count * 2 * t->b.level, 0, t->b.level, -1);
    CK(cudaMemcpyAsync(host, stage, nwords * 8, cudaMemcpyDeviceToHost, c.stream));
    c.free(stage);
    CK(cudaStreamSynchronize(c.stream));
  });
}

extern "C" int hegpu_ct_upload_compact(hegpu_ct* t, const uint8_t* host, size_t nbytes, double scale) {
  if (!t || !host) return HEGPU_ERR_ARG;
  Context& c = *t->b.ctx;
  return guarded(&c, [&] {
    const size_t per = c.client->compact_bytes(t->b.level);
    need(nbytes == per * t->b.count, HEGPU_ERR_SHAPE, "ct_upload_compact: byte count mismatch");
    u64d* stage = c.alloc((nbytes + 7) / 8);
    CK(cudaMemcpyAsync(stage, host, nbytes, cudaMemcpyHostToDevice, c.stream));
    launch_expand_compact(c, (const uint8_t*)stage, t->b.count, t->b.level, t->b.d);
    c.free(stage);
    t->b.scale = scale;
    CK(cudaStreamSynchronize(c.stream));
  });
}

extern "C" int hegpu_ct_info(const hegpu_ct* t, int* count, int* level, double* scale) {
  if (!t) return HEGPU_ERR_ARG;
  if (count) *count = t->b.count;
  if (level) *level = t->b.level;
  if (scale) *scale = t->b.scale;
  return HEGPU_OK;
}

extern "C" int hegpu_pt_create(hegpu_ctx* h, int count, int level, int with_p, hegpu_pt** out) {
  if (!h || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    need(count >= 1 && level >= 1 && level <= c.L(), HEGPU_ERR_ARG, "pt_create: bad count/level");
    auto* t = new hegpu_pt{PtBatch{&c, count, level, with_p ? 1 : 0, 1.0, nullptr}};
    cudaError_t e = cudaMalloc((void**)&t->b.d, t->b.words() * 8);
    if (e != cudaSuccess) { delete t; CK(e); }
    *out = t;
  });
}

extern "C" void hegpu_pt_destroy(hegpu_pt* t) {
  if (!t) return;
  try { bind_device(t->b.ctx); } catch (...) {}
  cudaStreamSynchronize(t->b.ctx->stream);
  cudaFree(t->b.d);
  delete t;
}

extern "C" int hegpu_pt_upload(hegpu_pt* t, const uint64_t* host, size_t nwords, double scale) {
  if (!t || !host) return HEGPU_ERR_ARG;
  Context& c = *t->b.ctx;
  return guarded(&c, [&] {
    need(nwords == t->b.words(), HEGPU_ERR_SHAPE, "pt_upload: word count mismatch");
    u64d* stage = c.alloc(nwords);
    CK(cudaMemcpyAsync(stage, host, nwords * 8, cudaMemcpyHostToDevice, c.stream));
    const int nl = t->b.limbs();
    launch_wire_to_slot(c, stage, t->b.d, (size_t)t->b.count * nl, 1, nl, t->b.with_p ? t->b.level : -1);
    c.free(stage);
    t->b.scale = scale;
    CK(cudaStreamSynchronize(c.stream));
  });
}

extern "C" int hegpu_pt_download(hegpu_pt* t, uint64_t* host, size_t nwords) {
  if (!t || !host) return HEGPU_ERR_ARG;
  Context& c = *t->b.ctx;
  return guarded(&c, [&] {
    need(nwords == t->b.words(), HEGPU_ERR_SHAPE, "pt_download: word count mismatch");
    u64d* stage = c.alloc(nwords);
    const int nl = t->b.limbs();
    launch_slot_to_wire(c, t->b.d, stage, (size_t)t->b.count * nl, 1, nl, t->b.with_p ? t->b.level : -1);
    CK(cudaMemcpyAsync(host, stage, nwords * 8, cudaMemcpyDeviceToHost, c.stream));
    c.free(stage);
    CK(cudaStreamSynchronize(c.stream));
  });
}

// ============================================================== evaluator ===
namespace {

void same_shape(const CtBatch& a, const CtBatch& b, const char* what) {
  need(a.ctx == b.ctx, HEGPU_ERR_ARG, std::string(what) + ": handles from different contexts");
  need(a.count == b.count && a.level == b.level, HEGPU_ERR_SHAPE,
       std::string(what) + ": count/level mismatch");
}

void plain_ok(const CtBatch& a, const PtBatch& p, const char* what) {
  need(p.ctx == a.ctx, HEGPU_ERR_ARG, std::string(what) + ": handles from different contexts");
  need(p.level == a.level, HEGPU_ERR_SHAPE, std::string(what) + ": plaintext level mismatch");
  need(p.count == 1 || p.count == a.count, HEGPU_ERR_SHAPE, std::string(what) + ": plaintext count mismatch");
}

}  // namespace

extern "C" int hegpu_add(hegpu_ctx* h, const hegpu_ct* a, const hegpu_ct* b, hegpu_ct* out) {
  if (!h || !a || !b || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    same_shape(a->b, b->b, "add");
    same_shape(a->b, out->b, "add");
    launch_add(c, a->b.d, b->b.d, out->b.d, a->b.count, a->b.level);
    out->b.scale = a->b.scale;
    c.meter.bump(HEGPU_ADD_CC, a->b.count);
  });
}

extern "C" int hegpu_add_plain(hegpu_ctx* h, const hegpu_ct* a, const hegpu_pt* p, hegpu_ct* out) {
  if (!h || !a || !p || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    plain_ok(a->b, p->b, "add_plain");
    same_shape(a->b, out->b, "add_plain");
    const long ps = p->b.count == 1 ? 0 : (long)p->b.limbs() * c.N();
    launch_add_plain(c, a->b.d, p->b.d, ps, out->b.d, a->b.count, a->b.level);
    out->b.scale = a->b.scale;
    c.meter.bump(HEGPU_ADD_PC, a->b.count);
  });
}

extern "C" int hegpu_mul_plain(hegpu_ctx* h, const hegpu_ct* a, const hegpu_pt* p, hegpu_ct* out) {
  if (!h || !a || !p || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    plain_ok(a->b, p->b, "mul_plain");
    same_shape(a->b, out->b, "mul_plain");
    const long ps = p->b.count == 1 ? 0 : (long)p->b.limbs() * c.N();
    launch_mul_plain(c, a->b.d, p->b.d, ps, out->b.d, a->b.count, a->b.level);
    out->b.scale = a->b.scale * p->b.scale;
    c.meter.bump(HEGPU_MUL_PC, a->b.count);
  });
}

extern "C" int hegpu_rescale(hegpu_ctx* h, const hegpu_ct* a, hegpu_ct* out) {
  if (!h || !a || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need(a->b.level >= 2, HEGPU_ERR_CAPACITY, "rescale: no prime left to drop");
    need(out->b.count == a->b.count && out->b.level == a->b.level - 1, HEGPU_ERR_SHAPE,
         "rescale: output must have level - 1");
    eval_rescale(c, a->b, out->b);
    out->b.scale = a->b.scale / (double)c.P->q(a->b.level - 1);
  });
}

static int rotate_impl(hegpu_ctx* h, const hegpu_ct* a, int64_t r, bool right, hegpu_ct* out) {
  if (!h || !a || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    const int S = c.S();
    need(r >= 0 && r < S, HEGPU_ERR_RANGE,
         "rotate: amount " + std::to_string(r) + " outside [0, " + std::to_string(S) + ")");
    same_shape(a->b, out->b, "rotate");
    need(a != out, HEGPU_ERR_ARG, "rotate: output must not alias the input");
    const int shift = right ? (int)((S - r) % S) : (int)r;
    if (shift == 0) {  // free no-op (slotvec.cpp:49)
      CK(cudaMemcpyAsync(out->b.d, a->b.d, a->b.words() * 8, cudaMemcpyDeviceToDevice, c.stream));
      out->b.scale = a->b.scale;
      return;
    }
    KeyRowMap km{};
    km.period = 1;
    km.shift[0] = shift;
    km.key[0] = c.rot_key(shift).data;
    eval_rotate(c, a->b.d, (long)a->b.stride(), a->b.count, a->b.level, km, out->b.d,
                (long)out->b.stride());
    out->b.scale = a->b.scale;
    c.meter.bump(HEGPU_ROT, a->b.count);
  });
}

extern "C" int hegpu_rotate_right(hegpu_ctx* h, const hegpu_ct* a, int64_t r, hegpu_ct* out) {
  return rotate_impl(h, a, r, true, out);
}
extern "C" int hegpu_rotate_left(hegpu_ctx* h, const hegpu_ct* a, int64_t r, hegpu_ct* out) {
  return rotate_impl(h, a, r, false, out);
}

extern "C" int hegpu_square(hegpu_ctx* h, const hegpu_ct* a, hegpu_ct* out) {
  if (!h || !a || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need(a->b.level >= 2, HEGPU_ERR_CAPACITY, "square: no prime left to rescale");
    need(out->b.count == a->b.count && out->b.level == a->b.level - 1, HEGPU_ERR_SHAPE,
         "square: output must have level - 1");
    square_layer(c, a->b, out->b);
    c.meter.bump(HEGPU_MUL_CC, a->b.count);
  });
}

extern "C" int hegpu_conv_packed_forward(hegpu_ctx* h, const hegpu_ct* taps, int ntaps, const double* weights,
                                         int c_out, const double* bias, int w_used, hegpu_ct* maps) {
  if (!h || !taps || !weights || !maps) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need(ntaps >= 1 && c_out >= 1 && taps->b.count % ntaps == 0, HEGPU_ERR_SHAPE,
         "conv_packed_forward: filter/tap shape mismatch");
    const int B = taps->b.count / ntaps;
    need(maps->b.count == B * c_out && maps->b.level == taps->b.level - 1, HEGPU_ERR_SHAPE,
         "conv_packed_forward: maps must be B*c_out at level - 1");
    need(w_used >= 0 && w_used <= c.S(), HEGPU_ERR_CAPACITY, "conv_packed_forward: w exceeds slots");
    ConvLayer layer(c, ntaps, c_out, weights, bias, w_used, taps->b.level, taps->b.scale);
    layer.run(c, taps->b, maps->b);
    c.meter.bump(HEGPU_MUL_PC, (int64_t)B * ntaps * c_out);
    c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (ntaps - 1) * c_out);
    c.meter.bump(HEGPU_ADD_PC, (int64_t)B * c_out);
  });
}

struct hegpu_conv_plan {
  std::unique_ptr<ConvLayer> layer;
  int ntaps, c_out;
};

extern "C" int hegpu_conv_plan_create(hegpu_ctx* h, int ntaps, const double* weights, int c_out, const double* bias,
                                      int w_used, int level, double tap_scale, hegpu_conv_plan** out) {
  if (!h || !weights || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    need(ntaps >= 1 && c_out >= 1, HEGPU_ERR_SHAPE, "conv_plan: bad shape");
    need(level >= 2 && level <= c.L(), HEGPU_ERR_CAPACITY, "conv_plan: level must leave a prime to rescale");
    need(w_used >= 0 && w_used <= c.S(), HEGPU_ERR_CAPACITY, "conv_plan: w exceeds slots");
    auto* p = new hegpu_conv_plan{nullptr, ntaps, c_out};
    try {
      p->layer = std::make_unique<ConvLayer>(c, ntaps, c_out, weights, bias, w_used, level, tap_scale);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

extern "C" void hegpu_conv_plan_destroy(hegpu_conv_plan* p) {
  if (!p) return;
  try { bind_device(p->layer ? p->layer->ctx : nullptr); } catch (...) {}
  delete p;
}

extern "C" int hegpu_conv_plan_run(hegpu_ctx* h, const hegpu_conv_plan* p, const hegpu_ct* taps, hegpu_ct* maps) {
  if (!h || !p || !taps || !maps) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    const int ntaps = p->ntaps, c_out = p->c_out;
    need(taps->b.level == p->layer->level && taps->b.count % ntaps == 0, HEGPU_ERR_SHAPE,
         "conv_plan_run: taps must be B*ntaps at the plan level");
    const int B = taps->b.count / ntaps;
    need(maps->b.count == B * c_out && maps->b.level == taps->b.level - 1, HEGPU_ERR_SHAPE,
         "conv_plan_run: maps must be B*c_out at level - 1");
    p->layer->run(c, taps->b, maps->b);
    c.meter.bump(HEGPU_MUL_PC, (int64_t)B * ntaps * c_out);
    c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (ntaps - 1) * c_out);
    c.meter.bump(HEGPU_ADD_PC, (int64_t)B * c_out);
  });
}

struct hegpu_masked_conv {
  std::unique_ptr<MaskedConv> layer;
};

extern "C" int hegpu_masked_conv_create(hegpu_ctx* h, int ntaps, const double* weights, int c_out, const double* bias,
                                        int w_used, int level, double tap_scale, hegpu_masked_conv** out) {
  if (!h || !weights || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    need(ntaps >= 1 && c_out >= 1, HEGPU_ERR_SHAPE, "masked_conv: bad shape");
    auto* p = new hegpu_masked_conv{nullptr};
    try {
      p->layer = std::make_unique<MaskedConv>(c, ntaps, c_out, weights, bias, w_used, level, tap_scale);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

extern "C" void hegpu_masked_conv_destroy(hegpu_masked_conv* p) {
  if (!p) return;
  try { bind_device(p->layer ? p->layer->ctx : nullptr); } catch (...) {}
  delete p;
}

extern "C" int hegpu_masked_conv_run(hegpu_ctx* h, const hegpu_masked_conv* p, const hegpu_ct* taps, hegpu_ct* maps) {
  if (!h || !p || !taps || !maps) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    const int ntaps = p->layer->ntaps, c_out = p->layer->c_out;
    need(taps->b.level == p->layer->level && taps->b.count % ntaps == 0, HEGPU_ERR_SHAPE,
         "masked_conv_run: taps must be ntaps * B at the plan level");
    const int B = taps->b.count / ntaps;
    need(maps->b.count == B * c_out && maps->b.level == taps->b.level - 1, HEGPU_ERR_SHAPE,
         "masked_conv_run: maps must be c_out * B at level - 1");
    p->layer->run(c, taps->b, maps->b);
    c.meter.bump(HEGPU_MUL_PC, (int64_t)B * ntaps * c_out);
    c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (ntaps - 1) * c_out);
    c.meter.bump(HEGPU_ADD_PC, (int64_t)B * c_out);
  });
}

extern "C" int hegpu_merge_maps(hegpu_ctx* h, const hegpu_ct* maps, int nmaps, int64_t w, hegpu_ct* out) {
  if (!h || !maps || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need(nmaps >= 1, HEGPU_ERR_SHAPE, "merge_maps: no maps");
    need(maps->b.count % nmaps == 0, HEGPU_ERR_SHAPE, "merge_maps: count not a multiple of c");
    need((int64_t)nmaps * w <= c.S(), HEGPU_ERR_CAPACITY,
         "merge_maps: " + std::to_string(nmaps) + " maps of " + std::to_string(w) + " slots exceed " +
             std::to_string(c.S()) + " slots");
    const int B = maps->b.count / nmaps;
    need(out->b.count == B && out->b.level == maps->b.level, HEGPU_ERR_SHAPE, "merge_maps: bad output");
    merge_maps(c, maps->b, nmaps, w, out->b);
    c.meter.bump(HEGPU_ROT, (int64_t)B * (nmaps - 1));
    c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (nmaps - 1));
  });
}

struct hegpu_hs_plan {
  HsPlan p;
};

extern "C" int hegpu_hs_plan_create(hegpu_ctx* h, const double* A, int m, int n, int level, int skip_zero,
                                    hegpu_hs_plan** out) {
  if (!h || !A || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    need(level >= 2 && level <= c.L(), HEGPU_ERR_ARG, "hs_plan: level must leave a prime to rescale");
    auto* pl = new hegpu_hs_plan();
    try {
      pl->p.build(c, A, m, n, level, skip_zero != 0);
    } catch (...) {
      delete pl;
      throw;
    }
    *out = pl;
  });
}

extern "C" void hegpu_hs_plan_destroy(hegpu_hs_plan* p) {
  if (!p) return;
  try { bind_device(p->p.ctx); } catch (...) {}
  p->p.release();
  delete p;
}

extern "C" int hegpu_hs_plan_rotations(const hegpu_hs_plan* p, int64_t* rots, int cap) {
  if (!p) return -1;
  const std::vector<int64_t> r = p->p.right_rotations();
  for (int i = 0; rots && i < cap && i < (int)r.size(); ++i) rots[i] = r[i];
  return (int)r.size();
}

extern "C" int hegpu_hs_plan_info(const hegpu_hs_plan* p, int* m_eff, int* folds, int* kept) {
  if (!p) return HEGPU_ERR_ARG;
  if (m_eff) *m_eff = p->p.m_eff;
  if (folds) *folds = p->p.folds;
  if (kept) *kept = (int)p->p.diag.size();
  return HEGPU_OK;
}

extern "C" size_t hegpu_hs_acc_words(const hegpu_hs_plan* p, int batch) {
  return p && p->p.ctx ? p->p.acc_words(batch, p->p.ctx->N()) : 0;
}

extern "C" int hegpu_hs_matvec_partial(hegpu_ctx* h, const hegpu_hs_plan* p, const hegpu_ct* v, int part, int nparts,
                                       void* dev_acc) {
  if (!h || !p || !v || !dev_acc) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    HsPlan& pl = const_cast<HsPlan&>(p->p);
    need(v->b.level == pl.level, HEGPU_ERR_LAYOUT, "hs_matvec_partial: input level does not match the plan");
    need(nparts >= 1 && part >= 0 && part < nparts, HEGPU_ERR_RANGE, "hs_matvec_partial: bad part");
    need(nparts <= 8, HEGPU_ERR_CAPACITY, "hs_matvec_partial: at most 8 parts (sums must stay < 2^64)");
    const int kept = (int)pl.diag.size(), B = v->b.count;
    const int i_lo = (int)((int64_t)kept * part / nparts), i_hi = (int)((int64_t)kept * (part + 1) / nparts);
    u64d* acc = static_cast<u64d*>(dev_acc);
    pl.accumulate(c, v->b, i_lo, i_hi, acc, acc + (size_t)B * 2 * (pl.level + 1) * c.N());
    int64_t rots = 0;
    for (int i = i_lo; i < i_hi; ++i) rots += pl.diag[i].right != 0;
    c.meter.bump(HEGPU_MUL_PC, (int64_t)B * (i_hi - i_lo));
    c.meter.bump(HEGPU_ROT, (int64_t)B * rots);
    c.meter.bump(HEGPU_ADD_CC, (int64_t)B * (i_hi - i_lo - (i_lo == 0 && i_hi > 0 ? 1 : 0)));
  });
}

extern "C" int hegpu_hs_matvec_finish(hegpu_ctx* h, const hegpu_hs_plan* p, const hegpu_ct* v, void* dev_acc,
                                      int nparts, hegpu_ct* out) {
  if (!h || !p || !v || !dev_acc || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    HsPlan& pl = const_cast<HsPlan&>(p->p);
    need(out->b.count == v->b.count && out->b.level == v->b.level - 1, HEGPU_ERR_SHAPE,
         "hs_matvec_finish: output must have level - 1");
    need(nparts >= 1 && nparts <= 8, HEGPU_ERR_RANGE, "hs_matvec_finish: 1..8 parts");
    const int B = v->b.count;
    u64d* acc = static_cast<u64d*>(dev_acc);
    pl.finish(c, B, v->b.scale, acc, acc + (size_t)B * 2 * (pl.level + 1) * c.N(), nparts, out->b);
    c.meter.bump(HEGPU_ROT, (int64_t)B * pl.folds);
    c.meter.bump(HEGPU_ADD_CC, (int64_t)B * pl.folds);
  });
}

extern "C" int hegpu_hs_matvec(hegpu_ctx* h, const hegpu_hs_plan* p, const hegpu_ct* v, hegpu_ct* out) {
  if (!h || !p || !v || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    const HsPlan& pl = p->p;
    need(v->b.level == pl.level, HEGPU_ERR_LAYOUT, "hs_matvec: input level does not match the plan");
    need(out->b.count == v->b.count && out->b.level == v->b.level - 1, HEGPU_ERR_SHAPE,
         "hs_matvec: output must have level - 1");
    need(v != out, HEGPU_ERR_ARG, "hs_matvec: output must not alias the input");
    const_cast<HsPlan&>(pl).run(c, v->b, out->b);
    const int64_t B = v->b.count, kept = (int64_t)pl.diag.size();
    int64_t rots = 0;
    for (const auto& d : pl.diag) rots += d.right != 0;
    c.meter.bump(HEGPU_MUL_PC, B * kept);
    c.meter.bump(HEGPU_ROT, B * (rots + pl.folds));
    c.meter.bump(HEGPU_ADD_CC, B * ((kept > 0 ? kept - 1 : 0) + pl.folds));
  });
}

// ---- LoLa comparators (proj/src/matvec.cpp:107-211) -------------------------
struct hegpu_lola_plan {
  LolaPlan p;
};

extern "C" int hegpu_lola_plan_create(hegpu_ctx* h, int kind, const double* A, int m, int n, int level,
                                      hegpu_lola_plan** out) {
  if (!h || !A || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    need_gpu(c);
    need(kind == HEGPU_LOLA_DENSE || kind == HEGPU_LOLA_STACKED, HEGPU_ERR_ARG, "lola: unknown kind");
    auto* pl = new hegpu_lola_plan();
    try {
      pl->p.build(c, kind, A, m, n, level);
    } catch (...) {
      delete pl;
      throw;
    }
    *out = pl;
  });
}

extern "C" void hegpu_lola_plan_destroy(hegpu_lola_plan* p) {
  if (!p) return;
  try { bind_device(p->p.ctx); } catch (...) {}
  p->p.release();
  delete p;
}

extern "C" int hegpu_lola_plan_rotations(const hegpu_lola_plan* p, int64_t* rots, int cap) {
  if (!p) return -1;
  const std::vector<int64_t> r = p->p.right_rotations();
  for (int i = 0; rots && i < cap && i < (int)r.size(); ++i) rots[i] = r[i];
  return (int)r.size();
}

extern "C" int hegpu_lola_plan_info(const hegpu_lola_plan* p, int* delta, int* k, int* batches, int* folds,
                                    int* per_input) {
  if (!p) return HEGPU_ERR_ARG;
  if (delta) *delta = p->p.delta;
  if (k) *k = p->p.k;
  if (batches) *batches = p->p.batches;
  if (folds) *folds = p->p.folds;
  if (per_input) *per_input = p->p.out_count(1);
  return HEGPU_OK;
}

extern "C" int64_t hegpu_lola_slot_of_row(const hegpu_lola_plan* p, int row) {
  if (!p || row < 0 || row >= p->p.m) return -1;
  return p->p.slot_of_row(row);
}

extern "C" int hegpu_lola_matvec(hegpu_ctx* h, const hegpu_lola_plan* p, const hegpu_ct* v, hegpu_ct* out) {
  if (!h || !p || !v || !out) return HEGPU_ERR_ARG;
  Context& c = h->c;
  return guarded(&c, [&] {
    const LolaPlan& pl = p->p;
    need(v->b.level == pl.level, HEGPU_ERR_LAYOUT, "lola_matvec: input level does not match the plan");
    need(out->b.count == pl.out_count(v->b.count) && out->b.level == v->b.level - 2, HEGPU_ERR_SHAPE,
         "lola_matvec: output must hold out_count ciphertexts at level - 2");
    need(v != out, HEGPU_ERR_ARG, "lola_matvec: output must not alias the input");
    const_cast<LolaPlan&>(pl).run(c, v->b, out->b);
    const int64_t B = v->b.count;
    if (pl.kind == HEGPU_LOLA_DENSE) {  // predict_lola_dense (matvec.cpp:189-195)
      c.meter.bump(HEGPU_MUL_PC, B * pl.m);
      c.meter.bump(HEGPU_ROT, B * pl.m * pl.folds);
      c.meter.bump(HEGPU_ADD_CC, B * pl.m * pl.folds);
    } else {  // predict_lola_stacked (matvec.cpp:197-211): the input is re-stacked per batch
      const int64_t r = (int64_t)pl.batches * (pl.k + pl.folds - 1) + pl.batches - 1;
      c.meter.bump(HEGPU_MUL_PC, B * pl.batches);
      c.meter.bump(HEGPU_ROT, B * r);
      c.meter.bump(HEGPU_ADD_CC, B * r);
    }
  });
}
