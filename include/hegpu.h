/*
 * hegpu.h -- C-ABI of the B200-native CKKS engine behind the reference's
 * evaluator / layer API (arXiv 2110.08321, reference `hesim`).
 *
 * The reference has no FFI: it is a static C++ library of free functions
 * over value types (proj/CMakeLists.txt:10-19).  This header is the
 * boundary SURVEY.md §8b specifies: opaque handles, plain pointers and
 * sizes, int status codes, a per-context last-error string.  Each entry
 * point names the reference interface it replaces (file:line, paths
 * relative to the reference root).  include/hegpu.hpp restores the hesim::
 * value-semantics names on top of it; INTEGRATION.md shows the bindings.
 *
 * Data formats ("wire format", what upload/download/encode/encrypt use):
 *   - a polynomial at level l is l limbs of N uint64 words, limb i reduced
 *     mod q_i, in the NTT domain with bit-reversed evaluation order (word k
 *     of a limb holds a(psi^(2*brv(k)+1))); the extended basis appends the
 *     special prime P as limb l;
 *   - a ciphertext is [2][l][N] (c0 then c1); a batch of `count`
 *     ciphertexts is [count][2][l][N]; a plaintext batch is [count][l'][N].
 * Device-internal layout differs (slot-ordered evaluations so Galois
 * rotations are cyclic shifts, Montgomery-form plaintexts); upload and
 * download convert, so wire limbs are bit-identical to the CPU oracle.
 *
 * Metering: every evaluator/layer call bumps the context's OpTally under
 * the current stage exactly like the reference (proj/src/slotvec.cpp:49-52,
 * 76-86): a call on a batch of `count` ciphertexts counts `count` ops.
 */
#ifndef HEGPU_H
#define HEGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; errors map onto proj/include/hesim/errors.hpp:9-26 and
 * std::out_of_range (proj/src/slotvec.cpp:45-48) */
enum {
  HEGPU_OK = 0,
  HEGPU_ERR_CAPACITY = 1, /* hesim::CapacityError */
  HEGPU_ERR_SHAPE = 2,    /* hesim::ShapeError    */
  HEGPU_ERR_LAYOUT = 3,   /* hesim::LayoutError   */
  HEGPU_ERR_RANGE = 4,    /* std::out_of_range    */
  HEGPU_ERR_IO = 5,       /* hesim::IoError       */
  HEGPU_ERR_CUDA = 6,     /* CUDA runtime failure / no device */
  HEGPU_ERR_NCCL = 7,
  HEGPU_ERR_ARG = 8,      /* null handle, bad parameter */
  HEGPU_ERR_KEY = 9       /* missing evaluation key */
};

/* tally field order, proj/include/hesim/meter.hpp:12-31 */
enum { HEGPU_ADD_PC = 0, HEGPU_ADD_CC = 1, HEGPU_MUL_PC = 2, HEGPU_MUL_CC = 3, HEGPU_ROT = 4 };

typedef struct hegpu_ctx hegpu_ctx;
typedef struct hegpu_ct hegpu_ct;
typedef struct hegpu_pt hegpu_pt;
typedef struct hegpu_hs_plan hegpu_hs_plan;
typedef struct hegpu_lola_plan hegpu_lola_plan;
typedef struct hegpu_net hegpu_net;

#define HEGPU_MAX_Q 15

typedef struct {
  int log_n;                 /* ring degree N = 2^log_n, slots S = N/2; the device evaluator takes
                              * 5 <= log_n <= 15 (log_n = 15 needs every prime below 2^45: those rows
                              * run on the FP64 NTT, split over two-CTA clusters) */
  int n_q;                   /* Q chain length L (L-1 rescales) */
  int q_bits[HEGPU_MAX_Q];   /* bit sizes of q_0..q_{L-1} (<= 60) */
  int p_bits;                /* special prime P (<= 60) */
  uint64_t seed;             /* secret / key / encryption randomness */
} hegpu_params;

/* ---- context ------------------------------------------------------------ */
/* device = HEGPU_CLIENT_ONLY creates a host-only context for the data-owner
 * side (encode / encrypt / decrypt / key export); every device call on it
 * fails with HEGPU_ERR_CUDA -- there is no CPU evaluator. */
#define HEGPU_CLIENT_ONLY (-1)
int hegpu_ctx_create(const hegpu_params* p, int device, hegpu_ctx** out);
void hegpu_ctx_destroy(hegpu_ctx* ctx);
const char* hegpu_last_error(const hegpu_ctx* ctx);
/* N, S, L and the L+1 primes (q_0..q_{L-1}, P) */
int hegpu_ctx_info(const hegpu_ctx* ctx, int* n, int* slots, int* n_q, uint64_t* primes);
int hegpu_sync(hegpu_ctx* ctx);
/* kernels launched by this context since creation (ours only) */
int64_t hegpu_kernel_launches(const hegpu_ctx* ctx);
/* per-kernel timing: bracket every launch of kernel `name` (e.g.
 * "k_hs_diag") with CUDA events on the context stream; NULL disables.
 * _read synchronises, returns the summed device time, launch count and
 * algorithmic HBM bytes since the timer was (re)armed, and
 * re-arms it. */
int hegpu_kernel_timer(hegpu_ctx* ctx, const char* name);
int hegpu_kernel_timer_read(hegpu_ctx* ctx, double* total_ms, int64_t* launches, double* alg_bytes);
/* as hegpu_kernel_timer_read, plus the launches' algorithmic modular
 * multiplies (multiply-accumulate terms, NTT butterflies) */
int hegpu_kernel_timer_read_ops(hegpu_ctx* ctx, double* total_ms, int64_t* launches, double* alg_bytes,
                                double* modmuls);
/* CUDA-graph capture of everything the context enqueues between begin and
 * end (e.g. one hegpu_net_run); replay with hegpu_graph_launch.  Metering
 * and launch counters advance only while capturing. */
typedef struct hegpu_graph hegpu_graph;
int hegpu_capture_begin(hegpu_ctx* ctx);
int hegpu_capture_end(hegpu_ctx* ctx, hegpu_graph** out);
int hegpu_graph_launch(hegpu_graph* g);
void hegpu_graph_destroy(hegpu_graph* g);
/* the cudaStream_t every kernel of this context is launched on (for
 * caller-side CUDA-event timing); NULL for a client-only context */
void* hegpu_stream(const hegpu_ctx* ctx);
/* copy a device ciphertext batch, in wire format, into caller-owned device
 * memory (e.g. a torch.cuda tensor handed to an NCCL gather) */
int hegpu_ct_export_device(hegpu_ct* ct, void* dev_dst, size_t nwords);

/* ---- metering: proj/include/hesim/meter.hpp:36-70 ----------------------- */
int hegpu_begin_stage(hegpu_ctx* ctx, const char* label);
int hegpu_num_stages(const hegpu_ctx* ctx);
int hegpu_stage_tally(const hegpu_ctx* ctx, int idx, char* label, int label_len, int64_t tally[5]);
int hegpu_total_tally(const hegpu_ctx* ctx, int64_t tally[5]);
int hegpu_reset_meter(hegpu_ctx* ctx);
/* key-switch work the engine actually executed since the last
 * hegpu_reset_meter (the OpTally above keeps the reference's HOP semantics,
 * where a hoisted or fused rotation still counts as one Rot): out[0] ModUps
 * (a polynomial decomposed and lifted to the extended basis), out[1] key
 * inner products (one evaluation key applied to one ModUp'd polynomial),
 * out[2] ModDowns (an extended-basis accumulator divided by P), out[3]
 * rescales (a ciphertext batch entry dropping one prime) */
int hegpu_ks_counters(const hegpu_ctx* ctx, int64_t out[4]);

/* ---- client side (host CPU; the reference's pack/conv_pack are client-side,
 *      proj/include/hesim/convlower.hpp:20-23, proj/src/slotvec.cpp:26-40) --- */
/* pack(values, n_slots, Plaintext) (proj/src/slotvec.cpp:26-36) as a CKKS
 * encoding at `scale`: out = level (+1 if with_p) limbs */
int hegpu_encode(hegpu_ctx* ctx, const double* z, int len, double scale, int level, int with_p,
                 uint64_t* out);
int hegpu_decode(hegpu_ctx* ctx, const uint64_t* pt, int level, double scale, double* slots);
/* pack(values, n_slots, Ciphertext): symmetric encryption of an encoded pt */
int hegpu_encrypt(hegpu_ctx* ctx, const uint64_t* pt, int level, uint64_t nonce, uint64_t* ct);
int hegpu_decrypt(hegpu_ctx* ctx, const uint64_t* ct, int level, uint64_t* pt);
/* compact fresh ciphertext: the `level` a-stream keys (u64), then c0 limb i
 * byte-packed in ceil(bits(q_i)/8) bytes per coefficient (wire order); c1 is
 * regenerated from the stream keys on upload -- bit-identical to
 * hegpu_encrypt's output, 2.9x fewer bytes for the config-0 chain */
size_t hegpu_compact_bytes(const hegpu_ctx* ctx, int level);
int hegpu_encrypt_compact(hegpu_ctx* ctx, const uint64_t* pt, int level, uint64_t nonce, uint8_t* out);
/* Galois keys for right rotations by r (slotvec.cpp:42-57 semantics) and the
 * relinearisation key; generated on the host, stored on the device */
int hegpu_gen_rotation_keys(hegpu_ctx* ctx, const int64_t* right_rots, int n);
int hegpu_gen_relin_key(hegpu_ctx* ctx);
/* host copy of a generated key, wire format [L][2][L+1][N] (for tests) */
int hegpu_export_rotation_key(hegpu_ctx* ctx, int64_t right_rot, uint64_t* out);
int hegpu_export_relin_key(hegpu_ctx* ctx, uint64_t* out);

/* ---- device ciphertext / plaintext batches ------------------------------ */
int hegpu_ct_create(hegpu_ctx* ctx, int count, int level, hegpu_ct** out);
void hegpu_ct_destroy(hegpu_ct* ct);
int hegpu_ct_upload(hegpu_ct* ct, const uint64_t* host, size_t nwords, double scale);
int hegpu_ct_download(hegpu_ct* ct, uint64_t* host, size_t nwords);
/* upload `count` compact ciphertexts (hegpu_encrypt_compact) back to back */
int hegpu_ct_upload_compact(hegpu_ct* ct, const uint8_t* host, size_t nbytes, double scale);
int hegpu_ct_info(const hegpu_ct* ct, int* count, int* level, double* scale);
/* a non-owning handle on ciphertexts [first, first + count) of `src` (the
 * reference slices std::vector<SlotVector>, proj/src/netcompile.cpp:338-342);
 * valid while `src` lives, released with hegpu_ct_destroy */
int hegpu_ct_view(hegpu_ct* src, int first, int count, hegpu_ct** out);
/* device copy between handles of equal count and level (value semantics of
 * SlotVector assignment) */
int hegpu_ct_copy(hegpu_ct* dst, const hegpu_ct* src);
/* dst[dst_first + i] = src[src_first + i * src_stride], i < count (one strided
 * device copy): regroups a batch between image-major and unit-major order */
int hegpu_ct_gather(hegpu_ct* dst, int dst_first, const hegpu_ct* src, int src_first, int src_stride, int count);
int hegpu_ct_set_scale(hegpu_ct* ct, double scale);
int hegpu_pt_create(hegpu_ctx* ctx, int count, int level, int with_p, hegpu_pt** out);
void hegpu_pt_destroy(hegpu_pt* pt);
int hegpu_pt_upload(hegpu_pt* pt, const uint64_t* host, size_t nwords, double scale);
int hegpu_pt_download(hegpu_pt* pt, uint64_t* host, size_t nwords);

/* ---- evaluator: proj/include/hesim/slotvec.hpp:44-52 -------------------- */
/* add(ct, ct): Add CC (slotvec.cpp:97-102) */
int hegpu_add(hegpu_ctx* ctx, const hegpu_ct* a, const hegpu_ct* b, hegpu_ct* out);
/* add(ct, pt): Add PC; pt count 1 broadcasts over the batch */
int hegpu_add_plain(hegpu_ctx* ctx, const hegpu_ct* a, const hegpu_pt* p, hegpu_ct* out);
/* mul(ct, pt): Mul PC (slotvec.cpp:104-109); pt count 1 broadcasts */
int hegpu_mul_plain(hegpu_ctx* ctx, const hegpu_ct* a, const hegpu_pt* p, hegpu_ct* out);
/* CKKS rescale (new; the reference models no levels): unmetered */
int hegpu_rescale(hegpu_ctx* ctx, const hegpu_ct* a, hegpu_ct* out);
/* rotate_right / rotate_left (slotvec.cpp:42-66): Rot, r=0 free,
 * r outside [0, S) -> HEGPU_ERR_RANGE */
int hegpu_rotate_right(hegpu_ctx* ctx, const hegpu_ct* a, int64_t r, hegpu_ct* out);
int hegpu_rotate_left(hegpu_ctx* ctx, const hegpu_ct* a, int64_t r, hegpu_ct* out);

/* ---- layers: proj/include/hesim/convlower.hpp:24-54, matvec.hpp:41-66 --- */
/* square_layer (convlower.cpp:141-143): Mul CC + relinearise + rescale */
int hegpu_square(hegpu_ctx* ctx, const hegpu_ct* a, hegpu_ct* out);
/* conv_packed_forward (convlower.cpp:39-74) + rescale: taps = count B*ntaps
 * ordered [b][t] (t = (ci*k+ky)*k+kx), weights [c_out][ntaps] (f64),
 * bias [c_out] (may be NULL), w_used = d_out^2 slots carrying the bias.
 * maps_out: count B*c_out ordered [b][co], level l-1. */
int hegpu_conv_packed_forward(hegpu_ctx* ctx, const hegpu_ct* taps, int ntaps, const double* weights,
                              int c_out, const double* bias, int w_used, hegpu_ct* maps_out);
/* the same layer with its plaintexts (scalar weights, bias encodings)
 * prepared once: plan at tap level `level`, tap scale `tap_scale` */
typedef struct hegpu_conv_plan hegpu_conv_plan;
int hegpu_conv_plan_create(hegpu_ctx* ctx, int ntaps, const double* weights, int c_out, const double* bias,
                           int w_used, int level, double tap_scale, hegpu_conv_plan** out);
void hegpu_conv_plan_destroy(hegpu_conv_plan* plan);
int hegpu_conv_plan_run(hegpu_ctx* ctx, const hegpu_conv_plan* plan, const hegpu_ct* taps, hegpu_ct* maps_out);
/* merge_maps (convlower.cpp:145-160): maps count B*c ordered [b][j];
 * out count B; CapacityError if c*w > S */
/* conv_packed_forward with the reference's masked constant plaintexts
 * pt(w[co,t] on slots < w_used) (convlower.cpp:55-63) for taps that are NOT
 * zero beyond w_used -- the RepackConv stage's rotated group ciphertexts
 * (netcompile.cpp:352-379).  taps: ntaps * B ciphertexts TAP-MAJOR [t][b] at
 * `level`; maps: c_out * B MAP-MAJOR [co][b] at level - 1 (MAC + masked bias
 * + rescale, one kernel over every map); metered as conv_packed_forward */
typedef struct hegpu_masked_conv hegpu_masked_conv;
int hegpu_masked_conv_create(hegpu_ctx* ctx, int ntaps, const double* weights, int c_out, const double* bias,
                             int w_used, int level, double tap_scale, hegpu_masked_conv** out);
void hegpu_masked_conv_destroy(hegpu_masked_conv* plan);
int hegpu_masked_conv_run(hegpu_ctx* ctx, const hegpu_masked_conv* plan, const hegpu_ct* taps, hegpu_ct* maps);
int hegpu_merge_maps(hegpu_ctx* ctx, const hegpu_ct* maps, int c, int64_t w, hegpu_ct* out);
/* extract_diagonals (matvec.cpp:45-65) + encode, once per matrix (offline);
 * A is m x n row-major, input ciphertexts at `level` */
int hegpu_hs_plan_create(hegpu_ctx* ctx, const double* A, int m, int n, int level,
                         int skip_zero_diagonals, hegpu_hs_plan** out);
void hegpu_hs_plan_destroy(hegpu_hs_plan* plan);
/* right rotations the plan needs keys for (diagonal offsets, then folds as
 * right-rotation amounts); returns the count, fills `rots` if non-NULL */
int hegpu_hs_plan_rotations(const hegpu_hs_plan* plan, int64_t* rots, int cap);
int hegpu_hs_plan_info(const hegpu_hs_plan* plan, int* m_eff, int* folds, int* kept);
/* hs_matvec (matvec.cpp:82-105): out level = level-1 (one rescale) */
int hegpu_hs_matvec(hegpu_ctx* ctx, const hegpu_hs_plan* plan, const hegpu_ct* v, hegpu_ct* out);
/* hs_matvec split over nparts GPUs (config 3: "partial sums reduced across
 * GPUs"): part p accumulates the kept diagonals of the p-th of nparts equal
 * ranges in the extended basis into a device buffer of hegpu_hs_acc_words
 * uint64 words; the buffers are summed element-wise (e.g. NCCL all-reduce,
 * int64 sum -- entries stay < nparts * 2^60); _finish reduces the sum and
 * runs the single ModDown, the rescale and the folds.  Bit-identical to
 * hegpu_hs_matvec; metering splits the same totals over the parts. */
size_t hegpu_hs_acc_words(const hegpu_hs_plan* plan, int batch);
int hegpu_hs_matvec_partial(hegpu_ctx* ctx, const hegpu_hs_plan* plan, const hegpu_ct* v, int part, int nparts,
                            void* dev_acc);
int hegpu_hs_matvec_finish(hegpu_ctx* ctx, const hegpu_hs_plan* plan, const hegpu_ct* v, void* dev_acc,
                           int nparts, hegpu_ct* out);

/* ---- LoLa comparators (proj/src/matvec.cpp:107-211) ---------------------- */
#define HEGPU_LOLA_DENSE 0   /* lola_dense_matvec   (matvec.cpp:107-123) */
#define HEGPU_LOLA_STACKED 1 /* lola_stacked_matvec (matvec.cpp:125-166) */
/* row plaintexts + clearing masks encoded once per matrix; input at `level`
 * (>= 3), outputs at level - 2 (product rescale + the value-level clearing,
 * done as a 0/1 mask multiply that is not metered, as in the reference);
 * CapacityError if m or n > S, or (stacked) next_pow2(n) > S */
int hegpu_lola_plan_create(hegpu_ctx* ctx, int kind, const double* A, int m, int n, int level,
                           hegpu_lola_plan** out);
void hegpu_lola_plan_destroy(hegpu_lola_plan* plan);
int hegpu_lola_plan_rotations(const hegpu_lola_plan* plan, int64_t* rots, int cap);
/* delta = next_pow2(n), k rows per batch (stacked), batches, folds =
 * log2(delta), outputs per input ciphertext (dense: m, stacked: 1) */
int hegpu_lola_plan_info(const hegpu_lola_plan* plan, int* delta, int* k, int* batches, int* folds, int* per_input);
/* InterleavedResult::slot_of_row (matvec.hpp:32-36); dense rows are slot 0 */
int64_t hegpu_lola_slot_of_row(const hegpu_lola_plan* plan, int row);
/* dense: out count = B * m (image-major); stacked: out count = B.  Metering
 * per input = predict_lola_dense / predict_lola_stacked (matvec.cpp:189-211) */
int hegpu_lola_matvec(hegpu_ctx* ctx, const hegpu_lola_plan* plan, const hegpu_ct* v, hegpu_ct* out);

/* ---- stage driver: execute (proj/src/netcompile.cpp:291-446) ------------ */
/* first-layer execution (hegpu_net_spec.first_layer):
 *  REFERENCE (default, 0): the reference's stages as lower() emits them
 *    (proj/src/netcompile.cpp:321-347): the client ships k^2 c_in conv_pack
 *    tap ciphertexts (proj/src/convlower.cpp:9-37), the server runs
 *    conv_packed_forward + rescale into c_out map ciphertexts, then
 *    merge_maps with c_out - 1 key-switched rotations (convlower.cpp:145-160);
 *  FUSED (1): Conv1 + Flat1 fused by client-side replicated, region-packed
 *    taps: ceil(k^2 c_in / R) tap ciphertexts, no merge key
 *    switches, R - 1 hoisted region-fold key switches.
 * Both meter the reference's per-stage HOPs. */
enum { HEGPU_FIRST_LAYER_REFERENCE = 0, HEGPU_FIRST_LAYER_FUSED = 1 };
typedef struct {
  int in_c, in_d, k, stride, c_out;  /* first-layer conv (ConvPack stage) */
  int n_dense;                       /* Square+Dense pairs that follow */
  int dense_out[4];
  int first_layer;                   /* HEGPU_FIRST_LAYER_* */
} hegpu_net_spec;
/* weights: conv_w [c_out][in_c][k][k], conv_b [c_out], then per dense layer
 * W (row-major m x n) and b [m]; all f64 */
int hegpu_net_create(hegpu_ctx* ctx, const hegpu_net_spec* spec, const double* conv_w,
                     const double* conv_b, const double* const* dense_w,
                     const double* const* dense_b, hegpu_net** out);
void hegpu_net_destroy(hegpu_net* net);
/* device-resident run: taps = count B * hegpu_net_tap_cts(net) at the top
 * level; out = count B at level L - 1 - 2 n_dense */
int hegpu_net_run(hegpu_net* net, const hegpu_ct* taps, hegpu_ct* out);
/* config 3 across GPUs ("partial sums reduced across GPUs"): the same run,
 * but dense layer `layer`'s HS accumulates only diagonal range `part` of
 * `nparts` (hegpu_hs_matvec_partial); `reduce(dev_words, words, user)` is
 * then called with the engine stream synchronised and must replace the
 * device accumulator by the element-wise int64 sum over all parts (an NCCL
 * all-reduce; return 0 on success); every rank then finishes the layer and
 * the rest of the net identically.  Bit-identical to hegpu_net_run. */
typedef int (*hegpu_reduce_fn)(void* dev_words, size_t words, void* user);
/* layer = HEGPU_SPLIT_FIRST_LAYER splits the first layer instead (reference
 * first layer only): rank `part` runs the conv-pack MAC + rescale of output
 * maps [c_out part / nparts, c_out (part+1) / nparts) and their merge
 * rotations into disjoint slot ranges; the partial (extended-basis key
 * inner products, Q-basis part) is summed by `reduce`, then every rank runs
 * the merge's one ModDown per image and the rest of the net (SURVEY.md §8e
 * config 3: conv/merge by output map).  Bit-identical to hegpu_net_run. */
#define HEGPU_SPLIT_FIRST_LAYER (-1)
/* both splits in one run: the first layer and dense layer k (each with its
 * own reduce call, first layer first) */
#define HEGPU_SPLIT_FIRST_AND_DENSE(k) (-2 - (k))
int hegpu_net_run_split(hegpu_net* net, const hegpu_ct* taps, hegpu_ct* out, int layer, int part, int nparts,
                        hegpu_reduce_fn reduce, void* user);
/* the same on device-resident compact taps (batch x hegpu_net_compact_image_bytes
 * bytes, as hegpu_net_encrypt_image_compact writes them): the conv MAC
 * decodes c0 and regenerates c1 on the fly */
int hegpu_net_run_compact(hegpu_net* net, const void* dev_taps, int batch, hegpu_ct* out);
/* end-to-end run from host buffers (wire format taps [B][tap_cts][2][L][N]
 * -> output cts [B][2][L-1-2 n_dense][N]); includes both host<->device copies */
int hegpu_net_run_host(hegpu_net* net, const uint64_t* host_taps, int batch, uint64_t* host_out);
/* client helper: conv_pack (convlower.cpp:9-37) + encode + encrypt of one
 * image [in_c][in_d][in_d] -> hegpu_net_tap_cts(net) wire ciphertexts at the top level */
int hegpu_net_encrypt_image(hegpu_net* net, const double* image, uint64_t nonce, uint64_t* taps_out);
/* tap ciphertexts per image: k^2 c_in for the reference first layer (tap t
 * = (ci*k+ky)*k+kx carries the window on slots [0, d_out^2)), ceil(k^2 c_in / R)
 * for the fused one (R taps packed per ciphertext) */
int hegpu_net_tap_cts(const hegpu_net* net);
/* HEGPU_FIRST_LAYER_* the net was built with */
int hegpu_net_first_layer(const hegpu_net* net);
/* the same taps in compact form (hegpu_net_compact_image_bytes per image) */
size_t hegpu_net_compact_image_bytes(const hegpu_net* net);
int hegpu_net_encrypt_image_compact(hegpu_net* net, const double* image, uint64_t nonce, uint8_t* taps_out);
/* end-to-end run from compact host taps [batch][tap_cts] -> output cts (wire);
 * the batch is processed in chunks of `chunk` images (0 = automatic) with the
 * next chunk's host->device copy overlapping the current chunk's compute */
int hegpu_net_run_host_compact(hegpu_net* net, const uint8_t* host_taps, int batch, int chunk, uint64_t* host_out);
/* the same pass without waiting: returns once the work is enqueued, so the
 * next submit's host->device copies overlap this pass's compute (serving
 * loop).  host_taps and host_out must stay valid (and host_out unread) until
 * hegpu_net_wait; at most two passes may be in flight per net (staging is
 * double-buffered; a third submit queues behind the first). */
int hegpu_net_submit_host_compact(hegpu_net* net, const uint8_t* host_taps, int batch, int chunk,
                                  uint64_t* host_out);
int hegpu_net_wait(hegpu_net* net);
/* ---- model / weights / input files (proj/src/modelio.cpp:106-248) ----------
 * model JSON {"name", "input": [c, d, d], "n_slots", "layers": [{"kind",
 * "k", "s", "out_channels" | "units", "groups", "policy", "label"}]} with
 * unknown keys rejected; weights a little-endian float32 stream in layer
 * order (conv [c_out][c_in][k][k] then [c_out]; dense [m][n] then [m]);
 * inputs [c][d][d] float32.  Errors: HEGPU_ERR_IO (hesim::IoError). */
typedef struct hegpu_model hegpu_model;
enum {
  HEGPU_LAYER_CONV = 0, HEGPU_LAYER_SUBCONV = 1, HEGPU_LAYER_AVGPOOL = 2,
  HEGPU_LAYER_SQUARE = 3, HEGPU_LAYER_FLATTEN = 4, HEGPU_LAYER_DENSE = 5
};
enum {
  HEGPU_POLICY_CONVPACK = 0, HEGPU_POLICY_HS = 1, HEGPU_POLICY_LOLA_DENSE = 2, HEGPU_POLICY_LOLA_STACKED = 3
};
int hegpu_model_parse(const char* json_text, hegpu_model** out);       /* parse_model_json */
int hegpu_model_load(const char* name_or_path, hegpu_model** out);      /* resolve_model ($HECNN_MODEL_DIR) */
const char* hegpu_model_last_error(const hegpu_model* model);          /* NULL: last parse/load failure */
void hegpu_model_destroy(hegpu_model* model);
int hegpu_model_info(const hegpu_model* model, int* in_c, int* in_d, int* n_slots, int* n_layers,
                     size_t* weight_floats);
/* policy = -1 when the layer names none */
int hegpu_model_layer(const hegpu_model* model, int i, int* kind, int* k, int* s, int* out, int* groups,
                      int* policy);
/* ModelSpec::default_policy (netcompile.hpp:33-35; the reference CLI's
 * --policy, hesim.cpp:43-48): the kernel of linear stages without a per-layer
 * policy (HEGPU_POLICY_HS / _LOLA_DENSE / _LOLA_STACKED); and --n-slots */
int hegpu_model_set_default_policy(hegpu_model* model, int policy);
int hegpu_model_set_n_slots(hegpu_model* model, int n_slots);
int hegpu_model_load_weights(hegpu_model* model, const char* path, double* out, size_t count); /* load_weights */
int hegpu_model_save_weights(hegpu_model* model, const char* path, const double* w, size_t count);
int hegpu_model_load_input(hegpu_model* model, const char* path, double* out);   /* load_input */
int hegpu_model_save_input(hegpu_model* model, const char* path, const double* x);
/* lower() for model files (proj/src/netcompile.cpp:106-278): a first
 * conv-pack conv, then Square stages alternating with maximal linear runs
 * (conv / avgpool / flatten / dense), each run's affine map composed on the
 * host (conv_to_matrix, pool_to_matrix, dense; FP64) into one HS layer
 * labelled by its joined layer labels.  HEGPU_ERR_SHAPE outside this family
 * (SubConv groups, RepackConv, LoLa policies: those run through hegpu_prog
 * below).  _net_spec gives the shapes;
 * _compose the composed M (rows x cols, row-major; may be NULL to query the
 * size) and bias b of linear stage `stage` from a flat weights stream. */
int hegpu_model_net_spec(const hegpu_model* model, hegpu_net_spec* spec);
int hegpu_model_compose(hegpu_model* model, const double* weights, size_t count, int stage, double* M, double* b,
                        int* rows, int* cols);
int hegpu_net_create_from_model(hegpu_ctx* ctx, hegpu_model* model, const char* weights_path, hegpu_net** out);
/* logits: decrypt + decode output ct (wire) into m_last values */
int hegpu_net_decrypt_logits(hegpu_net* net, const uint64_t* out_ct, double* logits);
double hegpu_net_output_scale(const hegpu_net* net);

/* ---- the general stage driver: lower() + execute() for every stage kind ----
 * (proj/src/netcompile.cpp:106-213 lower, :291-446 execute): ConvPack,
 * Merge into `groups` ciphertexts, Square, RepackConv (a stand-alone 1x1
 * conv-pack conv on rotated group ciphertexts, :352-379) and Linear runs
 * per channel group (SubConv, :380-434) under the HS or LoLa-dense policy;
 * a model without a first conv-pack conv is seeded with one dense input
 * ciphertext (:309-319).  Every stage executes the
 * C-ABI operators above (conv_plan_run, merge_maps, square, rotate_left,
 * mul_plain/add/add_plain/rescale with the reference's masked constants,
 * hs_matvec, lola_matvec) under hegpu_begin_stage(label), so the per-stage
 * HOP report is the reference's.  LoLa-stacked stages are rejected
 * (HEGPU_ERR_SHAPE): the reference de-interleaves their result on cleartext
 * values (:409-417), which has no homomorphic counterpart.
 * Levels: the context's chain must hold 1 + (primes consumed) limbs:
 * ConvPack, RepackConv, Square and Linear(HS) consume one prime each,
 * Linear(LoLa-dense) two (HEGPU_ERR_CAPACITY otherwise); the model's
 * n_slots must equal the context's slot count. */
typedef struct hegpu_prog hegpu_prog;
enum {
  HEGPU_STAGE_CONVPACK = 0, HEGPU_STAGE_MERGE = 1, HEGPU_STAGE_SQUARE = 2, HEGPU_STAGE_REPACKCONV = 3,
  HEGPU_STAGE_LINEAR = 4
};
/* weights: the flat stream of hegpu_model_load_weights (count values) */
int hegpu_prog_create(hegpu_ctx* ctx, const hegpu_model* model, const double* weights, size_t count,
                      hegpu_prog** out);
void hegpu_prog_destroy(hegpu_prog* prog);
/* stages, input ciphertexts per image (k^2 c_in conv_pack taps, or 1), the
 * output level and the number of logits */
int hegpu_prog_info(const hegpu_prog* prog, int* n_stages, int* input_cts, int* out_level, int* n_logits);
int hegpu_prog_stage(const hegpu_prog* prog, int i, char* label, int label_len, int* kind, int* groups,
                     int* policy);
/* lower() alone (no context): the stage list of a model; label/kind/groups/
 * policy arrays of capacity cap, returns the stage count or a negative error */
int hegpu_model_lower(const hegpu_model* model, int cap, char (*labels)[64], int* kinds, int* groups,
                      int* policies);
/* client: conv_pack (or the dense input vector) -> encode + encrypt at the
 * top level; input_cts wire ciphertexts, nonces nonce * input_cts + t */
int hegpu_prog_encrypt_input(hegpu_prog* prog, const double* image, uint64_t nonce, uint64_t* cts_out);
/* input: B x input_cts ciphertexts (image-major, as hegpu_prog_encrypt_input
 * writes them image after image) at the top level; out: B ciphertexts at
 * out_level.  Grouped stages run one batched operator call per group. */
int hegpu_prog_run(hegpu_prog* prog, hegpu_ct* input, hegpu_ct* out);
int hegpu_prog_decrypt_logits(hegpu_prog* prog, const uint64_t* out_ct, double* logits);
double hegpu_prog_output_scale(const hegpu_prog* prog);
/* prog == NULL: the last hegpu_prog_create / hegpu_model_lower error of this thread */
const char* hegpu_prog_last_error(const hegpu_prog* prog);

#ifdef __cplusplus
}
#endif
#endif /* HEGPU_H */
