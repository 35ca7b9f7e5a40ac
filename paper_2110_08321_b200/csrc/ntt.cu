// ntt.cu -- batched negacyclic NTT / INTT over 64-bit primes (sm_100a).
//
// One CTA transforms one N-word limb entirely in shared memory (N <= 16384:
// 128 KB).  Forward: Cooley-Tukey with psi powers in bit-reversed order and
// Shoup twiddle products; inverse: Gentleman-Sande.  Loads/stores fuse the
// surrounding RNS steps so every limb crosses HBM once per transform:
//   - forward stores scatter into the device SLOT ORDER (engine.hpp);
//   - the key-switch INTT loads apply the Galois shift on the fly;
//   - ModUp loads reduce a digit mod the target prime;
//   - the drop-limb NTT (rescale / ModDown) lifts the dropped residue,
//     transforms it and finishes (x - X) * q_d^{-1} (+ add term) in the store.
#include "engine.hpp"

namespace hegpu {

namespace {

__device__ __forceinline__ int ntt_threads(int N) { return N / 2 < 512 ? N / 2 : 512; }

// forward CT in smem (natural in, bit-reversed out)
__device__ __forceinline__ void fwd_core(u64d* a, int N, int logN, const u64d* __restrict__ w,
                                         const u64d* __restrict__ wp, u64d q) {
  const int half = N >> 1;
  for (int lt = logN - 1, m = 1; lt >= 0; --lt, m <<= 1) {
    const int tmask = (1 << lt) - 1;
    for (int b = threadIdx.x; b < half; b += blockDim.x) {
      const int i = b >> lt, j = b & tmask;
      const int x = (i << (lt + 1)) + j, y = x + (1 << lt);
      const u64d W = __ldg(w + m + i), Wp = __ldg(wp + m + i);
      const u64d U = a[x], V = shoup_mul_d(a[y], W, Wp, q);
      a[x] = add_mod_d(U, V, q);
      a[y] = sub_mod_d(U, V, q);
    }
    __syncthreads();
  }
}

// inverse GS in smem (bit-reversed in, natural out, without the N^{-1})
__device__ __forceinline__ void inv_core(u64d* a, int N, const u64d* __restrict__ iw,
                                         const u64d* __restrict__ iwp, u64d q) {
  const int half = N >> 1;
  for (int lt = 0, h = half; h >= 1; ++lt, h >>= 1) {
    const int tmask = (1 << lt) - 1;
    for (int b = threadIdx.x; b < half; b += blockDim.x) {
      const int i = b >> lt, j = b & tmask;
      const int x = (i << (lt + 1)) + j, y = x + (1 << lt);
      const u64d W = __ldg(iw + h + i), Wp = __ldg(iwp + h + i);
      const u64d U = a[x], V = a[y];
      a[x] = add_mod_d(U, V, q);
      a[y] = shoup_mul_d(sub_mod_d(U, V, q), W, Wp, q);
    }
    __syncthreads();
  }
}

// slot position p after a left rotation by s (inside each half)
__device__ __forceinline__ int shifted(int p, int s, int S) {
  const int h = p >= S ? S : 0;
  int j = p - h + s;
  if (j >= S) j -= S;
  return h + j;
}

struct TwArgs {
  const u64d* tw;
  const u64d* ninv;       // [np][2]
  const uint32_t* slot_src;
  int N, logN;
};

__device__ __forceinline__ const u64d* tw_of(const TwArgs& t, int pi, int which) {
  return t.tw + ((size_t)pi * 4 + which) * t.N;
}

// --------------------------------------------------------------------------
__global__ void k_ntt_rows(TwArgs ta, PrimeTable pt, const u64d* __restrict__ src,
                           u64d* __restrict__ dst, int nl, int p_limb, int p_index) {
  extern __shared__ u64d sm[];
  const int N = ta.N, r = blockIdx.x, limb = r % nl;
  const int pi = (limb == p_limb) ? p_index : limb;
  const u64d q = pt.p[pi].q;
  const u64d* s = src + (size_t)r * N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) sm[k] = s[k];
  __syncthreads();
  fwd_core(sm, N, ta.logN, tw_of(ta, pi, 0), tw_of(ta, pi, 1), q);
  u64d* d = dst + (size_t)r * N;
  for (int p = threadIdx.x; p < N; p += blockDim.x) d[p] = sm[__ldg(ta.slot_src + p)];
}

struct PMap {
  int8_t p[HEGPU_MAX_PRIMES];
};

__global__ void k_intt_rows(TwArgs ta, PrimeTable pt, const u64d* __restrict__ src,
                            u64d* __restrict__ dst, int n_inner, long so, long si, long dox,
                            long di, PMap pm) {
  extern __shared__ u64d sm[];
  const int N = ta.N;
  const int r = blockIdx.x, o = r / n_inner, i = r % n_inner;
  const int pi = pm.p[i];
  const u64d q = pt.p[pi].q;
  const u64d* s = src + o * so + i * si;
  for (int p = threadIdx.x; p < N; p += blockDim.x) sm[__ldg(ta.slot_src + p)] = s[p];
  __syncthreads();
  inv_core(sm, N, tw_of(ta, pi, 2), tw_of(ta, pi, 3), q);
  const u64d nv = ta.ninv[2 * pi], nvp = ta.ninv[2 * pi + 1];
  u64d* d = dst + o * dox + i * di;
  for (int k = threadIdx.x; k < N; k += blockDim.x) d[k] = shoup_mul_d(sm[k], nv, nvp, q);
}

// KS input: digit j of (shifted) poly b -> coefficient row tmp[b][j]; also
// writes the shifted NTT-form limb into D[b][j][j] (ModUp's own-prime row).
__global__ void k_ks_intt(TwArgs ta, PrimeTable pt, const u64d* __restrict__ src, long src_stride,
                          int l, KeyRowMap km, int use_shift, u64d* __restrict__ tmp,
                          u64d* __restrict__ D) {
  extern __shared__ u64d sm[];
  const int N = ta.N, S = N >> 1;
  const int r = blockIdx.x, b = r / l, j = r % l;
  const int s = use_shift ? km.shift[b % km.period] : 0;
  const u64d q = pt.p[j].q;
  const u64d* in = src + b * src_stride + (size_t)j * N;
  u64d* own = D + (((size_t)b * l + j) * (l + 1) + j) * N;
  for (int p = threadIdx.x; p < N; p += blockDim.x) {
    const u64d v = in[s ? shifted(p, s, S) : p];
    own[p] = v;
    sm[__ldg(ta.slot_src + p)] = v;
  }
  __syncthreads();
  inv_core(sm, N, tw_of(ta, j, 2), tw_of(ta, j, 3), q);
  const u64d nv = ta.ninv[2 * j], nvp = ta.ninv[2 * j + 1];
  u64d* d = tmp + ((size_t)b * l + j) * N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) d[k] = shoup_mul_d(sm[k], nv, nvp, q);
}

// ModUp: rows (b, j, t') with t = t' < j ? t' : t'+1 over the extended basis
// (t == l means P); NTT_t(tmp[b][j] mod q_t) -> D[b][j][t]
__global__ void k_ks_modup(TwArgs ta, PrimeTable pt, const u64d* __restrict__ tmp, int l, int P_index,
                           u64d* __restrict__ D) {
  extern __shared__ u64d sm[];
  const int N = ta.N;
  const int r = blockIdx.x;
  const int tp = r % l, bj = r / l, j = bj % l, b = bj / l;
  const int t = tp < j ? tp : tp + 1;
  const int pi = t == l ? P_index : t;
  const DevPrime pr = pt.p[pi];
  const u64d* s = tmp + ((size_t)b * l + j) * N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) sm[k] = reduce64(s[k], pr);
  __syncthreads();
  fwd_core(sm, N, ta.logN, tw_of(ta, pi, 0), tw_of(ta, pi, 1), pr.q);
  u64d* d = D + (((size_t)b * l + j) * (l + 1) + t) * N;
  for (int p = threadIdx.x; p < N; p += blockDim.x) d[p] = sm[__ldg(ta.slot_src + p)];
}

// drop-limb NTT: rows (b, p, t < nl)
__global__ void k_drop_ntt(TwArgs ta, PrimeTable pt, const u64d* __restrict__ qinv, int np_all,
                           DropArgs a, const u64d* __restrict__ tmpP, KeyRowMap km, int use_shift) {
  extern __shared__ u64d sm[];
  const int N = ta.N, S = N >> 1;
  const int r = blockIdx.x;
  const int t = r % a.nl, bp = r / a.nl, p = bp % 2, b = bp / 2;
  const DevPrime pr = pt.p[t];
  const u64d q = pr.q, qd = pt.p[a.pd].q, half = qd >> 1;
  const u64d* s = tmpP + ((size_t)b * 2 + p) * N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const u64d x = s[k];
    sm[k] = x > half ? sub_mod_d(0, reduce64(qd - x, pr), q) : reduce64(x, pr);
  }
  __syncthreads();
  fwd_core(sm, N, ta.logN, tw_of(ta, t, 0), tw_of(ta, t, 1), q);
  const u64d iv = qinv[((size_t)t * np_all + a.pd) * 2], ivp = qinv[((size_t)t * np_all + a.pd) * 2 + 1];
  const u64d* in = a.src + b * a.src_b + p * a.src_p + (size_t)t * N;
  u64d* out = a.dst + b * a.dst_b + p * a.dst_p + (size_t)t * N;
  const bool add = (a.add_mask >> p) & 1;
  const u64d* ad = add ? a.add + b * a.add_b + p * a.add_p + (size_t)t * N : nullptr;
  const int sh = (use_shift && p == 0) ? km.shift[b % km.period] : 0;
  for (int pos = threadIdx.x; pos < N; pos += blockDim.x) {
    u64d v = shoup_mul_d(sub_mod_d(in[pos], sm[__ldg(ta.slot_src + pos)], q), iv, ivp, q);
    if (add) v = add_mod_d(v, ad[sh ? shifted(pos, sh, S) : pos], q);
    out[pos] = v;
  }
}

// wire (bit-reversed) <-> slot order, optional Montgomery conversion
__global__ void k_wire_to_slot(const u64d* __restrict__ src, u64d* __restrict__ dst,
                               const uint32_t* __restrict__ slot_src, PrimeTable pt, int N, int to_mont,
                               int nl, int p_limb, int p_index) {
  const size_t r = blockIdx.y;
  const int limb = (int)(r % nl);
  const DevPrime pr = pt.p[limb == p_limb ? p_index : limb];
  const u64d* s = src + r * N;
  u64d* d = dst + r * N;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    u64d v = s[__ldg(slot_src + p)];
    d[p] = to_mont ? mont_mul(v, pr.r2_mod, pr.q, pr.qneg_inv) : v;
  }
}

__global__ void k_slot_to_wire(const u64d* __restrict__ src, u64d* __restrict__ dst,
                               const uint32_t* __restrict__ slot_src, PrimeTable pt, int N, int from_mont,
                               int nl, int p_limb, int p_index) {
  const size_t r = blockIdx.y;
  const int limb = (int)(r % nl);
  const DevPrime pr = pt.p[limb == p_limb ? p_index : limb];
  const u64d* s = src + r * N;
  u64d* d = dst + r * N;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < N; p += gridDim.x * blockDim.x) {
    u64d v = s[p];
    d[__ldg(slot_src + p)] = from_mont ? mont_mul(v, 1ull, pr.q, pr.qneg_inv) : v;
  }
}

TwArgs tw_args(Context& c) {
  return TwArgs{c.d_tw, c.ninv_tab(), c.d_slot_src, c.N(), c.P->log_n};
}

int threads_for(int N) { return N / 2 < 512 ? N / 2 : 512; }

template <typename K>
void set_smem(K kernel, size_t bytes) {
  static size_t done = 0;
  if (bytes > 48 * 1024 && bytes > done) {
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    done = bytes;
  }
}

}  // namespace

void launch_ntt_rows(Context& c, const u64d* src, u64d* dst, int rows, int nl, int p_limb) {
  if (rows <= 0) return;
  const size_t sm = (size_t)c.N() * 8;
  set_smem(k_ntt_rows, sm);
  k_ntt_rows<<<rows, threads_for(c.N()), sm, c.stream>>>(tw_args(c), c.primes, src, dst, nl, p_limb, c.L());
  c.launches++;
  CK(cudaGetLastError());
}

void launch_intt_rows(Context& c, const u64d* src, u64d* dst, int n_outer, int n_inner, long so, long si,
                      long dox, long di, const int* prime_of_inner) {
  if (n_outer * n_inner <= 0) return;
  if (n_inner > HEGPU_MAX_PRIMES) fail(HEGPU_ERR_ARG, "intt_rows: too many limbs");
  PMap pm{};
  for (int i = 0; i < n_inner; ++i) pm.p[i] = (int8_t)prime_of_inner[i];
  const size_t sm = (size_t)c.N() * 8;
  set_smem(k_intt_rows, sm);
  k_intt_rows<<<n_outer * n_inner, threads_for(c.N()), sm, c.stream>>>(
      tw_args(c), c.primes, src, dst, n_inner, so, si, dox, di, pm);
  c.launches++;
  CK(cudaGetLastError());
}

void launch_wire_to_slot(Context& c, const u64d* src, u64d* dst, size_t rows, int to_mont, int nl, int p_limb) {
  if (!rows) return;
  dim3 grid((c.N() + 255) / 256 < 8 ? (c.N() + 255) / 256 : 8, (unsigned)rows);
  k_wire_to_slot<<<grid, 256, 0, c.stream>>>(src, dst, c.d_slot_src, c.primes, c.N(), to_mont, nl, p_limb, c.L());
  c.launches++;
  CK(cudaGetLastError());
}

void launch_slot_to_wire(Context& c, const u64d* src, u64d* dst, size_t rows, int from_mont, int nl, int p_limb) {
  if (!rows) return;
  dim3 grid((c.N() + 255) / 256 < 8 ? (c.N() + 255) / 256 : 8, (unsigned)rows);
  k_slot_to_wire<<<grid, 256, 0, c.stream>>>(src, dst, c.d_slot_src, c.primes, c.N(), from_mont, nl, p_limb, c.L());
  c.launches++;
  CK(cudaGetLastError());
}

void ks_modup(Context& c, const u64d* src, long src_stride, int B, int l, const KeyRowMap* shifts,
              u64d* tmp, u64d* D) {
  const size_t sm = (size_t)c.N() * 8;
  KeyRowMap dummy{};
  dummy.period = 1;
  set_smem(k_ks_intt, sm);
  k_ks_intt<<<B * l, threads_for(c.N()), sm, c.stream>>>(tw_args(c), c.primes, src, src_stride, l,
                                                          shifts ? *shifts : dummy, shifts != nullptr, tmp, D);
  c.launches++;
  CK(cudaGetLastError());
  if (B * l * l > 0) {
    set_smem(k_ks_modup, sm);
    k_ks_modup<<<B * l * l, threads_for(c.N()), sm, c.stream>>>(tw_args(c), c.primes, tmp, l, c.L(), D);
    c.launches++;
    CK(cudaGetLastError());
  }
}

void drop_last_limb(Context& c, int B, const DropArgs& a, u64d* tmpP) {
  const int N = c.N();
  // INTT of the dropped limb of both polys -> tmpP[b][p]
  const int pmap[2] = {a.pd, a.pd};
  launch_intt_rows(c, a.src + (size_t)(a.src_limbs - 1) * N, tmpP, B, 2, a.src_b, a.src_p, 2L * N, N, pmap);
  if (a.nl <= 0) return;
  const size_t sm = (size_t)N * 8;
  KeyRowMap dummy{};
  dummy.period = 1;
  set_smem(k_drop_ntt, sm);
  k_drop_ntt<<<B * 2 * a.nl, threads_for(N), sm, c.stream>>>(tw_args(c), c.primes, c.qinv_tab(), c.P->np(), a,
                                                            tmpP, a.shifts ? *a.shifts : dummy,
                                                            a.shifts != nullptr);
  c.launches++;
  CK(cudaGetLastError());
}

}  // namespace hegpu
