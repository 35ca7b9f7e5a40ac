// conv_tc.cu -- the conv-pack MAC (conv_packed_forward, proj/src/convlower.cpp:39-74)
// on the 5th-generation tensor cores: tcgen05.mma.kind::i8 with the
// accumulator in tensor memory.
//
// Per (image b, poly p, limb t) the MAC out[co][k] = sum_s W[co][s] tap_s[k]
// (+ bias) mod q_t is an exact byte-plane GEMM with the positions k as M:
//   A[k][(s, i)]        = byte i of tap_s[k]                  (M = 128 positions, K = 8 ntaps)
//   B[(s, i)][(co, e)]  = byte e of w'[co][s][i] = W[co][s] 2^(8i) R mod q_t
//   C[k][(co, e)]       = sum_(s,i) A B < 2^26 (exact, s32)
//   out[co][k]          = mont_reduce(sum_e C 2^(8e) (+ bias R)) = sum_s W tap_s + bias
// so every (co, k) is combined by ONE thread from its own TMEM lane (the
// positions are the TMEM lanes, the weight byte planes e are columns): no
// cross-lane epilogue.  The K dimension keeps the tap words whole, so A is
// staged from the tap ciphertexts with 16-byte shared-memory stores (two
// taps' words per core-matrix row) and no byte shuffling; the weight
// operand B (the canonical K-major core-matrix image, built once per plan)
// is copied in per CTA.  One thread issues the MMAs (K = 32 per
// instruction), tcgen05.commit arrives on an mbarrier, the epilogue warps
// read the accumulator with tcgen05.ld.  Two accumulator and three A
// buffers: the MMA of tile i overlaps the epilogue of tile i - 1 and the
// cp.async staging of tiles i + 1, i + 2.  Limbs are the same residues as the IMAD / mma.sync paths.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "engine.hpp"

namespace hegpu {

namespace {

constexpr int kTcM = 128;       // positions per tile (MMA M)
constexpr int kTcThreads = 256;  // 8 warps: all stage, warps w and w + 4 share TMEM lanes 32 (w % 4)
constexpr int kTcTiles = 16;     // position tiles per CTA (HEGPU_TC_TILES)
constexpr int kTcBufs = 3;       // A (tap) tile buffers in flight (HEGPU_TC_BUFS, 2..4)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory matrix descriptor: K-major, no swizzle (core matrices
// of 8 rows x 16 bytes), lbo = byte stride between K-adjacent core
// matrices, sbo = between M/N-adjacent ones; version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor, kind::i8: D s32, A and B unsigned 8-bit, both K-major
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N) {
  return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tc_mma_u8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
// 8 consecutive accumulator columns of this thread's TMEM lane
__device__ __forceinline__ void tc_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

struct TcArgs {
  PrimeTable pt;
  const u64d* taps;   // [B][ntaps][2][l][N] device slot order
  const uint4* wb;    // [l][kb * npad bytes / 16] B operand images (K-major core matrices)
  const u64d* bias;   // [c_out][l][N] Montgomery (poly 0), or null
  u64d* out;          // [B][c_out][2][l][N]
  int B, ntaps, l, N, c_out;
  int kb;             // K bytes per row = 8 * ntaps rounded up to 32
  int npad[8];        // per limb: MMA N (c_out * planes rounded up to 16)
  int planes[8];      // per limb: weight byte planes (bytes of q_t)
  int nb;             // TMEM columns per accumulator buffer
  int tcols;          // TMEM columns allocated
  int chunks;         // CTAs per (b, p, t) row
  int nbufs;          // A tile buffers
};

__global__ void __launch_bounds__(kTcThreads, 1) k_conv_tc(TcArgs a) {
  extern __shared__ __align__(128) uint8_t tc_smem[];
  __shared__ __align__(8) uint64_t bars[2];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = a.N, l = a.l, KB = a.kb;
  const int chunk = blockIdx.x % a.chunks, row = blockIdx.x / a.chunks;
  const int t = row % l, bp = row / l, p = bp & 1, b = bp >> 1;
  const int npad = a.npad[t], PL = a.planes[t];
  const int ntile_all = N / kTcM;
  const int tile0 = chunk * ntile_all / a.chunks, tile1 = (chunk + 1) * ntile_all / a.chunks;
  // shared memory: A[kTcBufs] (kTcM x KB bytes each), then B (npad x KB bytes)
  uint8_t* sA = tc_smem;
  uint8_t* sB = tc_smem + a.nbufs * (size_t)kTcM * KB;
  const uint32_t sA_u = smem_u32(sA), sB_u = smem_u32(sB);
  const uint32_t bar0 = smem_u32(&bars[0]);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                 "r"(a.tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // the weight operand of limb t (K-major core-matrix image, npad x KB bytes)
  {
    const uint4* src = a.wb + (size_t)t * (KB * 256 / 16);  // images are laid out at npad = 256 stride
    uint4* dst = reinterpret_cast<uint4*>(sB);
    for (int i = tid; i < npad * KB / 16; i += kTcThreads) dst[i] = __ldg(src + i);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const uint32_t idesc = idesc_u8(kTcM, npad);
  // A core matrices: [K chunk c][position group g (16)][8 rows][16 B]
  const uint32_t a_lbo = 16 * 128, a_sbo = 128;
  // B core matrices: [K chunk c][column group (npad / 8)][8 rows][16 B]
  const uint32_t b_lbo = (uint32_t)(npad / 8) * 128, b_sbo = 128;
  const size_t ct_words = (size_t)2 * l * N;
  const u64d* tbase = a.taps + (size_t)b * a.ntaps * ct_words + (size_t)p * l * N + (size_t)t * N;
  const int npairs = KB / 16;  // tap pairs (16 K bytes each), incl. zero padding
  const DevPrime pr = a.pt.p[t];
  const int lane_grp = warp & 3;  // TMEM lanes 32 lane_grp .. (this warp's positions)
  const int pos = 32 * lane_grp + lane;
  // tile staging: cp.async copies of the tap words straight into the
  // core-matrix rows (no register round trip), three A buffers in flight;
  // the zero padding (taps >= ntaps) is written once per buffer
  const int NBF = a.nbufs;
  auto a_buf = [&](int k) { return sA + (size_t)(k % NBF) * kTcM * KB; };
  for (int bf = 0; bf < NBF; ++bf)
    for (int idx = tid; idx < npairs * kTcM; idx += kTcThreads) {
      const int sp = idx / kTcM, j = idx % kTcM, s = 2 * sp;
      uint64_t* row = reinterpret_cast<uint64_t*>(a_buf(bf) + ((size_t)(sp * 16 + (j >> 3)) * 8 + (j & 7)) * 16);
      if (s >= a.ntaps) row[0] = 0;
      if (s + 1 >= a.ntaps) row[1] = 0;
    }
  auto issue = [&](int it) {
    if (it < tile1) {
      uint8_t* A = a_buf(it - tile0);
      const int k0 = it * kTcM;
      for (int idx = tid; idx < npairs * kTcM; idx += kTcThreads) {
        const int sp = idx / kTcM, j = idx % kTcM, s = 2 * sp;
        const uint32_t dst = smem_u32(A + ((size_t)(sp * 16 + (j >> 3)) * 8 + (j & 7)) * 16);
        if (s < a.ntaps) cp_async8(dst, tbase + (size_t)s * ct_words + k0 + j);
        if (s + 1 < a.ntaps) cp_async8(dst + 8, tbase + (size_t)(s + 1) * ct_words + k0 + j);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  for (int d = 0; d < NBF - 1; ++d) issue(tile0 + d);
  for (int it = tile0; it <= tile1; ++it) {
    const int k = it - tile0;
    if (it < tile1) {
      // this thread's rows of tile it landed (NBF - 2 later groups may pend)
      if (NBF == 2) asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      else if (NBF == 3) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
      else asm volatile("cp.async.wait_group 2;\n" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (it < tile1 && tid == 0) {
      // ---- MMA issue (one thread): K in steps of 32 bytes = 2 core-matrix chunks
      const uint32_t a0 = sA_u + (uint32_t)((k % NBF) * kTcM * KB), d = tmem + (uint32_t)((k & 1) * a.nb);
      for (int ks = 0; ks < KB / 32; ++ks) {
        const uint64_t ad = umma_desc(a0 + (uint32_t)ks * 2 * a_lbo, a_lbo, a_sbo);
        const uint64_t bd = umma_desc(sB_u + (uint32_t)ks * 2 * b_lbo, b_lbo, b_sbo);
        tc_mma_u8(d, ad, bd, idesc, ks > 0);
      }
      tc_commit(bar0 + 8 * (k & 1));
    }
    if (k >= 1) {
      // ---- epilogue of tile it - 1: position pos, maps co = warp / 4 (mod 2)
      const int kp = k - 1, buf = kp & 1;
      mbar_wait(bar0 + 8 * buf, (uint32_t)((kp >> 1) & 1));
      tc_fence_after();
      const int kpos = (it - 1) * kTcM + pos;
      const uint32_t lanebase = tmem + ((uint32_t)(32 * lane_grp) << 16) + (uint32_t)(buf * a.nb);
      for (int co = warp >> 2; co < a.c_out; co += 2) {
        uint32_t r[8];
        tc_ld8(lanebase + (uint32_t)(co * PL), r);
        u64d lo = (p == 0 && a.bias) ? __ldg(a.bias + ((size_t)co * l + t) * N + kpos) : 0ull, hi = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e >= PL) break;
          const u64d v = (u64d)r[e];
          const u64d l_add = v << (8 * e), h_add = e ? v >> (64 - 8 * e) : 0ull;
          asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(l_add), "l"(h_add));
        }
        a.out[((size_t)b * a.c_out + co) * ct_words + (size_t)p * l * N + (size_t)t * N + kpos] =
            mont_reduce128(lo, hi, pr.q, pr.qneg_inv);
      }
      tc_fence_before();
    }
    // refill: buffer (k + NBF - 1) % NBF held tile it - 1, whose MMA the
    // epilogue above has waited for
    issue(it + NBF - 1);
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(a.tcols) : "memory");
  }
}

int planes_of(u64 q) {
  int n = 0;
  while (n < 8 && (q >> (8 * n)) != 0) ++n;
  return n;
}

}  // namespace

bool conv_tc_enabled() {
  const char* e = getenv("HEGPU_CONV_TC");
  return !(e && e[0] == '0');
}

bool conv_tc_supported(Context& c, int ntaps, int c_out, int l) {
  if (!conv_tc_enabled() || c.N() % kTcM != 0 || l > 8) return false;
  const int kb = (8 * ntaps + 31) / 32 * 32;
  for (int t = 0; t < l; ++t) {
    const int pl = planes_of(c.P->q(t));
    if (c_out * pl > 256) return false;
  }
  // A buffers + B at the widest limb
  const size_t sm = kTcBufs * (size_t)kTcM * kb + (size_t)kb * 256;
  return sm <= 200 * 1024;
}

// B operand images: per limb, [K chunk][column group][8 rows][16 B] with
// column n = co * planes + e, K byte kappa = 8 s + i: byte e of ws[co][s][i]
// (ws[li][co][s][i] = W[co][s] * 2^(8 i) * R mod q_li, layers.cu); laid out
// at a fixed 256-column stride per limb (the kernel copies npad columns)
std::vector<uint8_t> conv_tc_weights(Context& c, int ntaps, int c_out, int l, const std::vector<u64>& ws) {
  const int kb = (8 * ntaps + 31) / 32 * 32;
  std::vector<uint8_t> img((size_t)l * kb * 256, 0);
  for (int li = 0; li < l; ++li) {
    const int pl = planes_of(c.P->q(li));
    const int npad = (c_out * pl + 15) / 16 * 16, ng = npad / 8;
    uint8_t* base = img.data() + (size_t)li * kb * 256;
    for (int co = 0; co < c_out; ++co)
      for (int e = 0; e < pl; ++e) {
        const int n = co * pl + e;
        for (int s = 0; s < ntaps; ++s)
          for (int i = 0; i < 8; ++i) {
            const int kappa = 8 * s + i, ch = kappa / 16;
            const u64 w = ws[(((size_t)li * c_out + co) * ntaps + s) * 8 + i];
            base[((size_t)(ch * ng + n / 8) * 8 + n % 8) * 16 + kappa % 16] = (uint8_t)(w >> (8 * e));
          }
      }
  }
  return img;
}

void launch_conv_tc(Context& c, const u64d* taps, int B, int ntaps, int l, const uint8_t* wb, int c_out,
                    const u64d* bias, u64d* out) {
  TcArgs a{};
  a.pt = c.primes;
  a.taps = taps;
  a.wb = reinterpret_cast<const uint4*>(wb);
  a.bias = bias;
  a.out = out;
  a.B = B;
  a.ntaps = ntaps;
  a.l = l;
  a.N = c.N();
  a.c_out = c_out;
  a.kb = (8 * ntaps + 31) / 32 * 32;
  int maxn = 16;
  for (int t = 0; t < l; ++t) {
    a.planes[t] = planes_of(c.P->q(t));
    a.npad[t] = (c_out * a.planes[t] + 15) / 16 * 16;
    maxn = std::max(maxn, a.npad[t]);
  }
  a.nb = maxn + 8;  // 8 spare columns: the epilogue reads 8 from co * planes
  int cols = 32;
  while (cols < 2 * a.nb) cols *= 2;
  a.tcols = cols;
  const int ntile = c.N() / kTcM;
  const char* et = getenv("HEGPU_TC_TILES");
  const char* eb = getenv("HEGPU_TC_BUFS");
  const int tiles = et ? std::max(1, atoi(et)) : kTcTiles;
  a.nbufs = eb ? std::min(4, std::max(2, atoi(eb))) : kTcBufs;
  a.chunks = std::max(1, ntile / tiles);
  size_t sm = (size_t)a.nbufs * kTcM * a.kb + (size_t)a.kb * maxn;
  if (sm > 200 * 1024) {
    a.nbufs = kTcBufs;
    sm = (size_t)a.nbufs * kTcM * a.kb + (size_t)a.kb * maxn;
  }
  static PerDeviceOnce prepared;
  if (prepared.first())
    CK(cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const int N = c.N();
  const double bytes = 8.0 * N * l * (2.0 * B * ntaps + 2.0 * B * c_out + c_out);
  const double ops = 2.0 * N * l * B * ntaps * c_out;
  LAUNCH_BO(c, "k_conv_mac", bytes, ops,
            k_conv_tc<<<B * 2 * l * a.chunks, kTcThreads, sm, c.stream>>>(a));
}

}  // namespace hegpu
