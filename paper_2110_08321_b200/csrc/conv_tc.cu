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
constexpr int kTcThreads = 288;  // 9 warps: 4 producers, 1 MMA issuer, 4 epilogue
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
// try_wait with a suspend-time hint: a waiting warp is parked until the
// phase completes (or the hint expires) instead of spinning on issue slots
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(bar),
      "r"(parity), "r"(0x989680u)
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
  int kcb;            // K bytes per A buffer (a K chunk; kb when the whole row fits)
  int nkc;            // K chunks per tile
};

// Warp roles (9 warps): 0-3 producers (thread j stages position j of a
// tile: its tap words by cp.async into the core-matrix rows), 4 the MMA
// issuer (one lane), 5-8 the epilogue (warp w reads TMEM lanes 32 (w % 4)).
// mbarriers: full[buf] (128 producer arrivals, after each producer's
// cp.async.wait + proxy fence), empty[buf] and tfull[tb] (tcgen05.commit),
// tempty[tb] (128 epilogue arrivals) -- no CTA-wide barrier in the loop.
__global__ void __launch_bounds__(kTcThreads, 2) k_conv_tc(TcArgs a) {
  extern __shared__ __align__(128) uint8_t tc_smem[];
  __shared__ __align__(8) uint64_t bars[2 * 4 + 4];  // full[4], empty[4], tfull[2], tempty[2]
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = a.N, l = a.l, KB = a.kb;
  const int chunk = blockIdx.x % a.chunks, row = blockIdx.x / a.chunks;
  const int t = row % l, bp = row / l, p = bp & 1, b = bp >> 1;
  const int npad = a.npad[t], PL = a.planes[t];
  const int ntile_all = N / kTcM;
  const int tile0 = chunk * ntile_all / a.chunks, tile1 = (chunk + 1) * ntile_all / a.chunks, nt = tile1 - tile0;
  const int NBF = a.nbufs, KCB = a.kcb, NKC = a.nkc, nu = nt * NKC;
  // shared memory: A[NBF] (kTcM x KCB bytes each: one K chunk of a tile),
  // then B (npad x KB bytes, the whole K, resident for the CTA)
  uint8_t* sA = tc_smem;
  uint8_t* sB = tc_smem + NBF * (size_t)kTcM * KCB;
  const uint32_t sA_u = smem_u32(sA), sB_u = smem_u32(sB);
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = full0 + 32, tfull0 = full0 + 64, tempty0 = full0 + 80;
  const int npairs = KB / 16, cpairs = KCB / 16;  // tap pairs (16 K bytes each), incl. zero padding
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                 "r"(a.tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) {
      mbar_init(full0 + 8 * i, kTcM);
      mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull0 + 8 * i, 1);
      mbar_init(tempty0 + 8 * i, kTcM);
    }
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
  const size_t ct_words = (size_t)2 * l * N;
  if (warp < 4) {
    // ---- producers: position j of every tile
    const int j = tid;
    const u64d* src0 = a.taps + (size_t)b * a.ntaps * ct_words + (size_t)p * l * N + (size_t)t * N + j;
    const uint32_t roff = (uint32_t)(((j >> 3) * 8 + (j & 7)) * 16);
    // unit u = (tile u / NKC, K chunk u % NKC); the buffers cycle over units,
    // so the zero padding (taps >= ntaps, last chunk only) is rewritten each time
    for (int u = 0; u <= nu; ++u) {
      if (u < nu) {
        const int bf = u % NBF, k = u / NKC, kc = u - k * NKC;
        mbar_wait(empty0 + 8 * bf, (uint32_t)(((u / NBF) & 1) ^ 1));  // passes at once on a fresh barrier
        const uint32_t dst0 = sA_u + (uint32_t)(bf * kTcM * KCB) + roff;
        const u64d* src = src0 + (size_t)(tile0 + k) * kTcM;
        const int sp0 = kc * cpairs, sp1 = min(npairs, sp0 + cpairs);
        for (int sp = sp0; sp < sp1; ++sp) {
          const int s = 2 * sp;
          const uint32_t d = dst0 + (uint32_t)(sp - sp0) * 16 * 128;
          if (s < a.ntaps) cp_async8(d, src + (size_t)s * ct_words);
          else asm volatile("st.shared.u64 [%0], %1;\n" ::"r"(d), "l"(0ull) : "memory");
          if (s + 1 < a.ntaps) cp_async8(d + 8, src + (size_t)(s + 1) * ct_words);
          else asm volatile("st.shared.u64 [%0], %1;\n" ::"r"(d + 8), "l"(0ull) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      }
      if (u >= 1) {
        // unit u - 1 landed (this thread's rows): publish it to the MMA issuer
        if (u < nu) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(full0 + 8 * ((u - 1) % NBF)) : "memory");
      }
    }
  } else if (warp == 4) {
    // ---- MMA issuer (one lane): K in steps of 32 bytes = 2 core-matrix chunks
    if (lane == 0) {
      const uint32_t idesc = idesc_u8(kTcM, npad);
      const uint32_t a_lbo = 16 * 128, a_sbo = 128;                       // A: [K chunk][16 position groups][8][16 B]
      const uint32_t b_lbo = (uint32_t)(npad / 8) * 128, b_sbo = 128;     // B: [K chunk][npad / 8 groups][8][16 B]
      for (int u = 0; u < nu; ++u) {
        const int bf = u % NBF, k = u / NKC, kc = u - k * NKC, tb = k & 1;
        mbar_wait(full0 + 8 * bf, (uint32_t)((u / NBF) & 1));
        if (kc == 0) mbar_wait(tempty0 + 8 * tb, (uint32_t)(((k >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t a0 = sA_u + (uint32_t)(bf * kTcM * KCB), d = tmem + (uint32_t)(tb * a.nb);
        const int ks0 = kc * (KCB / 32), ks1 = min(KB, (kc + 1) * KCB) / 32;
        for (int ks = ks0; ks < ks1; ++ks) {
          const uint64_t ad = umma_desc(a0 + (uint32_t)(ks - ks0) * 2 * a_lbo, a_lbo, a_sbo);
          const uint64_t bd = umma_desc(sB_u + (uint32_t)ks * 2 * b_lbo, b_lbo, b_sbo);
          tc_mma_u8(d, ad, bd, idesc, ks > 0);
        }
        tc_commit(empty0 + 8 * bf);                    // the A buffer may be refilled
        if (kc == NKC - 1) tc_commit(tfull0 + 8 * tb);  // the accumulator is ready
      }
    }
    __syncwarp();
  } else {
    // ---- epilogue: position pos of each tile, every map
    const int lane_grp = warp & 3;
    const int pos = 32 * lane_grp + lane;
    const DevPrime pr = a.pt.p[t];
    for (int k = 0; k < nt; ++k) {
      const int tb = k & 1;
      mbar_wait(tfull0 + 8 * tb, (uint32_t)((k >> 1) & 1));
      tc_fence_after();
      const int kpos = (tile0 + k) * kTcM + pos;
      const uint32_t lanebase = tmem + ((uint32_t)(32 * lane_grp) << 16) + (uint32_t)(tb * a.nb);
      for (int co = 0; co < a.c_out; ++co) {
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
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tempty0 + 8 * tb) : "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(a.tcols) : "memory");
  }
}

int planes_of(u64 q) {
  int n = 0;
  while (n < 8 && (q >> (8 * n)) != 0) ++n;
  return n;
}

constexpr size_t kTcSmem = 200 * 1024;

// K bytes per A buffer: the whole row when A[nbufs] + B fit, else the
// fewest equal K chunks (multiples of 32 bytes) that do; 0 if even B plus
// 32-byte chunks does not fit
int pick_kcb(int kb, int maxn, int nbufs) {
  const size_t bsz = (size_t)kb * maxn, per32 = (size_t)nbufs * kTcM * 32;
  if (bsz + per32 > kTcSmem) return 0;
  const int kcmax = std::min(kb, (int)((kTcSmem - bsz) / per32) * 32);
  const int nkc = (kb + kcmax - 1) / kcmax;
  return ((kb + nkc - 1) / nkc + 31) / 32 * 32;
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
  int maxn = 16;
  for (int t = 0; t < l; ++t) maxn = std::max(maxn, (c_out * planes_of(c.P->q(t)) + 15) / 16 * 16);
  return pick_kcb(kb, maxn, kTcBufs) > 0;
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
  a.kcb = pick_kcb(a.kb, maxn, a.nbufs);
  if (a.kcb == 0 || a.kcb < a.kb) {  // the A ring is K-chunked: keep the default buffer count
    a.nbufs = kTcBufs;
    a.kcb = pick_kcb(a.kb, maxn, a.nbufs);
  }
  if (const char* ek = getenv("HEGPU_TC_KCB")) a.kcb = std::min(a.kb, std::max(32, atoi(ek) / 32 * 32));
  const size_t sm = (size_t)a.nbufs * kTcM * a.kcb + (size_t)a.kb * maxn;
  if (a.kcb == 0 || sm > kTcSmem) fail(HEGPU_ERR_ARG, "conv_tc: operands exceed shared memory");
  a.nkc = (a.kb + a.kcb - 1) / a.kcb;
  static PerDeviceOnce prepared;
  if (prepared.first())
    CK(cudaFuncSetAttribute(k_conv_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem));
  const int N = c.N();
  const double bytes = 8.0 * N * l * (2.0 * B * ntaps + 2.0 * B * c_out + c_out);
  const double ops = 2.0 * N * l * B * ntaps * c_out;
  LAUNCH_BO(c, "k_conv_mac", bytes, ops,
            k_conv_tc<<<B * 2 * l * a.chunks, kTcThreads, sm, c.stream>>>(a));
}

}  // namespace hegpu
