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
// cp.async staging of tiles i + 1, i + 2.  When B plus three whole-K A
// tiles exceed shared memory (config 3's 75-tap first layer: B alone is
// 117 KB) the A ring holds K chunks instead: a pipeline unit is (tile, K
// chunk), the chunks of one tile accumulate into the same TMEM buffer, and
// four buffers with two units in flight per producer keep the loads deep.
// The epilogue (8 warps, 4 maps per tcgen05.wait::ld) combines the byte
// planes with 32x32->64 multiply-adds and prefetches the next group's bias
// words.  Limbs are the same residues as the IMAD / mma.sync paths.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "engine.hpp"

namespace hegpu {

namespace {

constexpr int kTcM = 128;       // positions per tile (MMA M)
constexpr int kEpiWarps = 8;     // two epilogue warps per TMEM lane quarter (maps split between them)
constexpr int kTcThreads = 32 * (5 + kEpiWarps);  // 4 producers, 1 MMA issuer, the epilogue
constexpr int kTcTiles = 16;     // position tiles per CTA (HEGPU_TC_TILES)
constexpr int kTcBufs = 3;       // A (tap) tile buffers in flight (HEGPU_TC_BUFS, 2..kMaxBufs)
constexpr int kMaxBufs = 8;

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

// cp.async.wait_group takes an immediate: at most n (0..7) groups left pending
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
    case 5: asm volatile("cp.async.wait_group 5;\n" ::: "memory"); break;
    case 6: asm volatile("cp.async.wait_group 6;\n" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 7;\n" ::: "memory"); break;
  }
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
// 8 consecutive accumulator columns of this thread's TMEM lane (completed by tcgen05.wait::ld)
__device__ __forceinline__ void tc_ld8_nowait(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr));
}
// ties registers loaded by tc_ld8_nowait to a preceding tcgen05.wait::ld
// (the compiler may not hoist their uses above this volatile asm)
__device__ __forceinline__ void tc_after_wait(uint32_t (&r)[8]) {
  asm volatile("" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]));
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
  int lag;            // units a producer keeps in flight before publishing the oldest (1..nbufs - 1)
};

// Warp roles (13 warps): 0-3 producers (thread j stages position j of a
// tile: its tap words by cp.async into the core-matrix rows), 4 the MMA
// issuer (one lane), 5-12 the epilogue (warp w reads TMEM lanes 32 (w % 4);
// warps 5-8 take maps 0-3, 8-11, ..., warps 9-12 maps 4-7, 12-15, ...: four
// maps' columns loaded per tcgen05.wait::ld).
// mbarriers: full[buf] (128 producer arrivals, after each producer's
// cp.async.wait + proxy fence), empty[buf] and tfull[tb] (tcgen05.commit),
// tempty[tb] (128 epilogue arrivals) -- no CTA-wide barrier in the loop.
#ifndef HEGPU_TC_MINB
#define HEGPU_TC_MINB 1  // CTAs per SM the register allocation allows (2: <= 78 registers)
#endif
__global__ void __launch_bounds__(kTcThreads, HEGPU_TC_MINB) k_conv_tc(TcArgs a) {
  extern __shared__ __align__(128) uint8_t tc_smem[];
  __shared__ __align__(8) uint64_t bars[2 * kMaxBufs + 4];  // full[], empty[], tfull[2], tempty[2]
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
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = full0 + 8 * kMaxBufs, tfull0 = full0 + 16 * kMaxBufs,
                 tempty0 = tfull0 + 16;
  const int npairs = KB / 16, cpairs = KCB / 16;  // tap pairs (16 K bytes each), incl. zero padding
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                 "r"(a.tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < kMaxBufs; ++i) {
      mbar_init(full0 + 8 * i, kTcM);
      mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(tfull0 + 8 * i, 1);
      mbar_init(tempty0 + 8 * i, 32 * kEpiWarps);
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
    const int lag = a.lag;
    for (int u = 0; u < nu + lag; ++u) {
      if (u < nu) {
        const int bf = u % NBF, k = u / NKC, kc = u - k * NKC;
        mbar_wait(empty0 + 8 * bf, (uint32_t)(((u / NBF) & 1) ^ 1));  // passes at once on a fresh barrier
        const uint32_t dst0 = sA_u + (uint32_t)(bf * kTcM * KCB) + roff;
        const u64d* src = src0 + (size_t)(tile0 + k) * kTcM;
        const int sp0 = kc * cpairs, sp1 = min(npairs, sp0 + cpairs), spf = min(sp1, a.ntaps >> 1);
        // whole tap pairs: a running source pointer, no predicates
        uint32_t d = dst0;
        const u64d* sp_src = src + (size_t)(2 * sp0) * ct_words;
        for (int sp = sp0; sp < spf; ++sp, d += 16 * 128, sp_src += 2 * ct_words) {
          cp_async8(d, sp_src);
          cp_async8(d + 8, sp_src + ct_words);
        }
        // the last odd tap and the zero padding up to the 32-byte K step
        for (int sp = max(sp0, spf); sp < sp1; ++sp, d += 16 * 128) {
          const int s = 2 * sp;
          if (s < a.ntaps) cp_async8(d, src + (size_t)s * ct_words);
          else asm volatile("st.shared.u64 [%0], %1;\n" ::"r"(d), "l"(0ull) : "memory");
          asm volatile("st.shared.u64 [%0], %1;\n" ::"r"(d + 8), "l"(0ull) : "memory");
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      }
      if (u >= lag) {
        // unit u - lag landed (this thread's rows): publish it to the MMA issuer
        cp_async_wait_dyn(min(lag, nu - 1 - (u - lag)));
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(full0 + 8 * ((u - lag) % NBF)) : "memory");
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
    // ---- epilogue: position pos of each tile, every map.  The bias words
    // (poly 0) of the next map group are loaded while the current group's
    // accumulator columns come out of TMEM, so their L2 latency is hidden.
    const int lane_grp = warp & 3, half = (warp - 5) >> 2;
    const int pos = 32 * lane_grp + lane;
    const DevPrime pr = a.pt.p[t];
    const u64d* bias_t = (p == 0 && a.bias) ? a.bias + (size_t)t * N + pos : nullptr;
    const size_t bstride = (size_t)l * N;
    u64d* obase = a.out + (size_t)b * a.c_out * ct_words + (size_t)p * l * N + (size_t)t * N + (size_t)tile0 * kTcM + pos;
    auto load_bias = [&](u64d(&o)[4], int k, int c0) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
        o[g] = (bias_t && k < nt && c0 + g < a.c_out)
                   ? __ldg(bias_t + (size_t)(c0 + g) * bstride + (size_t)(tile0 + k) * kTcM)
                   : 0ull;
    };
    u64d bcur[4], bnxt[4];
    load_bias(bcur, 0, 4 * half);
    for (int k = 0; k < nt; ++k) {
      const int tb = k & 1;
      mbar_wait(tfull0 + 8 * tb, (uint32_t)((k >> 1) & 1));
      tc_fence_after();
      const uint32_t lanebase = tmem + ((uint32_t)(32 * lane_grp) << 16) + (uint32_t)(tb * a.nb);
      for (int c0 = 4 * half; c0 < a.c_out; c0 += 8) {
        const int ng = min(4, a.c_out - c0);
        uint32_t r[4][8];
#pragma unroll
        for (int g = 0; g < 4; ++g)
          if (g < ng) tc_ld8_nowait(lanebase + (uint32_t)((c0 + g) * PL), r[g]);
        if (c0 + 8 < a.c_out) load_bias(bnxt, k, c0 + 8);
        else load_bias(bnxt, k + 1, 4 * half);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          if (g >= ng) break;
          tc_after_wait(r[g]);
          const int co = c0 + g;
          // T = bias R + sum_e C_e 2^(8e): columns >= PL belong to the next map;
          // x = planes 0-3 and y = planes 4-7 stay below 2^51, T = x + y 2^32
          uint32_t cv[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) cv[e] = e < PL ? r[g][e] : 0u;
          u64d x = bcur[g] + (u64d)cv[0];
          x += (u64d)cv[1] << 8;
          x += (u64d)cv[2] << 16;
          x += (u64d)cv[3] << 24;
          u64d y = (u64d)cv[4];
          y += (u64d)cv[5] << 8;
          y += (u64d)cv[6] << 16;
          y += (u64d)cv[7] << 24;
          const u64d lo = x + (y << 32), hi = (y >> 32) + (lo < x);
          obase[(size_t)co * ct_words + (size_t)k * kTcM] = mont_reduce128(lo, hi, pr.q, pr.qneg_inv);
        }
#pragma unroll
        for (int g = 0; g < 4; ++g) bcur[g] = bnxt[g];
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
  a.nbufs = eb ? std::min(kMaxBufs, std::max(2, atoi(eb))) : kTcBufs;
  a.chunks = std::max(1, ntile / tiles);
  a.kcb = pick_kcb(a.kb, maxn, a.nbufs);
  bool chunked = a.kcb < a.kb;
  if (!eb && chunked) {  // K-chunked A ring: shorter units, one more buffer, two units in flight
    a.nbufs = kTcBufs + 1;
    a.kcb = pick_kcb(a.kb, maxn, a.nbufs);
    if (a.kcb == 0) {
      a.nbufs = kTcBufs;
      a.kcb = pick_kcb(a.kb, maxn, a.nbufs);
    }
  }
  if (const char* ek = getenv("HEGPU_TC_KCB")) a.kcb = std::min(a.kb, std::max(32, atoi(ek) / 32 * 32));
  chunked = a.kcb < a.kb;
  const char* el = getenv("HEGPU_TC_LAG");
  a.lag = std::min(a.nbufs - 1, std::max(1, el ? atoi(el) : chunked ? 2 : 1));
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
