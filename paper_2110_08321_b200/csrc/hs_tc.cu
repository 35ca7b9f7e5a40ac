// hs_tc.cu -- the Halevi-Shoup diagonal accumulation (hs_matvec,
// proj/src/matvec.cpp:82-105, hoisted: DESIGN.md §4.3) on the 5th-generation
// tensor cores: tcgen05.mma.kind::i8, accumulator in tensor memory
// (DESIGN.md §4.3d).
//
// The same banded byte-plane GEMM as hs_imma.cu (acc[b][p][t][k] =
// sum_kappa w_kappa(k, p) x_kappa(b), kappa = pos J + j over the window
// position pos = k - r and the J = l + 1 digits), cut for one MMA per K step
// of the whole CTA:
//   M = 128 rows (kl, p, e): 8 consecutive positions x 2 key parts x the 8
//       byte planes e of the Montgomery-form weight W = w R mod q_t;
//   N = 128 columns (img, d): 16 images x the 8 byte planes d of x;
//   K = the union window of the 8 positions (their bands shifted by one
//       position each; rows are zero outside their own band), 32 bytes per
//       MMA.
// C[(kl,p,e)][(img,d)] < 2^32 is exact; the lane of row (kl, p, e) forms
// T_e = sum_d C 2^(8d) (128 bit), u_e = T_e R^-1, v_e = u_e 2^(8e) (one
// Montgomery product with 2^(8e) R), and the 8 lanes of (kl, p) add their
// v_e with three shuffles: sum_e v_e = R^-1 sum_e T_e 2^(8e) = sum w x mod q.
//
// Operands: A (the weights, per 8-position tile and K step one 4 KB block of
// K-major core matrices, built once per plan) arrives by cp.async.bulk into
// a stage ring (mbarrier complete_tx); B (the window bytes, byte-plane
// transposed) is staged from the ModUp digits D and c0 into a shared-memory
// ring of 16-byte K chunks in core-matrix layout, each element once per
// strip of consecutive tiles.  Warp roles: 0-7 stage the window and run the
// epilogue (warp w: TMEM lanes 32 (w % 4), images 8 (w / 4) ..), 8 issues
// the MMAs (one lane), 9 streams A.
// Two accumulator buffers: MMA(tile u) overlaps epilogue(u - 1) and the
// staging of tile u + 1.  Limbs are the same residues as hs_imma.cu / the
// integer kernel / the oracle.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "engine.hpp"

namespace hegpu {

namespace {

constexpr int kTP = 8;           // positions per tile
constexpr int kNI = 16;          // images per CTA
constexpr int kN = kNI * 8;      // MMA N (columns (img, d))
constexpr int kNG = kN / 8;      // column groups of 8 (core matrices along N)
constexpr int kAStages = 3;      // A stages of kKPS K steps
constexpr int kAStep = 4096;     // one K step of A: [2 chunks][16 row groups][8][16 B]
constexpr int kKPS = 2;          // K steps per A stage (one TMA box, one commit)
constexpr int kThreads = 320;    // 10 warps: 0-7 window staging + epilogue, 8 MMA issuer, 9 A producer
constexpr int kRCMax = 48;       // ring chunks (16 K bytes x kN columns = 2 KB each)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
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
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// tensor-map TMA: one 4 KB box (256 bytes x 16 rows) of the A table
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar)
      : "memory");
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
__device__ __forceinline__ void tc_ld8_nowait(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// first / one-past-last 16-byte K chunk of tile kh0's union window, kappa =
// (pos + S) J + j (pos = kh - r for r in [r_lo, r_hi]); the first is even so
// no 32-byte MMA step straddles the ring's wrap
__host__ __device__ inline int tile_c_lo(int kh0, int r_hi, int S, int J) {
  return ((kh0 - r_hi + S) * J / 32) * 2;
}

struct HtArgs {
  PrimeTable pt;
  const u64d* D;       // [B][l][l+1][N] ModUp digits, slot order, canonical
  const u64d* v;       // [B][2][l][N] input ciphertexts (c0 = poly 0)
  const uint8_t* at;   // A tables: [l+1][2 halves][S/8 tiles][nks][4096]
  const u64d* ce;      // [np][8]: 2^(8e) R mod q (Montgomery form of 2^(8e))
  u64d* acc;           // [B][2][l+1][N]
  int B, L, N, l, nks, r_lo, r_hi, rc, strips, nig, accumulate;
  int dbg;  // HEGPU_HT_DBG bits (timing probes only, wrong limbs): 1 no epilogue math, 2 no A copies, 4 no staging
};

template <int J>
__global__ void __launch_bounds__(kThreads, 1) k_hs_tc(HtArgs a, const __grid_constant__ CUtensorMap amap) {
  constexpr int LV = J - 1;
  extern __shared__ __align__(128) uint8_t ht_smem[];
  __shared__ __align__(8) uint64_t bars[2 * kAStages + 8];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N = a.N, S = N >> 1, RC = a.rc, NKS = a.nks;
  const int ig = blockIdx.x % a.nig, strip = blockIdx.x / a.nig;
  const int tph = S / kTP;                      // tiles per half
  const long T = (long)(LV + 1) * 2 * tph;      // (limb, half, tile)
  const long u0 = T * strip / a.strips, u1 = T * (strip + 1) / a.strips;
  const int nt = (int)(u1 - u0);
  uint8_t* ring = ht_smem;                                   // [RC][kNG][8][16]
  uint8_t* astage = ht_smem + (size_t)RC * kNG * 128;        // [kAStages][kKPS * 4096]
  const uint32_t ring_u = smem_u32(ring), ast_u = smem_u32(astage);
  const uint32_t afull0 = smem_u32(&bars[0]), aempty0 = afull0 + 8 * kAStages;
  const uint32_t bfull0 = aempty0 + 8 * kAStages, done0 = bfull0 + 16, tempty0 = bfull0 + 32;
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_slot)),
                 "r"(2 * kN)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < kAStages; ++i) {
      mbar_init(afull0 + 8 * i, 1);
      mbar_init(aempty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bfull0 + 8 * i, 256);
      mbar_init(done0 + 8 * i, 1);
      mbar_init(tempty0 + 8 * i, 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  auto decode = [&](int u, int& t, int& half, int& kh0) {
    const long g = u0 + u;
    t = (int)(g / (2 * tph));
    half = (int)((g / tph) % 2);
    kh0 = (int)(g % tph) * kTP;
  };
  if (warp < 8) {
    // ---- window staging (all 8 warps) + epilogue: warp w reads TMEM lanes
    // 32 (w % 4) (rows m) for images 8 (w / 4) ..
    int cur_seg = -1, c_staged = 0;
    const int m = 32 * (warp & 3) + lane, kl = m >> 4, p = (m >> 3) & 1, e = m & 7;
    const int img0 = 8 * (warp >> 2);
    for (int u = 0; u <= nt; ++u) {
      if (u < nt) {
        int t, half, kh0;
        decode(u, t, half, kh0);
        const int seg = t * 2 + half;
        const int c_lo = tile_c_lo(kh0, a.r_hi, S, J);
        const int c_hi = ((kh0 + kTP - 1 - a.r_lo + S + 1) * J + 15) / 16;
        // ring slots of this tile's new chunks were last read by MMA(u - 2)
        // (by MMA(u - 1) too when a new (limb, half) segment restarts the ring)
        if (u >= 2) mbar_wait(done0 + 8 * (u & 1), (uint32_t)(((u - 2) >> 1) & 1));
        if (seg != cur_seg) {
          if (u >= 1) mbar_wait(done0 + 8 * ((u - 1) & 1), (uint32_t)(((u - 1) >> 1) & 1));
          cur_seg = seg;
          c_staged = c_lo;
        }
        const int cfrom = c_staged > c_lo ? c_staged : c_lo;
        // items: (image, 4 kappa bytes) of chunks [cfrom, c_hi)
        const int ng4 = 4 * (c_hi - cfrom), items = ng4 * kNI;
        const u64d* Dt = a.D + (size_t)t * N + (size_t)half * S;
        const u64d* ct = a.v + (size_t)t * N + (size_t)half * S;
        for (int it = tid; it < ((a.dbg & 4) ? 0 : items); it += 256) {
          const int img = it / ng4, g4 = 4 * cfrom + it % ng4, b = ig * kNI + img;
          const int k0 = 4 * g4;
          u64d w[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const int kap = k0 + x, pos = kap / J - S, j = kap % J;
            const int pm = pos < 0 ? pos + S : pos;
            u64d val = 0;
            if (b < a.B) {
              if (j < LV) val = __ldg(Dt + ((size_t)b * LV + j) * (LV + 1) * N + pm);
              else if (t < LV) val = __ldg(ct + (size_t)b * 2 * LV * N + pm);
            }
            w[x] = val;
          }
          const int slot = (k0 >> 4) % RC, off = k0 & 15;
#pragma unroll
          for (int d = 0; d < 8; ++d) {
            const int sh = 8 * (d & 3);
            uint32_t bw = 0;
#pragma unroll
            for (int x = 0; x < 4; ++x) bw |= (((uint32_t)((d < 4) ? w[x] : (w[x] >> 32)) >> sh) & 0xFFu) << (8 * x);
            const int n = img * 8 + d;
            *reinterpret_cast<uint32_t*>(ring + ((size_t)(slot * kNG + (n >> 3)) * 8 + (n & 7)) * 16 + off) = bw;
          }
        }
        c_staged = c_hi;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive(bfull0 + 8 * (u & 1));
      }
      if (u >= 1) {
        // ---- epilogue of tile u - 1
        const int up = u - 1, tb = up & 1;
        int t, half, kh0;
        decode(up, t, half, kh0);
        mbar_wait(done0 + 8 * tb, (uint32_t)((up >> 1) & 1));
        tc_fence_after();
        const int pi = t == LV ? a.L : t;
        const DevPrime pr = a.pt.p[pi];
        const u64d cst = __ldg(a.ce + (size_t)pi * 8 + e);
        const uint32_t lb = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(tb * kN);
        const int k = half * S + kh0 + kl;
#pragma unroll 1
        for (int i0 = img0; i0 < ((a.dbg & 1) ? img0 : img0 + 8); i0 += 4) {
          uint32_t r[4][8];
#pragma unroll
          for (int q = 0; q < 4; ++q) tc_ld8_nowait(lb + (uint32_t)((i0 + q) * 8), r[q]);
          tc_wait_ld();
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            // T = sum_d C_d 2^(8d): two 57-bit partial sums, then one 128-bit add
            const u64d s0 = (u64d)r[q][0] + ((u64d)r[q][1] << 8) + ((u64d)r[q][2] << 16) + ((u64d)r[q][3] << 24);
            const u64d s1 = (u64d)r[q][4] + ((u64d)r[q][5] << 8) + ((u64d)r[q][6] << 16) + ((u64d)r[q][7] << 24);
            u64d lo = s0, hi = s1 >> 32;
            asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(lo), "+l"(hi) : "l"(s1 << 32));
            u64d vv = mont_mul(mont_reduce128(lo, hi, pr.q, pr.qneg_inv), cst, pr.q, pr.qneg_inv);
            vv = add_mod_d(vv, __shfl_xor_sync(0xffffffffu, vv, 1), pr.q);
            vv = add_mod_d(vv, __shfl_xor_sync(0xffffffffu, vv, 2), pr.q);
            vv = add_mod_d(vv, __shfl_xor_sync(0xffffffffu, vv, 4), pr.q);
            const int b = ig * kNI + i0 + q;
            if (e == 0 && b < a.B) {
              u64d* dst = a.acc + ((size_t)b * 2 + p) * (LV + 1) * N + (size_t)t * N + k;
              *dst = a.accumulate ? add_mod_d(vv, *dst, pr.q) : vv;
            }
          }
        }
        tc_fence_before();
        mbar_arrive(tempty0 + 8 * tb);
      }
    }
  } else if (warp == 8) {
    // ---- MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_u8(128, kN);
      int cnt = 0;
      for (int u = 0; u < nt; ++u) {
        int t, half, kh0;
        decode(u, t, half, kh0);
        const int c_lo = tile_c_lo(kh0, a.r_hi, S, J);
        const int tb = u & 1;
        mbar_wait(bfull0 + 8 * tb, (uint32_t)((u >> 1) & 1));
        mbar_wait(tempty0 + 8 * tb, (uint32_t)(((u >> 1) & 1) ^ 1));
        tc_fence_after();
        const uint32_t d = tmem + (uint32_t)(tb * kN);
        for (int ks0 = 0; ks0 < NKS; ks0 += kKPS, ++cnt) {
          const int st = cnt % kAStages;
          mbar_wait(afull0 + 8 * st, (uint32_t)((cnt / kAStages) & 1));
          tc_fence_after();
#pragma unroll
          for (int h = 0; h < kKPS; ++h) {
            const int ks = ks0 + h;
            const uint64_t ad = umma_desc(ast_u + (uint32_t)((st * kKPS + h) * kAStep), 16 * 128, 128);
            const int slot = (c_lo + 2 * ks) % RC;
            const uint64_t bd = umma_desc(ring_u + (uint32_t)(slot * kNG * 128), kNG * 128, 128);
            tc_mma_u8(d, ad, bd, idesc, ks > 0);
          }
          tc_commit(aempty0 + 8 * st);
        }
        tc_commit(done0 + 8 * tb);
      }
    }
    __syncwarp();
  } else {
    // ---- A producer
    if (lane == 0) {
      int cnt = 0;
      for (int u = 0; u < nt; ++u) {
        int t, half, kh0;
        decode(u, t, half, kh0);
        const uint8_t* src = a.at + ((((size_t)t * 2 + half) * tph + kh0 / kTP) * NKS) * kAStep;
        for (int ks = 0; ks < NKS; ks += kKPS, ++cnt) {
          const int st = cnt % kAStages;
          mbar_wait(aempty0 + 8 * st, (uint32_t)(((cnt / kAStages) & 1) ^ 1));
          if (a.dbg & 2) {
            mbar_arrive(afull0 + 8 * st);
          } else {
            mbar_expect_tx(afull0 + 8 * st, kKPS * kAStep);
            // the A table as a 2D tensor [rows of 256 bytes]: this stage's kKPS x 16 rows
            const long row = (long)((src - a.at) + (size_t)ks * kAStep) / 256;
            tma_load_2d(ast_u + (uint32_t)(st * kKPS * kAStep), &amap, 0, (int)row, afull0 + 8 * st);
          }
        }
      }
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(2 * kN) : "memory");
  }
}

// A tables: one thread per 16-byte core-matrix row of (limb t, half, tile,
// K step ks, chunk c2, row group mg, row): bytes e of the Montgomery-form
// weight of row (kl, p, e) at kappa = 16 (c_lo + 2 ks + c2) + i
template <int J>
__global__ void k_hs_tc_tiles(PrimeTable pt, const u64d* __restrict__ fk, size_t fk_words, int first_keyed,
                              const u64d* __restrict__ masks, const int* __restrict__ rdiag,
                              const u64d* __restrict__ pR, int L, int N, int nks, int r_lo, int r_hi,
                              uint4* __restrict__ at) {
  constexpr int LV = J - 1;
  const int S = N >> 1, tph = S / kTP;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t total = (size_t)(LV + 1) * 2 * tph * nks * 256;
  if (gid >= total) return;
  const int rowi = (int)(gid & 255);  // (c2, mg, row) = 2 x 16 x 8
  size_t q = gid >> 8;
  const int ks = (int)(q % nks);
  q /= nks;
  const int tile = (int)(q % tph);
  q /= tph;
  const int half = (int)(q % 2), t = (int)(q / 2);
  const int c2 = rowi >> 7, m = rowi & 127;  // M row (kl, p, e)
  const int kl = m >> 4, p = (m >> 3) & 1, e = m & 7;
  const int kh0 = tile * kTP, kh = kh0 + kl, k = half * S + kh;
  const int pi = t == LV ? L : t;
  const DevPrime pr = pt.p[pi];
  const int kap0 = 16 * (tile_c_lo(kh0, r_hi, S, J) + 2 * ks + c2);
  uint32_t wd[4] = {0, 0, 0, 0};
  for (int i = 0; i < 16; ++i) {
    const int kap = kap0 + i, pos = kap / J - S, j = kap % J, r = kh - pos;
    if (r < r_lo || r > r_hi) continue;
    const int di = rdiag[r];
    if (di < 0) continue;
    u64d w = 0;
    if (j < LV) {
      if (r != 0) w = unsplit31(fk[(size_t)(di - first_keyed) * fk_words + ((size_t)(j * 2 + p) * (LV + 1) + t) * N + k]);
    } else if (p == 0 && t < LV) {
      w = mont_mul(unsplit31(masks[((size_t)di * (LV + 1) + t) * N + k]), pR[t], pr.q, pr.qneg_inv);
    }
    wd[i >> 2] |= (uint32_t)((w >> (8 * e)) & 0xFF) << (8 * (i & 3));
  }
  at[gid] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

}  // namespace

bool hs_tc_enabled() {
  const char* e = getenv("HEGPU_HS_TC");
  return !(e && e[0] == '0');
}

int hs_tc_chunk_span(int l) {
  // ring: window chunks ceil(((span + 8) J + 32) / 16) + 2, plus one tile's
  // advance ceil(8 J / 16) + 1, plus 2, within kRCMax
  const int J = l + 1;
  const int room = kRCMax - 2 - ((kTP * J + 15) / 16 + 1) - 2;
  return std::max(1, (room * 16 - 32) / J - kTP);
}

int hs_tc_nks(int l, int span) {
  const int n = ((span + kTP) * (l + 1) + 32 + 31) / 32 + 1;
  return (n + kKPS - 1) / kKPS * kKPS;  // whole A stages
}

size_t hs_tc_table_bytes(Context& c, int l, int span) {
  return (size_t)(l + 1) * c.N() / kTP * hs_tc_nks(l, span) * kAStep;
}

void launch_hs_tc_tiles(Context& c, int l, const HsDiagTable& t, const u64d* pR, const int* rdiag, int r_lo,
                        int r_hi, uint8_t* at) {
  const int nks = hs_tc_nks(l, r_hi - r_lo + 1);
  const size_t threads = (size_t)(l + 1) * 2 * (c.S() / kTP) * nks * 256;
  const unsigned grid = (unsigned)((threads + 255) / 256);
  uint4* a4 = reinterpret_cast<uint4*>(at);
#define HT_TILES(JJ)                                                                                           \
  case JJ:                                                                                                     \
    LAUNCH(c, "k_hs_tc_tiles",                                                                                 \
           k_hs_tc_tiles<JJ><<<grid, 256, 0, c.stream>>>(c.primes, t.fk, t.fk_words, t.first_keyed, t.masks, rdiag, \
                                                         pR, c.L(), c.N(), nks, r_lo, r_hi, a4));              \
    break;
  switch (l + 1) {
    HT_TILES(2) HT_TILES(3) HT_TILES(4) HT_TILES(5) HT_TILES(6) HT_TILES(7) HT_TILES(8) HT_TILES(9)
    default: fail(HEGPU_ERR_ARG, "hs_tc: level out of range");
  }
#undef HT_TILES
}

// the A table of one chunk as a 2D uint8 tensor map: rows of 256 bytes,
// boxes of 16 rows (one 4 KB K step); the driver entry point is fetched
// through the runtime, so the library does not link libcuda directly
static void make_amap(CUtensorMap* map, const uint8_t* at, size_t bytes) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !encode) fail(HEGPU_ERR_CUDA, "hs_tc: cuTensorMapEncodeTiled unavailable");
  }
  const cuuint64_t dims[2] = {256, (cuuint64_t)(bytes / 256)};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {256, 16 * kKPS}, estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(at), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(HEGPU_ERR_CUDA, "hs_tc: cuTensorMapEncodeTiled failed");
}

void launch_hs_tc(Context& c, const u64d* v, int B, int l, const u64d* D, int r_lo, int r_hi, const uint8_t* at,
                  const u64d* ce, int accumulate, u64d* acc, int keyed, int ndiag) {
  const int N = c.N(), J = l + 1, span = r_hi - r_lo + 1;
  HtArgs a{};
  a.pt = c.primes;
  a.D = D;
  a.v = v;
  a.at = at;
  a.ce = ce;
  a.acc = acc;
  a.B = B;
  a.L = c.L();
  a.N = N;
  a.l = l;
  a.nks = hs_tc_nks(l, span);
  a.r_lo = r_lo;
  a.r_hi = r_hi;
  a.accumulate = accumulate;
  a.nig = (B + kNI - 1) / kNI;
  const char* dbg = getenv("HEGPU_HT_DBG");
  a.dbg = dbg ? atoi(dbg) : 0;
  int rc = ((span + kTP) * J + 32 + 15) / 16 + 2 + (kTP * J + 15) / 16 + 1 + 2;
  rc = (rc + 1) / 2 * 2;
  if (rc > kRCMax) fail(HEGPU_ERR_ARG, "hs_tc: chunk span exceeds the window ring");
  a.rc = rc;
  const long T = (long)J * 2 * (c.S() / kTP);
  long strips = (long)device_sms() * 2 / a.nig;
  if (strips < 1) strips = 1;
  if (strips > T) strips = T;
  a.strips = (int)strips;
  const size_t smem = (size_t)rc * kNG * 128 + (size_t)kAStages * kKPS * kAStep;
  alignas(64) CUtensorMap amap;
  make_amap(&amap, at, hs_tc_table_bytes(c, l, span));
  const double NB = 8.0 * N;
  const double bytes = (double)hs_tc_table_bytes(c, l, span) + NB * B * (l * J + l) + NB * B * 2 * J * (accumulate ? 2 : 1);
  const double ops = (double)N * B * (keyed * l * J * 2.0 + ndiag * l);
#define HT_GO(JJ)                                                                                    \
  case JJ: {                                                                                         \
    static PerDeviceOnce prepared;                                                                   \
    if (prepared.first())                                                                            \
      CK(cudaFuncSetAttribute(k_hs_tc<JJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); \
    LAUNCH_BO(c, "k_hs_imma", bytes, ops,                                                           \
              (k_hs_tc<JJ><<<(unsigned)(a.nig * strips), kThreads, smem, c.stream>>>(a, amap)));      \
    break;                                                                                           \
  }
  switch (J) {
    HT_GO(2) HT_GO(3) HT_GO(4) HT_GO(5) HT_GO(6) HT_GO(7) HT_GO(8) HT_GO(9)
    default: fail(HEGPU_ERR_ARG, "hs_tc: level out of range");
  }
#undef HT_GO
}

}  // namespace hegpu
