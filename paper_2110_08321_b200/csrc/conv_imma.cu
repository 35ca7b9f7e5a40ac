// conv_imma.cu -- the conv-pack multiply-accumulate on the int8 tensor cores.
//
// out[co][k] = sum_s W[co][s] * tap_s[k] mod q (per image, poly, limb) is a
// GEMM: the weights are shared by every slot position.  It runs exactly on
// IMMA.16832 (mma.sync m16n8k32 u8 x u8 -> s32, measured 1.1 POPS on this
// B200, tools/ubench_mma.cu) through a byte decomposition:
//   tap x = sum_i x_i 2^(8i)             (x_i = byte i, i < 8: the B operand
//                                         is just the two 32-bit halves of x)
//   w_{co,s,i} = W[co][s] 2^(8i) R mod q (precomputed per limb; R = 2^64
//                                         Montgomery form, so the single
//                                         reduction below lands in standard form)
//   w_{co,s,i} = sum_e w_e 2^(8e)        (e < 8: the A operand)
//   T_e[co][k] = sum_{s,i} w_e[co,s,i] x_i[s][k]        <- the GEMM, K = 8 ntaps
//   out = (sum_e T_e 2^(8e) + bias R) R^-1 mod q   (T_e < 2^29: < 2^86
//                                         total, one Montgomery reduction)
// so the result is the same residue as the IMAD path, bit for bit.
// Tile: a warp owns 4 x 8 slot positions (n8 tiles) and 4 output-map pairs
// (m16 = 2 maps x 8 byte planes e) with k32 = 4 taps x 8 bytes per step.
#include <cstdint>

#include "engine.hpp"

namespace hegpu {

namespace {

constexpr int kImmaWarps = 8;                   // warps per CTA
constexpr int kImmaNT = 4;                      // n8 position tiles per warp (A fragment reuse)
constexpr int kImmaCPG = 4;                     // map pairs per warp pass (B fragment reuse)
constexpr int kImmaPos = 8 * kImmaNT * kImmaWarps;  // slot positions per CTA
#ifndef HEGPU_IMMA_DEPTH
#define HEGPU_IMMA_DEPTH 8  // measured: 3: -, 4: 3.77, 6: 3.49, 8: 3.22, 10: 3.49, 12+: 4.8 ms (cfg3 conv)
#endif
constexpr int kImmaDepth = HEGPU_IMMA_DEPTH;    // cp.async pipeline stages (k32 steps)
constexpr int kBRow = 2 * kImmaPos + 16;        // u32 words per staged tap row (+16: bank offset)

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ void mma_u8(int (&c)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// a warp: kImmaNT tiles of 8 positions x kImmaCPG map groups; per k32 step
// the B fragments of the NT tiles are loaded once and reused by CPG map
// groups, each A fragment by NT tiles.  MPT = maps per MMA row tile: 2 (rows
// = map x 8 byte planes e) or, for limbs of primes < 2^40 whose weight
// digits have 5 bytes, 3 (rows = map x 5 planes, row 15 unused).
struct ConvLimbs {
  int n;
  unsigned long long t;  // the limbs, 4 bits each (a register, not a local array)
  int stride;            // map groups per limb in the fragment table (the pair count)
};
template <int MPT>
__global__ void __launch_bounds__(32 * kImmaWarps) k_conv_imma(PrimeTable pt, const u64d* __restrict__ taps,
                                                              int ntaps, int l, int N,
                                                              const uint4* __restrict__ wa, int cps, int kbn,
                                                              int c_out, const u64d* __restrict__ bias,
                                                              u64d* __restrict__ out, ConvLimbs lim) {
  constexpr int EP = MPT == 2 ? 8 : 5;  // byte planes per map row block
  extern __shared__ __align__(16) uint4 dyn_smem[];
  // [kImmaDepth][kImmaCPG][32] A fragments, then [kImmaDepth][4 taps][kBRow]
  // tap words of the CTA's positions (rows padded: conflict-free reads)
  auto a_s = reinterpret_cast<uint4 (*)[kImmaCPG][32]>(dyn_smem);
  auto b_s = reinterpret_cast<uint32_t (*)[4][kBRow]>(dyn_smem + kImmaDepth * kImmaCPG * 32);
  // epilogue transpose scratch reuses the pipeline buffers
  auto scratch = reinterpret_cast<int (*)[2][16][9]>(dyn_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = (int)((lim.t >> (4 * (blockIdx.y % lim.n))) & 15), poly = blockIdx.y / lim.n;
  // the map-pair group varies fastest, so the CTAs reading the same taps
  // run together and the taps come from L2 after the first group
  const int groups = (cps + kImmaCPG - 1) / kImmaCPG;
  const int b = blockIdx.z, cp0 = (blockIdx.x % groups) * kImmaCPG;
  const int kc = (blockIdx.x / groups) * kImmaPos;      // first position of the CTA
  const int kw = kc + warp * 8 * kImmaNT;               // ... of the warp
  const size_t ct_words = (size_t)2 * l * N;
  const u64d* tap0 = taps + (size_t)b * ntaps * ct_words + (size_t)poly * l * N + (size_t)t * N + kc;
  // B operand: the half (lane & 1) of tap word x[4 kb + sub (+2)][kw + 8 nt + lane/4]
  const int sub = (lane & 3) >> 1;
  const int boff = sub * kBRow + 2 * (warp * 8 * kImmaNT + (lane >> 2)) + (lane & 1);
  int c[kImmaCPG][kImmaNT][4];
#pragma unroll
  for (int j = 0; j < kImmaCPG; ++j)
#pragma unroll
    for (int n = 0; n < kImmaNT; ++n) c[j][n][0] = c[j][n][1] = c[j][n][2] = c[j][n][3] = 0;
  const uint4* wt = wa + (size_t)t * lim.stride * kbn * 32;
  // kImmaDepth-stage cp.async pipeline: A fragments of the CTA's map pairs
  // (shared by its warps) and each lane's own B words
  auto issue = [&](int kb) {
    const int st = kb % kImmaDepth;
    if (threadIdx.x < kImmaCPG * 32) {
      const int j = threadIdx.x >> 5;
      if (cp0 + j < cps) cp_async16(&a_s[st][j][lane], wt + ((size_t)(cp0 + j) * kbn + kb) * 32 + lane);
    }
    // 4 taps x kImmaPos words in 16-byte copies, 2 per thread
#pragma unroll
    for (int r = 0; r < 4 * kImmaPos / 2 / (32 * kImmaWarps); ++r) {
      const int idx = threadIdx.x + r * 32 * kImmaWarps, q = idx / (kImmaPos / 2), ch = idx % (kImmaPos / 2);
      uint32_t* dst = &b_s[st][q][4 * ch];
      if (4 * kb + q < ntaps) cp_async16(dst, tap0 + (size_t)(4 * kb + q) * ct_words + 2 * ch);
      else *reinterpret_cast<uint4*>(dst) = make_uint4(0, 0, 0, 0);
    }
  };
#pragma unroll
  for (int d = 0; d < kImmaDepth - 1; ++d) {
    if (d < kbn) issue(d);
    cp_async_commit();
  }
  for (int kb = 0; kb < kbn; ++kb) {
    if (kb + kImmaDepth - 1 < kbn) issue(kb + kImmaDepth - 1);
    cp_async_commit();
    cp_async_wait<kImmaDepth - 1>();
    __syncthreads();  // every thread's copies of stage kb are visible
    const int st = kb % kImmaDepth;
    uint32_t b0[kImmaNT], b1[kImmaNT];
    const uint32_t* bs = &b_s[st][0][0] + boff;
#pragma unroll
    for (int n = 0; n < kImmaNT; ++n) {
      b0[n] = bs[16 * n];
      b1[n] = bs[2 * kBRow + 16 * n];
    }
#pragma unroll
    for (int j = 0; j < kImmaCPG; ++j) {
      if (cp0 + j < cps) {
        const uint4 a = a_s[st][j][lane];
#pragma unroll
        for (int n = 0; n < kImmaNT; ++n) mma_u8(c[j][n], a, b0[n], b1[n]);
      }
    }
    __syncthreads();  // stage kb may be refilled
  }
  const DevPrime pr = pt.p[t];
  const int row = lane >> 2, col = 2 * (lane & 3);
  if constexpr (MPT == 2) {
    // epilogue: fragments go through shared memory two at a time; each lane
    // combines the 8 byte planes of one (map, position) of one fragment
    const int half = (lane >> 3) & 1, pc = lane & 7, fsel = lane >> 4;
#pragma unroll
    for (int f0 = 0; f0 < kImmaCPG * kImmaNT; f0 += 2) {
      const int j = f0 / kImmaNT;  // fragments f0, f0 + 1 share j (NT even)
      if (cp0 + j >= cps) break;
      __syncwarp();
#pragma unroll
      for (int f = 0; f < 2; ++f) {
        const int n = (f0 + f) % kImmaNT;
        scratch[warp][f][row][col] = c[j][n][0];
        scratch[warp][f][row][col + 1] = c[j][n][1];
        scratch[warp][f][row + 8][col] = c[j][n][2];
        scratch[warp][f][row + 8][col + 1] = c[j][n][3];
      }
      __syncwarp();
      const int co = 2 * (cp0 + j) + half;
      if (co < c_out) {
        const int k = kw + 8 * ((f0 + fsel) % kImmaNT) + pc;
        // + bias R (the stored Montgomery bias) before the reduction
        u64d lo = (poly == 0 && bias) ? bias[((size_t)co * l + t) * N + k] : 0ull, hi = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const u64d v = (u64d)(uint32_t)scratch[warp][fsel][half * 8 + e][pc];
          const u64d l_add = v << (8 * e), h_add = e ? v >> (64 - 8 * e) : 0ull;
          asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(l_add), "l"(h_add));
        }
        // (hi:lo) < 2^87 < q 2^64: one Montgomery reduction -> standard form
        out[((size_t)b * c_out + co) * ct_words + (size_t)poly * l * N + (size_t)t * N + k] =
            mont_reduce128(lo, hi, pr.q, pr.qneg_inv);
      }
    }
  } else {
    // epilogue (3 maps x 5 planes): one fragment per round; lanes < 24
    // combine planes e < 5 of (map lane / 8, position lane % 8)
    const int m = lane >> 3, pc = lane & 7;
#pragma unroll
    for (int f = 0; f < kImmaCPG * kImmaNT; ++f) {
      const int j = f / kImmaNT, n = f % kImmaNT;
      if (cp0 + j >= cps) break;
      __syncwarp();
      scratch[warp][0][row][col] = c[j][n][0];
      scratch[warp][0][row][col + 1] = c[j][n][1];
      scratch[warp][0][row + 8][col] = c[j][n][2];
      scratch[warp][0][row + 8][col + 1] = c[j][n][3];
      __syncwarp();
      const int co = 3 * (cp0 + j) + m;
      if (m < 3 && co < c_out) {
        const int k = kw + 8 * n + pc;
        u64d lo = (poly == 0 && bias) ? bias[((size_t)co * l + t) * N + k] : 0ull, hi = 0;
#pragma unroll
        for (int e = 0; e < EP; ++e) {
          const u64d v = (u64d)(uint32_t)scratch[warp][0][m * 5 + e][pc];
          const u64d l_add = v << (8 * e), h_add = e ? v >> (64 - 8 * e) : 0ull;
          asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(l_add), "l"(h_add));
        }
        out[((size_t)b * c_out + co) * ct_words + (size_t)poly * l * N + (size_t)t * N + k] =
            mont_reduce128(lo, hi, pr.q, pr.qneg_inv);
      }
    }
  }
}

}  // namespace

bool conv_imma_supported(Context& c) { return c.N() % kImmaPos == 0; }

template <int MPT>
void conv_imma_go(Context& c, dim3 grid, size_t sm, double bytes, double ops, const u64d* taps, int ntaps, int l,
                  const uint4* w4, int groups_n, int kbn, int c_out, const u64d* bias, u64d* out, const ConvLimbs& lim) {
  static PerDeviceOnce prepared;
  if (sm > 48 * 1024 && prepared.first())
    CK(cudaFuncSetAttribute(k_conv_imma<MPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  LAUNCH_BO(c, "k_conv_mac", bytes, ops,
            k_conv_imma<MPT><<<grid, 32 * kImmaWarps, sm, c.stream>>>(c.primes, taps, ntaps, l, c.N(), w4, groups_n,
                                                                     kbn, c_out, bias, out, lim));
}

void launch_conv_imma(Context& c, const u64d* taps, int B, int ntaps, int l, const uint32_t* wa, int cps, int kbn,
                      int c_out, const u64d* bias, u64d* out) {
  const int N = c.N();
  const uint4* w4 = reinterpret_cast<const uint4*>(wa);
  const size_t sm = (size_t)kImmaDepth * (kImmaCPG * 32 * 16 + 4 * kBRow * 4);
  // limbs by weight-digit width: primes < 2^40 pack 3 maps per row tile
  ConvLimbs lim[2]{};
  for (int t = 0; t < l; ++t) {
    ConvLimbs& L = lim[conv_imma_triples(c, t, c_out) ? 1 : 0];
    L.t |= (unsigned long long)t << (4 * L.n++);
    L.stride = cps;
  }
  for (int k = 0; k < 2; ++k) {
    if (!lim[k].n) continue;
    const int groups_n = k ? (c_out + 2) / 3 : cps;
    const int groups = (groups_n + kImmaCPG - 1) / kImmaCPG;
    dim3 grid(N / kImmaPos * groups, 2 * lim[k].n, B);
    const double fr = (double)lim[k].n / l;
    const double bytes = fr * 8.0 * N * l * (2.0 * B * ntaps + 2.0 * B * c_out + c_out);
    const double ops = fr * 2.0 * N * l * B * ntaps * c_out;  // modular MAC terms (as the IMAD path)
    if (k) conv_imma_go<3>(c, grid, sm, bytes, ops, taps, ntaps, l, w4, groups_n, kbn, c_out, bias, out, lim[k]);
    else conv_imma_go<2>(c, grid, sm, bytes, ops, taps, ntaps, l, w4, groups_n, kbn, c_out, bias, out, lim[k]);
  }
}

// (few maps -- cfg 0's 5 -- leave the MAC bound by the tap stream, where the
// extra epilogue rounds of the triple layout cost more than the MMAs saved:
// measured 0.552 vs 0.568 ms at 5 maps, 3 % faster cfg 3 at 32 maps)
bool conv_imma_triples(Context& c, int t, int c_out) { return c_out > 6 && c.P->q(t) < (1ull << 40); }

}  // namespace hegpu
