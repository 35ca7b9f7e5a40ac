// hs_imma.cu -- the Halevi-Shoup diagonal accumulation on the int8 tensor
// cores.
//
// Per output position k (slot order, inside one half), ext limb t, image b
// and key part p the hoisted HS layer accumulates
//   acc[b][p][t][k] = sum_{r kept} ( sum_{j<l} D_j[b][t][k - r] fk_{r,j,p}[t][k]
//                                    + [p == 0] c0[b][t][k - r] P m_r[t][k] )
// (the c0 * mask term is folded into the extended-basis accumulator as
// P * c0 * m: the ModDown divides it back out exactly, so the result is the
// same residue as ModDown(acc) + c0 * m).  Indexing the sum by the window
// position pos = k - r instead of r turns it into a BANDED GEMM over
// kappa = pos * J + j (J = l + 1 "digits": the l ModUp digits and c0):
//   A[(k, p, e)][kappa] = byte e of the weight (fk or P m) -- per position,
//                         precomputed once per plan in mma fragment order
//   B[kappa][(b, d)]    = byte d of the window element x_kappa of image b
//   C[(k,p,e)][(b,d)]   = sum_kappa A B   (exact: < 2^32 for kappa < 66k)
//   value(k, b, p)      = sum_{e,d} C 2^(8(e+d)) = sum_kappa w x  (exact)
// on mma.sync m16n8k32 u8 (rows = (p, e) of one position, columns = the 8
// byte planes of one image).  Consecutive positions share the B fragments
// (the window slides by J bytes per position), so a warp owns 4 positions x
// 4 images and a CTA streams a strip of 16-position blocks through a ring
// buffer of window bytes (each element staged once per strip).
#include <cstdint>
#include <vector>

#include "engine.hpp"

namespace hegpu {

namespace {

constexpr int kHiWarps = 16;              // 4 position groups x 4 image groups
constexpr int kHiKB = 16;                 // output positions per block
constexpr int kHiBc = 16;                 // images per CTA
constexpr int kHiRSMax = 24;              // max ring size in 32-byte k-steps (runtime RS <= this)
constexpr int kHiMaxDepth = 8;            // A-fragment pipeline stages (runtime D <= this)
constexpr int kHiStage = 4 * 4 * 32;      // uint4 per stage: 4 position groups x 4 positions x 32 lanes
constexpr int kHiERow = 68;               // epilogue scratch row (u32): 64 values + pad
constexpr int kHiE5Row = 44;              // 5-plane epilogue row (u32): 40 columns + pad
constexpr int kHiE5Rows = 20;             // (position, part, plane e < 5)
constexpr size_t kHiEpiBytes = (size_t)kHiWarps * 16 * kHiERow * 4;
constexpr size_t kHiEpi5Bytes = (size_t)kHiWarps * kHiE5Rows * kHiE5Row * 4;
constexpr size_t kHiSmemMax = 226 * 1024;  // dynamic (227 KB less the static barriers)
// padded column stride of an RS-step ring (== 16 mod 128: conflict-free ldmatrix)
__host__ __device__ constexpr int hi_rkp(int rs) { return (32 * rs + 127) / 128 * 128 + 16; }

__device__ __forceinline__ int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ void mma_u8(int (&c)[4], const uint4& a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];\n" : "=r"(r0), "=r"(r1) : "r"(addr));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}

// mbarrier / bulk-copy (TMA) pipeline primitives
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

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// byte d of four words -> one u32 (word i in byte i)
__device__ __forceinline__ uint32_t gather_byte(const u64d (&w)[4], int d) {
  const int sh = 8 * (d & 3);
  uint32_t x[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = (uint32_t)(d < 4 ? w[i] : (w[i] >> 32)) >> sh;
  return (x[0] & 0xFF) | ((x[1] & 0xFF) << 8) | ((x[2] & 0xFF) << 16) | (x[3] << 24);
}

struct HiArgs {
  PrimeTable pt;
  const u64d* D;      // [B][l][l+1][N] ModUp digits, slot order, canonical
  const u64d* v;      // [B][2][l][N] input ciphertexts (c0 = poly 0)
  const uint4* wt;    // [l+1][N/16][NSG][4][4][32] A fragments of this chunk
  const u64d* ec;     // [np][2][4][2] (2^(24 g + 32 h) mod q, Shoup companion)
  u64d* acc;          // [B][2][l+1][N]
  int B, L, N, NSG, r_hi, nig, strips, accumulate;
  int RS, RKP, depth;  // ring steps, ring column stride (bytes), pipeline stages
  int ntl, tl[8];      // the ext-basis limbs this launch covers (one byte-plane class)
};

// k-step (32 kappa bytes) holding the first kappa of position kh's band
template <int J>
__device__ __forceinline__ int sfirst(int kh, int r_hi) {
  return floor_div((kh - r_hi) * J, 32);
}

// PL = byte planes of the window elements (8; 5 for limbs of primes < 2^40,
// whose residues have 5 bytes): PL = 8 warps own 4 positions x 4 images
// (n-tile = one image's 8 planes), PL = 5 warps own 2 positions x 8 images
// (5 n-tiles of 8 (image, plane) columns)
template <int J, int PL>
__global__ void __launch_bounds__(32 * kHiWarps, 1) k_hs_imma(HiArgs a) {
  constexpr int LV = J - 1;
  constexpr int COLS = kHiBc * PL;
  extern __shared__ __align__(16) uint8_t hi_smem[];
  __shared__ __align__(8) uint64_t bars[2 * kHiMaxDepth];  // full[d], empty[d]
  const int RS = a.RS, RK = 32 * a.RS, RKP = a.RKP, DEP = a.depth;
  uint8_t* ring = hi_smem;  // [COLS][RKP]
  uint4* astage = reinterpret_cast<uint4*>(hi_smem + (size_t)COLS * RKP);  // [DEP][kHiStage]
  uint32_t* epi = reinterpret_cast<uint32_t*>(astage + DEP * kHiStage);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // PL = 8: position group mg (4 positions), images 4 ng ..; PL = 5:
  // position pair mg (2 positions), images 8 ng ..
  const int mg = PL == 8 ? warp >> 2 : warp >> 1, ng = PL == 8 ? warp & 3 : warp & 1;
  const int N = a.N, S = N >> 1, bps = S / kHiKB, NSG = a.NSG;
  const int ig = blockIdx.x % a.nig, strip = blockIdx.x / a.nig;
  const long T = (long)a.ntl * 2 * bps;
  const long blk0 = T * strip / a.strips, blk1 = T * (strip + 1) / a.strips;
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring);
  const uint32_t astage_s = (uint32_t)__cvta_generic_to_shared(astage);
  uint32_t* E = epi + warp * (PL == 8 ? 16 * kHiERow : kHiE5Rows * kHiE5Row);
  // ldmatrix row address of this lane (before the k-step offset): matrix
  // lane/8 = (n-tile pair member, kappa half), row lane%8 = byte plane
  const int lm = lane >> 3, lrow = lane & 7;
  constexpr int NT = PL == 8 ? 4 : 5;  // n-tiles per warp
  const int nt0 = ng * NT;              // first n-tile of the warp
  const uint32_t lbase0 = ring_s + (uint32_t)((nt0 + (lm >> 1)) * 8 + lrow) * RKP + 16 * (lm & 1);
  const uint32_t lbase1 = lbase0 + 2 * 8 * RKP;  // n-tiles +2, +3
  const uint32_t lbase2 = ring_s + (uint32_t)((nt0 + 4) * 8 + lrow) * RKP + 16 * ((lane >> 3) & 1);  // n-tile +4 (x2)
  const uint32_t full_s = (uint32_t)__cvta_generic_to_shared(bars), empty_s = full_s + 8 * kHiMaxDepth;
  if (threadIdx.x == 0) {
    for (int d = 0; d < DEP; ++d) {
      mbar_init(full_s + 8 * d, 1);
      mbar_init(empty_s + 8 * d, kHiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // A-fragment stages: one bulk copy (8 KB) per k-step, issued by thread 0
  // into stage pst (phase pph); consumers read stage cst (phase cph)
  uint32_t pst = 0, pph = 0, cst = 0, cph = 0;
  auto produce = [&](const uint4* src) {
    mbar_wait(empty_s + 8 * pst, pph ^ 1);  // passes at once on a fresh barrier
    mbar_expect_tx(full_s + 8 * pst, kHiStage * 16);
    bulk_g2s(astage_s + pst * kHiStage * 16, src, kHiStage * 16, full_s + 8 * pst);
    if (++pst == (uint32_t)DEP) pst = 0, pph ^= 1;
  };
  int cur_seg = -1, st_hi = 0;
  for (long blk = blk0; blk < blk1; ++blk) {
    const int seg = (int)(blk / bps), kb = (int)(blk % bps);
    const int t = a.tl[seg >> 1], half = seg & 1, kh0 = kb * kHiKB;
    const int lo_s = sfirst<J>(kh0, a.r_hi), hi_s = sfirst<J>(kh0 + kHiKB - 4, a.r_hi) + NSG;
    __syncthreads();  // all warps are done with the previous block's ring
    if (seg != cur_seg) {
      cur_seg = seg;
      st_hi = lo_s;
    }
    // ---- A-fragment pipeline prologue: steps 0 .. D-2
    const uint4* wsrc = a.wt + ((size_t)t * (N / kHiKB) + (size_t)half * bps + kb) * NSG * kHiStage;
    if (threadIdx.x == 0)
      for (int d = 0; d < DEP - 1 && d < NSG; ++d) produce(wsrc + (size_t)d * kHiStage);
    // ---- stage window steps [st_hi, hi_s): items = (image, 4 kappa bytes)
    {
      const int nk4 = 8 * (hi_s - st_hi), items = nk4 * kHiBc;
      const u64d* Dt = a.D + (size_t)t * N + (size_t)half * S;
      const u64d* ct = a.v + (size_t)t * N + (size_t)half * S;
      for (int it = threadIdx.x; it < items; it += 32 * kHiWarps) {
        const int img = it / nk4, k4 = 8 * st_hi + it % nk4, b = ig * kHiBc + img;
        u64d w[4];
        int pos = floor_div(4 * k4, J), j = 4 * k4 - pos * J;
        const u64d* Db = Dt + (size_t)b * LV * (LV + 1) * N;
        const u64d* cb = ct + (size_t)b * 2 * LV * N;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const int pm = pos & (S - 1);  // S is a power of two
          u64d val = 0;
          if (b < a.B) {
            if (j < LV) val = __ldg(Db + (size_t)j * (LV + 1) * N + pm);
            else if (t < LV) val = __ldg(cb + pm);
          }
          w[x] = val;
          if (++j == J) j = 0, ++pos;
        }
        int off = (4 * k4) % RK;
        if (off < 0) off += RK;
#pragma unroll
        for (int d = 0; d < PL; ++d)
          *reinterpret_cast<uint32_t*>(ring + (size_t)(img * PL + d) * RKP + off) = gather_byte(w, d);
      }
      st_hi = hi_s;
    }
    __syncthreads();  // the window is staged
    // ---- warp: PL = 8: positions kh0 + 4 mg + u (u < 4), images ig*16 +
    // 4 ng + n; PL = 5: positions kh0 + 2 mg + u (u < 2), images ig*16 + 8 ng
    // + ...; every warp walks the same NSG local steps of its 4-position group
    constexpr int MT = PL == 8 ? 4 : 2;
    const int kw = kh0 + MT * mg, grp = PL == 8 ? mg : mg >> 1, u0 = PL == 8 ? 0 : 2 * (mg & 1);
    const int s0 = sfirst<J>(kh0 + 4 * grp, a.r_hi);
    int c[MT][NT][4];
#pragma unroll
    for (int u = 0; u < MT; ++u)
#pragma unroll
      for (int n = 0; n < NT; ++n) c[u][n][0] = c[u][n][1] = c[u][n][2] = c[u][n][3] = 0;
    const uint4* arow = astage + (grp * 4 + u0) * 32 + lane;
    int off = (32 * s0) % RK;
    if (off < 0) off += RK;
    for (int ls = 0; ls < NSG; ++ls) {
      const uint32_t st = cst;
      mbar_wait(full_s + 8 * st, cph);
      if (++cst == (uint32_t)DEP) cst = 0, cph ^= 1;
      const uint4* as = arow + st * kHiStage;
      uint4 ac[MT];
#pragma unroll
      for (int u = 0; u < MT; ++u) ac[u] = as[u * 32];
      uint32_t b0[NT], b1[NT];
      ldsm_x4(lbase0 + off, b0[0], b1[0], b0[1], b1[1]);
      ldsm_x4(lbase1 + off, b0[2], b1[2], b0[3], b1[3]);
      if constexpr (NT == 5) ldsm_x2(lbase2 + off, b0[4], b1[4]);
      off += 32;
      if (off == RK) off = 0;
      __syncwarp();
      if (lane == 0) mbar_arrive(empty_s + 8 * st);  // this warp is done with the stage
      if (threadIdx.x == 0 && ls + DEP - 1 < NSG) produce(wsrc + (size_t)(ls + DEP - 1) * kHiStage);
#pragma unroll
      for (int u = 0; u < MT; ++u)
#pragma unroll
        for (int n = 0; n < NT; ++n) mma_u8(c[u][n], ac[u], b0[n], b1[n]);
    }
    const int pi = t == LV ? a.L : t;
    const DevPrime pr = a.pt.p[pi];
    if constexpr (PL == 8) {
      // ---- epilogue: two rounds of 2 positions x 4 images x 2 parts = 16
      // outputs through the warp's scratch; lane (o, dh) combines the byte
      // planes e < 8, d in [4 dh, 4 dh + 4) of output o
      const int o = lane & 15, dh = lane >> 4;
      const u64d* ecp = a.ec + ((size_t)pi * 2 + dh) * 8;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        __syncwarp();
#pragma unroll
        for (int uu = 0; uu < 2; ++uu)
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            const int o0 = (uu * 4 + n) * 2, col = (lane >> 2) * 8 + 2 * (lane & 3);
            *reinterpret_cast<uint2*>(E + o0 * kHiERow + col) =
                make_uint2((uint32_t)c[2 * h + uu][n][0], (uint32_t)c[2 * h + uu][n][1]);
            *reinterpret_cast<uint2*>(E + (o0 + 1) * kHiERow + col) =
                make_uint2((uint32_t)c[2 * h + uu][n][2], (uint32_t)c[2 * h + uu][n][3]);
          }
        __syncwarp();
        u64d A[4] = {0, 0, 0, 0};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint4 q4 = *reinterpret_cast<const uint4*>(E + o * kHiERow + e * 8 + 4 * dh);
          const uint32_t cv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
          for (int dd = 0; dd < 4; ++dd) {
            const int sp = e + dd;  // + 4 dh (applied through the constants)
            A[sp / 3] += (u64d)cv[dd] << (8 * (sp % 3));
          }
        }
        u64d sum = 0;  // < 8q
#pragma unroll
        for (int g = 0; g < 4; ++g) sum += shoup_mul_lazy(A[g], __ldg(ecp + 2 * g), __ldg(ecp + 2 * g + 1), pr.q);
        sum = shoup_mul_d(sum, 1ull, pr.one_sh, pr.q);
        sum = add_mod_d(sum, __shfl_xor_sync(0xffffffffu, sum, 16), pr.q);
        if (dh == 0) {
          const int uu = o >> 3, n = (o >> 1) & 3, p = o & 1;
          const int b = ig * kHiBc + 4 * ng + n, k = half * S + kw + 2 * h + uu;
          if (b < a.B) {
            u64d* dst = a.acc + ((size_t)b * 2 + p) * (LV + 1) * N + (size_t)t * N + k;
            *dst = a.accumulate ? add_mod_d(sum, *dst, pr.q) : sum;
          }
        }
      }
    } else {
      // ---- epilogue (5 planes): the warp's 2 positions x 8 images x 2 parts
      // = 32 outputs, one per lane; weight planes e >= 5 are zero (q < 2^40)
      // so only rows e < 5 are kept: scratch [(u, p, e)][40 columns]
      const int e = lane >> 2;
      __syncwarp();
      if (e < 5) {
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int n = 0; n < 5; ++n) {
            const int col = n * 8 + 2 * (lane & 3);
            *reinterpret_cast<uint2*>(E + ((u * 2 + 0) * 5 + e) * kHiE5Row + col) =
                make_uint2((uint32_t)c[u][n][0], (uint32_t)c[u][n][1]);
            *reinterpret_cast<uint2*>(E + ((u * 2 + 1) * 5 + e) * kHiE5Row + col) =
                make_uint2((uint32_t)c[u][n][2], (uint32_t)c[u][n][3]);
          }
      }
      __syncwarp();
      const int u = lane >> 4, img = (lane >> 1) & 7, p = lane & 1;
      u64d A[3] = {0, 0, 0};
#pragma unroll
      for (int ee = 0; ee < 5; ++ee)
#pragma unroll
        for (int d = 0; d < 5; ++d) {
          const int sp = ee + d;
          A[sp / 3] += (u64d)E[((u * 2 + p) * 5 + ee) * kHiE5Row + img * 5 + d] << (8 * (sp % 3));
        }
      const u64d* ecp = a.ec + (size_t)pi * 2 * 8;  // 2^(24 g), g < 3
      u64d sum = 0;  // < 6q
#pragma unroll
      for (int g = 0; g < 3; ++g) sum += shoup_mul_lazy(A[g], __ldg(ecp + 2 * g), __ldg(ecp + 2 * g + 1), pr.q);
      sum = shoup_mul_d(sum, 1ull, pr.one_sh, pr.q);
      const int b = ig * kHiBc + 8 * ng + img, k = half * S + kw + u;
      if (b < a.B) {
        u64d* dst = a.acc + ((size_t)b * 2 + p) * (LV + 1) * N + (size_t)t * N + k;
        *dst = a.accumulate ? add_mod_d(sum, *dst, pr.q) : sum;
      }
    }
  }
}

// A fragments of one chunk: thread = (t, block, local step, group, position, lane)
template <int J>
__global__ void k_hs_imma_tiles(PrimeTable pt, const u64d* __restrict__ fk, size_t fk_words, int first_keyed,
                                const u64d* __restrict__ masks, const int* __restrict__ rdiag, const u64d* pmod,
                                int L, int N, int NSG, int r_lo, int r_hi, uint4* __restrict__ wt) {
  constexpr int LV = J - 1;
  const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(gid & 31), u = (int)((gid >> 5) & 3), g4 = (int)((gid >> 7) & 3);
  const size_t item = gid >> 9;  // (t, kb, ls)
  const int nkb = N / kHiKB;
  const size_t total = (size_t)(LV + 1) * nkb * NSG;
  if (item >= total) return;
  const int ls = (int)(item % NSG), kb = (int)((item / NSG) % nkb), t = (int)(item / ((size_t)NSG * nkb));
  const int S = N >> 1, k = kb * kHiKB + 4 * g4 + u, kh = k & (S - 1);
  const int pi = t == LV ? L : t;
  const DevPrime pr = pt.p[pi];
  const int s = floor_div((kh - u - r_hi) * J, 32) + ls, e = lane >> 2;
  uint32_t reg[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int p = i & 1, kk = (i >> 1) * 16 + 4 * (lane & 3);
    uint32_t word = 0;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int kap = 32 * s + kk + x, pos = floor_div(kap, J), j = kap - pos * J, r = kh - pos;
      if (r < r_lo || r > r_hi) continue;
      const int di = rdiag[r];
      if (di < 0) continue;
      u64d w = 0;
      if (j < LV) {
        if (r != 0) {
          const u64d f = fk[(size_t)(di - first_keyed) * fk_words + ((size_t)(j * 2 + p) * (LV + 1) + t) * N + k];
          w = mont_mul(unsplit31(f), 1ull, pr.q, pr.qneg_inv);
        }
      } else if (p == 0 && t < LV) {
        const u64d m = masks[((size_t)di * (LV + 1) + t) * N + k];
        w = mont_mul(unsplit31(m), pmod[t], pr.q, pr.qneg_inv);
      }
      word |= (uint32_t)((w >> (8 * e)) & 0xFF) << (8 * x);
    }
    reg[i] = word;
  }
  wt[gid] = make_uint4(reg[0], reg[1], reg[2], reg[3]);
}

// cacc for the IMMA path: the c0 * mask term lives in acc (P-scaled), so
// cacc holds only diagonal 0's c1 * mask term (part 1)
__global__ void k_hs_cacc(const u64d* __restrict__ v, const u64d* __restrict__ m0, PrimeTable pt, int B, int l,
                          int N, int c1_term, u64d* __restrict__ cacc) {
  const size_t total = (size_t)B * 2 * l * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % N), t = (int)((i / N) % l), p = (int)((i / ((size_t)l * N)) % 2);
    const size_t b = i / ((size_t)2 * l * N);
    u64d r = 0;
    if (p == 1 && c1_term) {
      const DevPrime pr = pt.p[t];
      r = mont_mul(v[(b * 2 + 1) * l * N + (size_t)t * N + k], unsplit31(m0[(size_t)t * N + k]), pr.q, pr.qneg_inv);
    }
    cacc[i] = r;
  }
}

template <int J, int PL>
void hs_imma_go(Context& c, const HiArgs& a, size_t smem, int grid, double bytes, double ops) {
  static PerDeviceOnce prepared;
  if (prepared.first())
    CK(cudaFuncSetAttribute(k_hs_imma<J, PL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHiSmemMax));
  LAUNCH_BO(c, "k_hs_imma", bytes, ops, (k_hs_imma<J, PL><<<grid, 32 * kHiWarps, smem, c.stream>>>(a)));
}

template <int J>
void hs_tiles_go(Context& c, const HsDiagTable& t, const u64d* pmod, const int* rdiag, const HsImmaChunk& ch,
                 uint4* wt) {
  const size_t threads = (size_t)J * c.N() * ch.ns * 32;  // (t, position, local step, lane)
  LAUNCH(c, "k_hs_imma_tiles",
         k_hs_imma_tiles<J><<<(unsigned)((threads + 255) / 256), 256, 0, c.stream>>>(
             c.primes, t.fk, t.fk_words, t.first_keyed, t.masks, rdiag, pmod, c.L(), c.N(), ch.ns, ch.r_lo,
             ch.r_hi, wt));
}

}  // namespace

int hs_imma_chunk_span(int l) {
  const int J = l + 1;
  // ring: NSG + ceil(12 J / 32) + 1 <= kHiRSMax, NSG = floor((span J + 62) / 32) + 1
  const int span = ((kHiRSMax - 2 - (12 * J + 31) / 32) * 32 - 31) / J;
  return span < 128 ? span : 128;
}

bool hs_imma_supported(Context& c, int l) { return l >= 1 && l <= 6 && c.S() % kHiKB == 0 && c.S() >= 64; }

size_t hs_imma_tile_words(Context& c, int l, const HsImmaChunk& ch) {
  return (size_t)(l + 1) * c.N() * ch.ns * 32 * 2;  // uint4 = 2 words; ns = NSG (group steps)
}

void launch_hs_imma_tiles(Context& c, int l, const HsDiagTable& t, const u64d* pmod, const int* rdiag,
                          const HsImmaChunk& ch, u64d* wt) {
  uint4* w4 = reinterpret_cast<uint4*>(wt);
  switch (l + 1) {
    case 2: hs_tiles_go<2>(c, t, pmod, rdiag, ch, w4); break;
    case 3: hs_tiles_go<3>(c, t, pmod, rdiag, ch, w4); break;
    case 4: hs_tiles_go<4>(c, t, pmod, rdiag, ch, w4); break;
    case 5: hs_tiles_go<5>(c, t, pmod, rdiag, ch, w4); break;
    case 6: hs_tiles_go<6>(c, t, pmod, rdiag, ch, w4); break;
    case 7: hs_tiles_go<7>(c, t, pmod, rdiag, ch, w4); break;
    default: fail(HEGPU_ERR_ARG, "hs_imma: level out of range");
  }
}

void launch_hs_imma(Context& c, const u64d* v, int B, int l, const u64d* D, const HsImmaChunk& ch,
                    const u64d* ec, int accumulate, u64d* acc) {
  const int keyed = ch.keyed, ndiag = ch.ndiag;
  const int N = c.N(), S = N / 2, J = l + 1;
  HiArgs a{};
  a.pt = c.primes;
  a.D = D;
  a.v = v;
  a.wt = reinterpret_cast<const uint4*>(ch.wt);
  a.ec = ec;
  a.acc = acc;
  a.B = B;
  a.L = c.L();
  a.N = N;
  a.NSG = ch.ns;
  a.r_hi = ch.r_hi;
  a.nig = (B + kHiBc - 1) / kHiBc;
  a.accumulate = accumulate;
  const int sms = device_sms();
  // ring: the block's steps [sfirst(kh0), sfirst(kh0 + 12) + NSG)
  a.RS = ch.ns + (12 * J + 31) / 32 + 1;
  if (a.RS > kHiRSMax) fail(HEGPU_ERR_ARG, "hs_imma: chunk span exceeds the window ring");
  a.RKP = hi_rkp(a.RS);
  // limbs by byte-plane class: residues of primes < 2^40 have 5 bytes
  std::vector<int> cls[2];  // [0]: 8 planes, [1]: 5 planes
  for (int t = 0; t <= l; ++t) {
    const u64 q = c.P->q(t == l ? c.L() : t);
    cls[q < (1ull << 40) ? 1 : 0].push_back(t);
  }
  for (int ci = 0; ci < 2; ++ci) {
    if (cls[ci].empty()) continue;
    const int PL = ci ? 5 : 8;
    a.ntl = (int)cls[ci].size();
    for (int i = 0; i < a.ntl; ++i) a.tl[i] = cls[ci][i];
    const long T = (long)a.ntl * 2 * (S / kHiKB);
    long strips = sms / a.nig;
    if (strips < 1) strips = 1;
    if (strips > T) strips = T;
    a.strips = (int)strips;
    // the rest of shared memory goes to A-fragment stages
    const size_t fixed = (size_t)kHiBc * PL * a.RKP + (PL == 8 ? kHiEpiBytes : kHiEpi5Bytes);
    int depth = (int)((kHiSmemMax - 64 - fixed) / (kHiStage * 16));
    if (depth > kHiMaxDepth) depth = kHiMaxDepth;
    if (depth < 2) fail(HEGPU_ERR_ARG, "hs_imma: shared memory too small");
    a.depth = depth;
    const size_t smem = fixed + (size_t)depth * kHiStage * 16;
    // the chunk's A fragments once, D/c0 windows once per strip (~once), acc
    // written (and read back when accumulating) -- for this launch's limbs
    const double NB = 8.0 * N, fr = (double)a.ntl / J;
    const double bytes =
        fr * (16.0 * ch.ns * 32 * J * N + NB * B * (l * J + l) + NB * B * 2 * J * (accumulate ? 2 : 1));
    const double ops = fr * (double)N * B * (keyed * l * J * 2.0 + ndiag * l);  // modular MAC terms
    const int grid = (int)(a.nig * strips);
#define HI_GO(JJ)                                                               \
  case JJ:                                                                      \
    if (PL == 8) hs_imma_go<JJ, 8>(c, a, smem, grid, bytes, ops);               \
    else hs_imma_go<JJ, 5>(c, a, smem, grid, bytes, ops);                       \
    break;
    switch (J) {
      HI_GO(2) HI_GO(3) HI_GO(4) HI_GO(5) HI_GO(6) HI_GO(7)
      default: fail(HEGPU_ERR_ARG, "hs_imma: level out of range");
    }
#undef HI_GO
  }
}

void launch_hs_cacc(Context& c, const u64d* v, const u64d* m0, int B, int l, int c1_term, u64d* cacc) {
  const size_t total = (size_t)B * 2 * l * c.N();
  unsigned g = (unsigned)((total + 255) / 256);
  if (g > 148 * 16) g = 148 * 16;
  LAUNCH_B(c, "k_hs_cacc", 8.0 * total * (c1_term ? 1.5 : 1.0),
           k_hs_cacc<<<g, 256, 0, c.stream>>>(v, m0, c.primes, B, l, c.N(), c1_term, cacc));
}

}  // namespace hegpu
