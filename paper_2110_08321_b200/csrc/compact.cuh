// compact.cuh -- device decoding of compact fresh ciphertexts.
//
// One compact ct at level l is [l a-stream keys (u64)] then, per limb t,
// N coefficients of c0 byte-packed in device slot order (position p holds
// wire index slot_src[p]) with nb[t] = ceil(bits(q_t)/8) bytes each.  c1 = a
// is regenerated:
//   a_t[k] = umulhi(sm_mix(key_t + (k + 1) * gamma), q_t)   (client.cpp)
// Used by the expansion kernel (io.cu) and fused into the conv MAC (eval.cu)
// so fresh taps never have to be materialised in HBM.
#pragma once
#include "modarith.cuh"

namespace hegpu {

struct CompactLayout {
  int level;
  int nb[HEGPU_MAX_PRIMES];    // bytes per coefficient of limb t
  long off[HEGPU_MAX_PRIMES];  // byte offset of limb t inside one compact ct
  long ct_bytes;
};

__device__ __forceinline__ u64d sm_mix_d(u64d z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// a-stream word of wire index k (k = slot_src[position])
__device__ __forceinline__ u64d compact_a(u64d key, u64d k, u64d q) {
  return __umul64hi(sm_mix_d(key + (k + 1) * 0x9E3779B97F4A7C15ull), q);
}

// c0 coefficient at byte offset boff (= position * nb) of a packed limb
// of `words` 8-byte words: two aligned loads (the limb is 8-byte aligned)
__device__ __forceinline__ u64d compact_c0(const u64d* __restrict__ limb, int boff, int nb, int words) {
  const int w = boff >> 3, sh = (boff & 7) * 8;
  u64d v = __ldg(limb + w) >> sh;
  if (sh + 8 * nb > 64) v |= __ldg(limb + (w + 1 < words ? w + 1 : w)) << (64 - sh);
  return nb >= 8 ? v : v & ((1ull << (8 * nb)) - 1);
}

}  // namespace hegpu
