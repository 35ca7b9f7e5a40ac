// io.cu -- expansion of compact fresh ciphertexts on the device.
//
// A fresh symmetric encryption is (c0, c1 = a) with a uniform and generated
// from a counter-based stream.  The compact wire form
// (Client::encrypt_compact) ships only c0, byte-packed per prime
// (ceil(bits(q_i)/8) bytes per coefficient: 5 for the 40-bit primes), plus
// the per-limb a-stream keys; this kernel unpacks c0, regenerates a, and
// writes the device layout (slot order) directly -- 2.9x fewer bytes over
// PCIe for the config-0 taps, bit-identical ciphertexts.
#include "engine.hpp"

namespace hegpu {

namespace {

__device__ __forceinline__ u64d sm_mix_d(u64d z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct CompactLayout {
  int level;
  int nb[HEGPU_MAX_PRIMES];       // bytes per coefficient of limb t
  long off[HEGPU_MAX_PRIMES];     // byte offset of limb t inside one compact ct
  long ct_bytes;
};

// rows (ct, p, t); positions p in slot order
__global__ void k_expand_compact(const uint8_t* __restrict__ src, u64d* __restrict__ dst, CompactLayout lay,
                                 PrimeTable pt, const uint32_t* __restrict__ slot_src, int N) {
  const int l = lay.level;
  const int row = blockIdx.y, t = row % l, p = (row / l) & 1, c = row / (2 * l);
  const uint8_t* base = src + (size_t)c * lay.ct_bytes;
  u64d* out = dst + ((size_t)c * 2 * l + (size_t)p * l + t) * N;
  const u64d q = pt.p[t].q;
  if (p == 0) {
    const int nb = lay.nb[t];
    const uint8_t* limb = base + lay.off[t];
    for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < N; pos += gridDim.x * blockDim.x) {
      const uint8_t* b = limb + (size_t)__ldg(slot_src + pos) * nb;
      u64d v = 0;
      for (int i = nb - 1; i >= 0; --i) v = (v << 8) | __ldg(b + i);
      out[pos] = v;
    }
  } else {
    const u64d key = reinterpret_cast<const u64d*>(base)[t];
    for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < N; pos += gridDim.x * blockDim.x) {
      const u64d k = __ldg(slot_src + pos);
      const u64d w = sm_mix_d(key + (k + 1) * 0x9E3779B97F4A7C15ull);
      out[pos] = __umul64hi(w, q);
    }
  }
}

}  // namespace

size_t compact_ct_bytes(Context& c, int level) { return c.client->compact_bytes(level); }

void launch_expand_compact(Context& c, const uint8_t* src, int count, int level, u64d* dst) {
  CompactLayout lay{};
  lay.level = level;
  long off = (long)level * 8;
  for (int t = 0; t < level; ++t) {
    lay.nb[t] = c.client->limb_bytes(t);
    lay.off[t] = off;
    off += (long)c.N() * lay.nb[t];
  }
  lay.ct_bytes = off;
  dim3 grid((c.N() + 255) / 256 < 8 ? (c.N() + 255) / 256 : 8, (unsigned)(count * 2 * level));
  LAUNCH_B(c, "k_expand_compact", (double)count * (off + 16.0 * level * c.N()),
           k_expand_compact<<<grid, 256, 0, c.stream>>>(src, dst, lay, c.primes, c.d_slot_src, c.N()));
}

}  // namespace hegpu
