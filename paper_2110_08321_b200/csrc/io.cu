// io.cu -- expansion of compact fresh ciphertexts on the device.
//
// A fresh symmetric encryption is (c0, c1 = a) with a uniform and generated
// from a counter-based stream.  The compact wire form
// (Client::encrypt_compact) ships only c0, byte-packed per prime
// (ceil(bits(q_i)/8) bytes per coefficient: 5 for the 40-bit primes), plus
// the per-limb a-stream keys; this kernel unpacks c0, regenerates a, and
// writes the device layout (slot order) directly -- 2.9x fewer bytes over
// PCIe for the config-0 taps, bit-identical ciphertexts.
#include "compact.cuh"
#include "engine.hpp"

namespace hegpu {

namespace {

// c0 rows (ct, t): the packed limb is already in slot order, so position
// pos reads bytes [pos * nb, pos * nb + nb) -- a linear, coalesced unpack
__global__ void k_expand_c0(const uint8_t* __restrict__ src, u64d* __restrict__ dst, CompactLayout lay,
                            const uint32_t* __restrict__ slot_src, int N) {
  const int l = lay.level;
  const int row = blockIdx.y, t = row % l, c = row / l;
  const int nb = lay.nb[t];
  const u64d* limb = reinterpret_cast<const u64d*>(src + (size_t)c * lay.ct_bytes + lay.off[t]);
  const int words = (N * nb) >> 3;
  u64d* out = dst + ((size_t)c * 2 * l + t) * N;
#pragma unroll 4
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < N; pos += gridDim.x * blockDim.x)
    out[pos] = compact_c0(limb, pos * nb, nb, words);
}

// c1 = a rows (ct, t): regenerated from the limb's a-stream key
__global__ void k_expand_a(const uint8_t* __restrict__ src, u64d* __restrict__ dst, CompactLayout lay,
                           PrimeTable pt, const uint32_t* __restrict__ slot_src, int N) {
  const int l = lay.level;
  const int row = blockIdx.y, t = row % l, c = row / l;
  const u64d key = reinterpret_cast<const u64d*>(src + (size_t)c * lay.ct_bytes)[t];
  const u64d q = pt.p[t].q;
  u64d* out = dst + ((size_t)c * 2 * l + l + t) * N;
#pragma unroll 4
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < N; pos += gridDim.x * blockDim.x)
    out[pos] = compact_a(key, __ldg(slot_src + pos), q);
}

}  // namespace

size_t compact_ct_bytes(Context& c, int level) { return c.client->compact_bytes(level); }

CompactLayout compact_layout(Context& c, int level) {
  CompactLayout lay{};
  lay.level = level;
  long off = (long)level * 8;
  for (int t = 0; t < level; ++t) {
    lay.nb[t] = c.client->limb_bytes(t);
    lay.off[t] = off;
    off += (long)c.N() * lay.nb[t];
  }
  lay.ct_bytes = off;
  return lay;
}

void launch_expand_compact(Context& c, const uint8_t* src, int count, int level, u64d* dst) {
  const CompactLayout lay = compact_layout(c, level);
  const long off = lay.ct_bytes;
  const int N = c.N();
  dim3 grid((N + 255) / 256 < 8 ? (N + 255) / 256 : 8, (unsigned)(count * level));
  const double c0_bytes = (double)count * (off - 8.0 * level + 8.0 * level * N);
  LAUNCH_B(c, "k_expand_compact", c0_bytes,
           k_expand_c0<<<grid, 256, 0, c.stream>>>(src, dst, lay, c.d_slot_src, N));
  LAUNCH_B(c, "k_expand_compact", (double)count * (8.0 * level + 8.0 * level * N),
           k_expand_a<<<grid, 256, 0, c.stream>>>(src, dst, lay, c.primes, c.d_slot_src, N));
}

}  // namespace hegpu
