// tools/ubench_mma.cu -- legacy mma.sync int8 (m16n8k32, s32 accumulate)
// throughput on this GPU (informs the conv-MAC design)
#include <cstdio>
#include <cstdint>

__global__ void k_mma(int* out, int iters) {
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x55, b1 = a0 ^ 0x33;
  int c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+r"(c[u][0]), "+r"(c[u][1]), "+r"(c[u][2]), "+r"(c[u][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int u = 0; u < 8; ++u) s += c[u][0] + c[u][1] + c[u][2] + c[u][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int* out;
  const int blocks = 148 * 4, threads = 256, iters = 4096;
  cudaMalloc(&out, blocks * threads * 4);
  k_mma<<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mma<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * (blocks * threads / 32);
  std::printf("mma.sync m16n8k32 u8: %.3f ms, %.1f TOPS (int8 ops, 2 per MAC)\n", ms, ops / ms / 1e9);
  return 0;
}
