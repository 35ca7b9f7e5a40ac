// tools/ubench_int.cu -- throughput of the integer / FP64 primitives the
// RNS kernels are built from, on the B200 this runs on (informs DESIGN.md §5).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_int tools/ubench_int.cu
#include <cstdio>
#include <cstdint>

#define ITERS 4096
#define ACC 8

__global__ void k_imad_wide(uint64_t* out, uint32_t a, uint32_t b) {
  uint64_t acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = threadIdx.x + i;
  uint32_t x = a ^ threadIdx.x, y = b;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      uint64_t r;
      asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(x + i), "r"(y), "l"(acc[i]));
      acc[i] = r;
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_imad32(uint64_t* out, uint32_t a, uint32_t b) {
  uint32_t acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = threadIdx.x + i;
  uint32_t x = a ^ threadIdx.x, y = b;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      uint32_t r;
      asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x + i), "r"(y), "r"(acc[i]));
      acc[i] = r;
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_mulhi64(uint64_t* out, uint64_t a, uint64_t b) {
  uint64_t acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = a + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = __umul64hi(acc[i], b) + acc[i];
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dfma(uint64_t* out, double a, double b) {
  double acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = a + threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) acc[i] = fma(acc[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (uint64_t)s;
}

__global__ void k_iadd3(uint64_t* out, uint32_t a, uint32_t b) {
  uint32_t acc[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) acc[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      uint32_t r;
      asm volatile("add.u32 %0, %1, %2;" : "=r"(r) : "r"(acc[i]), "r"(a ^ i));
      acc[i] = r;
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s ^= acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K, typename... A>
void run(const char* name, K k, int ops_per_iter, A... args) {
  int blocks = 148 * 8, threads = 256;
  uint64_t* out;
  cudaMalloc(&out, (size_t)blocks * threads * 8);
  k<<<blocks, threads>>>(out, args...);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, args...);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * ITERS * ACC * ops_per_iter;
  std::printf("%-14s %8.3f ms  %8.2f Tops/s  (%.1f per SM per clk @1.965GHz)\n", name, ms, ops / ms / 1e9,
              ops / (ms * 1e-3) / 148 / 1.965e9);
  cudaFree(out);
}

int main() {
  run("imad32", k_imad32, 1, 3u, 5u);
  run("imad.wide.u32", k_imad_wide, 1, 3u, 5u);
  run("iadd32", k_iadd3, 1, 3u, 5u);
  run("umul64hi+add", k_mulhi64, 1, (uint64_t)3, (uint64_t)0x9E3779B97F4A7C15ull);
  run("dfma", k_dfma, 1, 1.0000001, 0.9999999);
  return 0;
}
