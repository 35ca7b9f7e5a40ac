// ntt_fp8.cu -- FP64-only NTT kernels (every prime below 2^45) with 8 words
// per thread and two 1024-thread CTAs per SM for N <= 2^13 (32 registers:
// twice the warps of the other builds to hide FP64 and shared-memory latency).
#define HEGPU_NTT_LR13 3
#define HEGPU_NTT_MINB13 2
#define HEGPU_NTT_FPONLY
#define HEGPU_NTT_R8_VARIANT
#define HEGPU_NTT_SUFFIX _fp8
#include "ntt.cu"
