// ntt_r8.cu -- the NTT kernels again with 8 words per thread for N <= 2^13
// (1024-thread CTAs, one per SM, no register spills); ntt.cu dispatches the
// row INTT and drop-limb entry points here (measured faster for those).
#define HEGPU_NTT_LR13 3
#define HEGPU_NTT_MINB13 1
#define HEGPU_NTT_R8_VARIANT
#include "ntt.cu"
