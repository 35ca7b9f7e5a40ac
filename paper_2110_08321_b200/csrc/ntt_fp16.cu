// ntt_fp16.cu -- the NTT kernels again for contexts whose primes are all
// below 2^45: FP64 butterflies only (no integer-butterfly code, so no
// register spills), 16 words per thread, two 512-thread CTAs per SM.
#define HEGPU_NTT_LR13 4
#define HEGPU_NTT_MINB13 2
#define HEGPU_NTT_FPONLY
#define HEGPU_NTT_R8_VARIANT
#define HEGPU_NTT_SUFFIX _fp16
#include "ntt.cu"
