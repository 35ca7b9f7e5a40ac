// ntt_fp16n.cu -- the drop-limb / fused ModDown + rescale entry points of the
// FP64-only 16-word build without the shared-memory staging of the
// epilogue operands (69 KB per CTA: two 512-thread CTAs per SM; the rows
// are prefetched towards L2 instead).
#define HEGPU_NTT_LR13 4
#define HEGPU_NTT_MINB13 2
#define HEGPU_NTT_FPONLY
#define HEGPU_NTT_R8_VARIANT
#define HEGPU_NTT_ONLY_DROP
#define HEGPU_DROP_PRE 0
#define HEGPU_NTT_SUFFIX _fp16n
#include "ntt.cu"
