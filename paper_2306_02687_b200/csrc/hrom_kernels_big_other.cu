// k_increment_big for the widths outside BASELINE configs 3/4 (NP = 40, 48,
// 56, 80, 96, 112) in their own translation unit, with the assembly pass
// forced inline (NVVM otherwise calls it as a function there: a 1.3 KB stack
// frame per thread).
#define FE2_BIG_OTHER_TU
#define FE2_BIG_INLINE_PASS
#include "hrom_kernels_big.cu"
