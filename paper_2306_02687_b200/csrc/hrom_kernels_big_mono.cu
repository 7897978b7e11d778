// The monolithic-iteration instantiations of k_increment_big (MONO = true,
// fe2_hrom_mono_iterate for n > 32) in their own translation unit: sharing
// one with the increment kernels changed NVVM's inlining of the assembly pass
// there (a second call site) and cost the n = 128 kernel its registers.
#define FE2_BIG_MONO_TU
#include "hrom_kernels_big.cu"
