// k_increment_big for models whose history-carrying points follow an
// iterative material (power law / creep: GEN = true, every width), in their
// own translation unit so the J2 instantiations keep their inlining and
// registers; the assembly pass is forced inline here.
#define FE2_BIG_GEN_TU
#define FE2_BIG_INLINE_PASS
#include "hrom_kernels_big.cu"
