// apply_level_p2.cu -- part 2 of the d >= 2 level kernels' template instantiations (see the
// top of apply_level.cu): compiled as its own translation unit so the parts build in parallel.
#define GPM_LEVEL_PART 2
#include "apply_level.cu"
