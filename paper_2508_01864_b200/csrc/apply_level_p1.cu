// apply_level_p1.cu -- part 1 of the d >= 2 level kernels' template instantiations (see the
// top of apply_level.cu): compiled as its own translation unit so the parts build in parallel.
#define GPM_LEVEL_PART 1
#include "apply_level.cu"
