// apply_level_p3.cu -- part 3 of the d >= 2 level kernels' template instantiations (see the
// top of apply_level.cu): compiled as its own translation unit so the parts build in parallel.
#define GPM_LEVEL_PART 3
#include "apply_level.cu"
