// Part 6 of kernels_scalar.cu, compiled as its own translation unit (see _build.py).
#define FQNM_SCALAR_PART 6
#include "kernels_scalar.cu"
