// Part 9 of kernels_scalar.cu, compiled as its own translation unit (see _build.py).
#define FQNM_SCALAR_PART 9
#include "kernels_scalar.cu"
