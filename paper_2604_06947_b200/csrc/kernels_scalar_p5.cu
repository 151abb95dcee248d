// Part 5 of kernels_scalar.cu, compiled as its own translation unit (see _build.py).
#define FQNM_SCALAR_PART 5
#include "kernels_scalar.cu"
