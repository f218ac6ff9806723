// Kernels for degree k=3 (see patch_kernels.cuh).
#define IPMG_K 3
#include "patch_kernels.cuh"
