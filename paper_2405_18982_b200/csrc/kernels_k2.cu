// Kernels for degree k=2 (see patch_kernels.cuh).
#define IPMG_K 2
#include "patch_kernels.cuh"
