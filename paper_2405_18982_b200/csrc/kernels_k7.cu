// Kernels for degree k=7 (see patch_kernels.cuh).
#define IPMG_K 7
#include "patch_kernels.cuh"
