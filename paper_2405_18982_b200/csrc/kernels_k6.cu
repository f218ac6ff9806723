// Kernels for degree k=6 (see patch_kernels.cuh).
#define IPMG_K 6
#include "patch_kernels.cuh"
