// Kernels for degree k=1 (see patch_kernels.cuh).
#define IPMG_K 1
#include "patch_kernels.cuh"
