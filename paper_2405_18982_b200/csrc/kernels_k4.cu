// Kernels for degree k=4 (see patch_kernels.cuh).
#define IPMG_K 4
#include "patch_kernels.cuh"
