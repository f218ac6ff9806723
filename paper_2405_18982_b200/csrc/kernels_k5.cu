// Kernels for degree k=5 (see patch_kernels.cuh).
#define IPMG_K 5
#include "patch_kernels.cuh"
