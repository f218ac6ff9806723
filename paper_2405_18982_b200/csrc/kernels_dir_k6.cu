// Dirichlet-kernel smoother for degree k=6 (see patch_kernels.cuh, IPMG_DIRICHLET).
#define IPMG_K 6
#define IPMG_DIRICHLET 1
#include "patch_kernels.cuh"
