// Dirichlet-kernel smoother for degree k=5 (see patch_kernels.cuh, IPMG_DIRICHLET).
#define IPMG_K 5
#define IPMG_DIRICHLET 1
#include "patch_kernels.cuh"
