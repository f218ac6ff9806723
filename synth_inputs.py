"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA-path
tests/bench (the ONLY module both sides use).  It holds no arithmetic of the
method: only random vectors and the workload shapes of BASELINE.json /
SURVEY.md section 8(d) ("Synthetic inputs": x ~ U(-1,1) i.i.d. from numpy PCG64,
seed 0; fp32 inputs are the cast of the fp64 draw).
"""
import numpy as np


def uniform(n, seed=0, lo=-1.0, hi=1.0):
    """x ~ U(lo, hi) i.i.d., numpy PCG64 with the given seed, float64."""
    return np.random.Generator(np.random.PCG64(seed)).uniform(lo, hi, size=int(n))


def n_levels_for(cells_per_dir_finest, n0=2):
    """Number of levels l = 0..L-1 so that n0 * 2^(L-1) = cells_per_dir_finest."""
    L, c = 1, n0
    while c < cells_per_dir_finest:
        c *= 2
        L += 1
    if c != cells_per_dir_finest:
        raise ValueError("finest cell count must be n0 * 2^m")
    return L


# Workloads; dofs = prod(cells) * (k+1)^d.
WORKLOADS = {
    # BASELINE.json configs[0]: oracle-sized, CPU seconds
    "C1": dict(dim=2, degree=2, coarse=(2, 2), n_levels=3),
    # BASELINE.json configs[1]: 2D k=7, 1024^2 cells, 67,108,864 dofs, mixed fp32/fp64
    "C2": dict(dim=2, degree=7, coarse=(2, 2), n_levels=10),
}
