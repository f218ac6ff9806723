"""Vertex-patch Schwarz smoothers with dense local solves (TEST INFRASTRUCTURE
ONLY, see oracle/__init__.py).

Full kernel: V_j = all dofs of the 2^d patch cells; the local
correction is r = b - A x (eq. residual), x <- x + R_j^T A_j^{-1} R_j r
(eq. local-solver), with A_j = R_j A R_j^T *extracted from the assembled
matrix* and factorised by dense LU -- no fast diagonalisation here, so the GPU
path's FD is checked against an independent direct solve.

Multiplicative (Algorithm 1): colours in sequence, patches of
one colour in parallel; the residual is computed globally once per colour from
the pre-colour state ("we decided for updating residuals globally",
PAPER.md:257; reading A9).  Post-smoothing may visit colours in reverse
(reading A7, symmetric V-cycle).

Additive (BASELINE.json configs[4]; not in the paper): x <- x + omega sum_j
R_j^T A_j^{-1} R_j (b - A x), omega = 1/2^d by default (reading A17).
"""
import numpy as np
import scipy.linalg as sla

from . import mesh


class PatchSmoother:
    def __init__(self, level, k, A, dtype=np.float64, cache_by_signature=True):
        self.level, self.k, self.dtype = level, k, np.dtype(dtype)
        self.A = A.astype(self.dtype)
        self.ncolours = 2 ** level.dim
        # groups[c] = list of (lu, idx (npatch, nloc))
        self.groups = []
        for c, plist in enumerate(mesh.coloured_patches(level)):
            bysig = {}
            for c0, cells in plist:
                key = mesh.boundary_signature(level, c0) if cache_by_signature else (c0,)
                bysig.setdefault(key, []).append(mesh.patch_dofs(level, cells, k))
            grp = []
            for key, idxs in bysig.items():
                idx = np.array(idxs)
                Aj = self.A[idx[0]][:, idx[0]].toarray()          # R_j A R_j^T
                grp.append((sla.lu_factor(Aj), idx))
            self.groups.append(grp)

    def local_solves(self, c, r):
        """Corrections delta_j = A_j^{-1} R_j r for every patch j of colour c,
        returned as (idx, delta) pairs."""
        out = []
        for lu, idx in self.groups[c]:
            rhs = r[idx].T                                         # (nloc, npatch)
            out.append((idx, sla.lu_solve(lu, rhs).T))
        return out

    def smooth(self, x, b, reverse=False):
        """One multiplicative step S(x, b) (Algorithm 1); returns a new x."""
        x = np.array(x, dtype=self.dtype)
        b = np.asarray(b, dtype=self.dtype)
        order = range(self.ncolours - 1, -1, -1) if reverse else range(self.ncolours)
        for c in order:
            r = b - self.A @ x                                     # pre-colour residual
            for idx, delta in self.local_solves(c, r):
                x[idx] += delta                                    # patches of c are disjoint
        return x

    def smooth_additive(self, x, b, omega=None):
        """One additive Schwarz step x + omega sum_j R_j^T A_j^{-1} R_j (b - A x)."""
        if omega is None:
            omega = 1.0 / self.ncolours
        x = np.array(x, dtype=self.dtype)
        r = np.asarray(b, dtype=self.dtype) - self.A @ x
        corr = np.zeros_like(x)
        for c in range(self.ncolours):
            for idx, delta in self.local_solves(c, r):
                corr[idx] += delta
        return x + self.dtype.type(omega) * corr
