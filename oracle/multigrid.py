"""Geometric multigrid V-cycle (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

PAPER.md:155-172: P_0^{-1} = A_0^{-1}; for l >= 1
  (1) pre-smoothing     x_l <- S_l(x_l, b_l)
  (2) coarse correction x_l <- x_l + I^up P_{l-1}^{-1} I^down (b_l - A_l x_l)
  (3) post-smoothing    x_l <- S_l(x_l, b_l)
with one pre- and one post-smoothing step, x_l = 0 on entry.
Coarse operators are re-discretised on each level (not Galerkin, reading A4);
A_0^{-1} is a dense LU solve (reading A10).  Mixed precision
(PAPER.md:465): the whole V-cycle in float32, input/output converted.
"""
import numpy as np
import scipy.linalg as sla

from . import assemble, mesh, transfer
from .smoother import PatchSmoother


class VCycle:
    def __init__(self, dim, k, n_levels, n0=None, h0=0.5, dtype=np.float64,
                 smoother="multiplicative", omega=None, post_reverse=True,
                 penalty_scale=1.0, operators=None, kernel="full", basis_kind=None,
                 boundary_penalty_scale=1.0):
        self.dim, self.k, self.n_levels = dim, k, n_levels
        self.dtype = np.dtype(dtype)
        self.levels = mesh.hierarchy(dim, n_levels, n0, h0)
        # the clamped kernel lives on the Hermite-type basis (the whole hierarchy)
        self.basis_kind = basis_kind or ("hermite" if kernel == "clamped" else "lagrange")
        if operators is None:
            operators = [assemble.assemble(lv, k, penalty_scale, kind=self.basis_kind,
                                           boundary_penalty_scale=boundary_penalty_scale) for lv in self.levels]
        self.A64 = operators
        self.A = [A.astype(self.dtype) for A in operators]
        self.P = [None] + [transfer.prolongation(self.levels[l - 1], self.levels[l], k, self.basis_kind).astype(self.dtype)
                           for l in range(1, n_levels)]
        self.S = [None] + [PatchSmoother(self.levels[l], k, operators[l], self.dtype, kernel=kernel,
                                         penalty_scale=penalty_scale)
                           for l in range(1, n_levels)]
        self.coarse_lu = sla.lu_factor(self.A[0].toarray())
        self.kind, self.omega, self.post_reverse = smoother, omega, post_reverse

    def _smooth(self, l, x, b, post):
        if self.kind == "additive":
            return self.S[l].smooth_additive(x, b, self.omega)
        return self.S[l].smooth(x, b, reverse=(post and self.post_reverse))

    def cycle(self, l, b):
        """P_l^{-1} b_l (recursive definition of)."""
        b = np.asarray(b, dtype=self.dtype)
        if l == 0:
            return sla.lu_solve(self.coarse_lu, b)
        x = np.zeros_like(b)
        x = self._smooth(l, x, b, post=False)
        r = b - self.A[l] @ x
        e = self.cycle(l - 1, self.P[l].T @ r)
        x = x + self.P[l] @ e
        return self._smooth(l, x, b, post=True)

    def __call__(self, r):
        """z = P_L^{-1} r on the finest level; converts to the V-cycle precision
        on entry and back to float64 on exit."""
        r = np.asarray(r)
        z = self.cycle(self.n_levels - 1, r.astype(self.dtype))
        return z.astype(np.float64)
