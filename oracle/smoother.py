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

Clamped kernel (NEXT-3, reading A19): the same update on the
Hermite-type basis (oracle/basis.hermite) with V_j = patch functions whose value
and normal derivative vanish on the mesh-interior patch faces ((2k-2)^d dofs);
the patch-only residual is then exact (pinned: A[V_j, outside] = 0).

Dirichlet kernel (reading A20): V_j = the
patch dofs whose node index is not on a patch-boundary face that is a
mesh-interior face (omitting "the functions associated to boundary
interpolation points"; (2k)^d dofs for an interior patch, domain-boundary
nodes kept, see interior_mask), domain of dependence = the patch cells only ("we use only the functions
on patch j"): r_j = R_j b - A[V_j, patch] x_patch (the coupling to cells
outside the patch is dropped -- the inconsistent residual of PAPER.md:225),
x_{V_j} += A[V_j, V_j]^{-1} r_j, colours as in Algorithm 1.  Both matrices are
extracted from the assembled A.
"""
import numpy as np
import scipy.linalg as sla

from . import mesh


def interior_mask(dim, k, signature=None, width=1):
    """Dirichlet-kernel subspace inside the patch-lexicographic ordering: True
    unless some direction's node index lies on a patch-boundary face that is a
    MESH-INTERIOR face (index 0 or 2k+1).  Nodes on the domain boundary stay
    in V_j (reading A20: there is no exterior trace to drop there, and the
    domain-boundary dofs of the DG space would otherwise never be smoothed).
    signature: mesh.boundary_signature of the patch (None: interior patch)."""
    npatch = 2 * (k + 1)
    sig = signature or ((False, False),) * dim
    m = np.ones(npatch ** dim, dtype=bool)
    for lex in range(npatch ** dim):
        rem = lex
        for a in range(dim):
            i = rem % npatch
            if (i < width and not sig[a][0]) or (i >= npatch - width and not sig[a][1]):
                m[lex] = False
            rem //= npatch
    return m


class PatchSmoother:
    def __init__(self, level, k, A, dtype=np.float64, cache_by_signature=True, kernel="full", penalty_scale=1.0):
        self.level, self.k, self.dtype = level, k, np.dtype(dtype)
        self.penalty_scale = penalty_scale
        self.A = A.astype(self.dtype)
        self.ncolours = 2 ** level.dim
        self.kernel = kernel
        # groups[c] = list of (lu, idx (npatch, nloc)) ; Dirichlet: (lu, idx_I, idx_P, A_IP)
        self.groups = []
        for c, plist in enumerate(mesh.coloured_patches(level)):
            bysig = {}
            for c0, cells in plist:
                key = mesh.boundary_signature(level, c0) if cache_by_signature else (c0,)
                bysig.setdefault(key, []).append(mesh.patch_dofs(level, cells, k))
            grp = []
            for key, idxs in bysig.items():
                idx = np.array(idxs)
                if kernel in ("dirichlet", "clamped"):
                    assert cache_by_signature
                    # clamped (Hermite-type basis): V_j drops value AND
                    # derivative functions at mesh-interior patch faces (width 2); for
                    # those test functions every outer face term vanishes, so the
                    # assembled rows are already the exact patch-local residual
                    mask = interior_mask(level.dim, k, key, 2 if kernel == "clamped" else 1)
                    iI = idx[:, mask]
                    APP = self.A[idx[0]][:, idx[0]].toarray()
                    if kernel == "dirichlet":
                        APP = APP - self._outer_face_terms(key).astype(self.dtype)
                    AIP = APP[mask, :]                            # patch operator, rows V_j
                    AII = AIP[:, mask]                            # = A[V_j, V_j] (checked by the pins)
                    grp.append((sla.lu_factor(AII), iI, idx, AIP))
                else:
                    Aj = self.A[idx[0]][:, idx[0]].toarray()      # R_j A R_j^T
                    grp.append((sla.lu_factor(Aj), idx))
            self.groups.append(grp)

    def _outer_face_terms(self, sig):
        """Contribution of the patch's MESH-INTERIOR outer faces to A[patch, patch]
        (the patch cells' own side of those faces; patch-lexicographic order).
        The Dirichlet kernel's residual drops these terms entirely -- for test
        functions in V_j only the consistency term -[[u]].{grad v} survives there,
        and "the last face term ... does not vanish" is the
        inconsistency the paper accepts (reading A20)."""
        from .assemble import Reference
        from . import basis
        d, k, h = self.level.dim, self.k, self.level.h
        nc, npatch = k + 1, 2 * (k + 1)
        ref = Reference(d, k)
        B = None
        C = np.zeros((npatch ** d, npatch ** d))
        # lex position of (cell q, local node l)
        pos = np.empty((2 ** d, nc ** d), dtype=np.int64)
        for lex in range(npatch ** d):
            rem, q, loc = lex, 0, 0
            for a in range(d):
                pa = rem % npatch
                rem //= npatch
                q |= (pa // nc) << a
                loc += (pa % nc) * nc ** a
            pos[q, loc] = lex
        gamma = basis.penalty(k, h, h, self.penalty_scale)
        for a in range(d):
            blocks = ref.interior_face_blocks(a, h, gamma)
            for side in (0, 1):
                if sig[a][side]:
                    continue                     # domain boundary: Nitsche terms are exact
                Bs = blocks[1][1] if side == 0 else blocks[0][0]   # patch cell is K+ (low) / K- (high)
                for q in range(2 ** d):
                    if ((q >> a) & 1) != side:
                        continue
                    C[np.ix_(pos[q], pos[q])] += Bs
        return C

    def colour_step_dirichlet(self, c, x, b):
        """One colour of Algorithm 1 with the Dirichlet kernel; returns a new x."""
        x = np.array(x, dtype=self.dtype)
        upd = []
        for (lu, iI, _, _), (_, r) in zip(self.groups[c], self.local_residuals_dirichlet(c, x, b)):
            upd.append((iI, sla.lu_solve(lu, r.T).T))
        for iI, delta in upd:                                      # disjoint patches of colour c
            x[iI] += delta
        return x

    def local_residuals_dirichlet(self, c, x, b):
        """[(idx_I, r_j)] of colour c: r_j = b[V_j] - A[V_j, patch] x[patch]."""
        return [(iI, b[iI] - x[iP] @ AIP.T) for _, iI, iP, AIP in self.groups[c]]

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
        if self.kernel in ("dirichlet", "clamped"):
            for c in order:
                x = self.colour_step_dirichlet(c, x, b)
            return x
        for c in order:
            r = b - self.A @ x                                     # pre-colour residual
            for idx, delta in self.local_solves(c, r):
                x[idx] += delta                                    # patches of c are disjoint
        return x

    def smooth_additive(self, x, b, omega=None):
        """One additive Schwarz step x + omega sum_j R_j^T A_j^{-1} R_j (b - A x)."""
        if self.kernel != "full":
            raise NotImplementedError("additive smoothing is defined for the full kernel")
        if omega is None:
            omega = 1.0 / self.ncolours
        x = np.array(x, dtype=self.dtype)
        r = np.asarray(b, dtype=self.dtype) - self.A @ x
        corr = np.zeros_like(x)
        for c in range(self.ncolours):
            for idx, delta in self.local_solves(c, r):
                corr[idx] += delta
        return x + self.dtype.type(omega) * corr
