"""Pins of the oracle's Dirichlet-kernel smoother (SURVEY.md
NEXT-1, reading A20) against what the paper and the mathematics fix:

* the local space has (2k)^d dofs on an interior patch (6^3 for Q3);
* its local matrix A[V_j, V_j] is the Kronecker sum of the 1D interior blocks
  (the outer-face terms vanish on V_j), identical for every interior patch;
* the patch-only residual equals the true residual for globally continuous
  functions (the dropped consistency term -[[u]].{grad v} vanishes) and differs
  for discontinuous ones (the inconsistency PAPER.md:225 describes);
* the V-cycle is h-independent and reproduces the Dirichlet column of the
  paper's Table 2.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import read_golden
from oracle import assemble, krylov, mesh, multigrid
from oracle.assemble import Reference
from oracle.smoother import PatchSmoother, interior_mask


def test_subspace_sizes():
    for k in (1, 3, 4):
        assert interior_mask(3, k).sum() == (2 * k) ** 3
        assert interior_mask(2, k).sum() == (2 * k) ** 2
    assert interior_mask(3, 3).sum() == 6 ** 3
    sig = ((True, False), (False, False))                        # low x face on the domain boundary
    assert interior_mask(2, 3, sig).sum() == (2 * 3 + 1) * (2 * 3)


def _kron_interior(k, h, dim):
    """Kronecker sum of the 1D interior blocks of a 2-cell patch inside a 4-cell line."""
    lv = mesh.Level(1, [4], h)
    A1 = assemble.assemble(lv, k).toarray()
    nc = k + 1
    P = np.arange(nc, 3 * nc)                                    # cells 1, 2
    I1 = P[1:-1]
    L1 = A1[np.ix_(I1, I1)]
    _, Mc = Reference(1, k).cell_matrices(h)
    M1 = np.kron(np.eye(2), Mc)[1:-1, 1:-1]
    if dim == 2:
        return np.kron(M1, L1) + np.kron(L1, M1)
    return (np.kron(M1, np.kron(M1, L1)) + np.kron(M1, np.kron(L1, M1)) + np.kron(L1, np.kron(M1, M1)))


@pytest.mark.parametrize("dim,k,n", [(2, 2, 6), (2, 3, 4), (3, 2, 4)])
def test_local_matrix_is_kronecker_sum(dim, k, n):
    lv = mesh.Level(dim, [n] * dim, 1.0 / n)
    A = assemble.assemble(lv, k)
    S = PatchSmoother(lv, k, A, kernel="dirichlet")
    ref = _kron_interior(k, lv.h, dim)
    seen = 0
    for c, plist in enumerate(mesh.coloured_patches(lv)):
        for c0, cells in plist:
            if mesh.boundary_signature(lv, c0) != ((False, False),) * dim:
                continue
            idx = mesh.patch_dofs(lv, cells, k)[interior_mask(dim, k)]
            AII = A[idx][:, idx].toarray()
            assert np.abs(AII - ref).max() <= 1e-12 * np.abs(ref).max()
            seen += 1
    assert seen > 0
    # the smoother's cached local matrices are these blocks
    for grp in S.groups:
        for lu, iI, iP, AIP in grp:
            assert AIP.shape == (iI.shape[1], iP.shape[1])


def _continuous_interpolant(lv, k):
    """DG interpolant of a globally continuous polynomial of degree <= k: equal
    traces from both sides on every face (GLL nodes on the faces)."""
    X = assemble.cell_nodes(lv, k)                               # (ndofs, dim)
    u = np.ones(X.shape[0])
    for i in range(lv.dim):
        u *= X[:, i] * (1.0 - X[:, i]) + 0.3 * X[:, i]
    return u


@pytest.mark.parametrize("dim,k,n", [(2, 3, 4), (3, 2, 4)])
def test_patch_residual_consistency(dim, k, n):
    lv = mesh.Level(dim, [n] * dim, 1.0 / n)
    A = assemble.assemble(lv, k)
    S = PatchSmoother(lv, k, A, kernel="dirichlet")
    b = np.zeros(A.shape[0])
    u = _continuous_interpolant(lv, k)
    Au = A @ u
    rng = np.random.default_rng(3)
    w = rng.uniform(-1, 1, A.shape[0])
    Aw = A @ w
    worst_c, worst_d = 0.0, 0.0
    for c in range(S.ncolours):
        for (iI, r), (_, rw) in zip(S.local_residuals_dirichlet(c, u, b), S.local_residuals_dirichlet(c, w, b)):
            worst_c = max(worst_c, np.abs(-r - Au[iI]).max())     # r = b - A~ u with b = 0
            worst_d = max(worst_d, np.abs(-rw - Aw[iI]).max())
    assert worst_c <= 1e-10 * np.abs(Au).max()                   # consistent on continuous functions
    assert worst_d >= 1e-3 * np.abs(Aw).max()                    # inconsistent in general


def _table2():
    t = {}
    for r in read_golden("table2_dirichlet_clamped.txt"):
        for j, v in enumerate(r[1:6]):
            if v != "---":
                t[(int(r[0]), 3 + j)] = float(v)
    return t


def test_vcycle_h_independent_2d():
    nus = []
    for L in (4, 5):
        V = multigrid.VCycle(2, 3, L, kernel="dirichlet")
        A = V.A64[-1]
        _, h, c = krylov.gmres(A, assemble.rhs(V.levels[-1], 3), V)
        assert c
        nus.append(krylov.nu(h))
    assert abs(nus[0] - nus[1]) <= 0.5, nus


@pytest.mark.parametrize("L,k", [(2, 3), (2, 4), (3, 3)])
def test_table2_dirichlet_column(L, k):
    """Table 2, Dirichlet kernel, GMRES to 1e-8, f == 1,
    readings A5 (row L = 2^L cells) and A7 (reverse post-smoothing); tolerance
    +-0.5."""
    V = multigrid.VCycle(3, k, L, kernel="dirichlet")
    A = V.A64[-1]
    _, h, c = krylov.gmres(A, assemble.rhs(V.levels[-1], k), V)
    assert c
    assert abs(krylov.nu(h) - _table2()[(L, k)]) <= 0.5, krylov.nu(h)
