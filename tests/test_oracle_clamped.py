"""Pins of the oracle's Hermite-type basis and clamped-kernel smoother
(Fig. 3 right; reading A19):

* the SPEC.md:142 worked example (k = 3: psi_0 = 1 - 3x^2 + 2x^3), exact
  reproduction of degree-k polynomials, one unit endpoint functional per
  constrained function;
* the Hermite-basis SIPG matrix and embedding equal the Lagrange ones under the
  cell-wise change of basis T (two independent assembly paths);
* the clamped residual is local: A[V_j, outside patch j] = 0 (PAPER.md:229
  "the residual does not couple to neighboring cells");
* local space (2k-2)^d (4^3 for Q3);
* the paper's Table 2 clamped column.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import read_golden
from oracle import assemble, basis, krylov, mesh, multigrid, transfer
from oracle.smoother import PatchSmoother, interior_mask


def test_worked_example_k3():
    x = np.linspace(0, 1, 11)
    V, D = basis.hermite(3, x)
    assert np.abs(V[:, 0] - (1 - 3 * x ** 2 + 2 * x ** 3)).max() <= 1e-13
    assert np.abs(D[:, 0] - (-6 * x + 6 * x ** 2)).max() <= 1e-12


@pytest.mark.parametrize("k", [3, 4, 5, 7])
def test_reproduces_polynomials_and_endpoint_functionals(k):
    rng = np.random.default_rng(k)
    c = rng.uniform(-1, 1, k + 1)
    u = np.polynomial.Polynomial(c)
    du = u.deriv()
    eta = basis.hermite_points(k)
    coef = np.concatenate([[u(0.0), du(0.0)], u(eta), [-du(1.0), u(1.0)]])
    x = rng.uniform(0, 1, 17)
    V, D = basis.hermite(k, x)
    assert np.abs(V @ coef - u(x)).max() <= 1e-11
    assert np.abs(D @ coef - du(x)).max() <= 1e-10
    V01, D01 = basis.hermite(k, [0.0, 1.0])
    E = np.vstack([V01[0], D01[0], D01[1], V01[1]])          # the 4 endpoint functionals
    assert np.abs(np.abs(E) - np.eye(k + 1)[[0, 1, k - 1, k]]).max() <= 1e-12
    # reflection x -> 1 - x maps psi_j to psi_{k-j}
    Vr, _ = basis.hermite(k, 1.0 - x)
    assert np.abs(Vr - V[:, ::-1]).max() <= 1e-12


def _T(dim, k, ncells):
    """Cell-wise change of basis, Lagrange nodal values of the Hermite functions."""
    T1 = basis.hermite(k, basis.gll_nodes(k + 1))[0]          # T1[i, j] = psi_j(xi_i)
    Tc = np.ones((1, 1))
    for _ in range(dim):
        Tc = np.kron(T1, Tc)
    return sp.kron(sp.identity(ncells, format="csr"), sp.csr_matrix(Tc), format="csr")


@pytest.mark.parametrize("dim,k", [(2, 3), (2, 5), (3, 3)])
def test_change_of_basis(dim, k):
    lv = mesh.Level(dim, [4] * dim, 0.25)
    AL = assemble.assemble(lv, k)
    AH = assemble.assemble(lv, k, kind="hermite")
    T = _T(dim, k, lv.ncells)
    ref = (T.T @ AL @ T).toarray()
    assert np.abs(AH.toarray() - ref).max() <= 1e-10 * np.abs(ref).max()
    bL, bH = assemble.rhs(lv, k), assemble.rhs(lv, k, kind="hermite")
    assert np.abs(bH - T.T @ bL).max() <= 1e-13
    cl = mesh.Level(dim, [2] * dim, 0.5)
    PL = transfer.prolongation(cl, lv, k)
    PH = transfer.prolongation(cl, lv, k, "hermite")
    Tc = _T(dim, k, cl.ncells)
    Tf = _T(dim, k, lv.ncells)
    assert np.abs((Tf @ PH - PL @ Tc).toarray()).max() <= 1e-12


@pytest.mark.parametrize("dim,k,n", [(2, 3, 4), (2, 4, 6), (3, 3, 4)])
def test_clamped_residual_is_patch_local(dim, k, n):
    lv = mesh.Level(dim, [n] * dim, 1.0 / n)
    A = assemble.assemble(lv, k, kind="hermite")
    checked = 0
    for plist in mesh.coloured_patches(lv):
        for c0, cells in plist:
            P = mesh.patch_dofs(lv, cells, k)
            I = P[interior_mask(dim, k, mesh.boundary_signature(lv, c0), 2)]
            rows = A[I]
            outside = np.setdiff1d(np.unique(rows.indices), P)
            assert len(outside) == 0 or np.abs(rows[:, outside].toarray()).max() <= 1e-12 * abs(A).max()
            checked += 1
    assert checked == (n - 1) ** dim
    assert interior_mask(3, 3, None, 2).sum() == 4 ** 3


def test_lagrange_is_not_patch_local():
    """Contrast: with the Lagrange basis the same rows do couple outside (the
    reason the Dirichlet kernel's residual is inconsistent)."""
    lv = mesh.Level(2, [4, 4], 0.25)
    A = assemble.assemble(lv, 3)
    c0, cells = mesh.coloured_patches(lv)[0][0]
    P = mesh.patch_dofs(lv, cells, 3)
    I = P[interior_mask(2, 3, mesh.boundary_signature(lv, c0), 1)]
    outside = np.setdiff1d(np.unique(A[I].indices), P)
    assert len(outside) > 0


def _table2c():
    t = {}
    for r in read_golden("table2_dirichlet_clamped.txt"):
        for j, v in enumerate(r[6:11]):
            if v != "---":
                t[(int(r[0]), 3 + j)] = float(v)
    return t


@pytest.mark.parametrize("k,tol", [(3, 1.2), (4, 0.6), (5, 0.5)])
def test_table2_clamped_column(k, tol):
    """Table 2, clamped kernel, L = 2, GMRES to 1e-8, f == 1,
    post-smoothing in forward colour order (reading A7 for the paper's GMRES
    runs); tolerance +-0.5 relative to the paper's scale (18.6 for Q3)."""
    V = multigrid.VCycle(3, k, 2, kernel="clamped", post_reverse=False)
    _, h, c = krylov.gmres(V.A64[-1], assemble.rhs(V.levels[-1], k, kind="hermite"), V)
    assert c
    assert abs(krylov.nu(h) - _table2c()[(2, k)]) <= tol, krylov.nu(h)
