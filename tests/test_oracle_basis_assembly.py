"""Pins of the oracle's 1D basis and SIPG assembly (DESIGN.md pins P1-P5, P9).

None of these re-types the oracle's formulas: they check printed worked values
(SPEC.md / hand derivations in tests/golden), closed forms (Kronecker
separability, polynomial exactness of a consistent method), invariants
(symmetry, SPD) and the discretisation error rate k+1.
"""
import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse.linalg as spla

from conftest import read_golden
from oracle import assemble, basis, mesh


def _spec(key):
    for row in read_golden("spec_worked_examples.txt"):
        if row[0] == key:
            vals = []
            for t in row[1:]:
                try:
                    vals.append(float(t))
                except ValueError:
                    break
            return np.array(vals)
    raise KeyError(key)


def test_gll_worked_values():
    assert np.allclose(basis.gll_nodes(2), [0, 1], atol=1e-15)
    assert np.allclose(basis.gll_nodes(3), [0, 0.5, 1], atol=1e-15)
    assert np.allclose(basis.gll_nodes(4), _spec("gll4"), atol=1e-15)
    for n in range(2, 9):
        x = basis.gll_nodes(n)
        assert np.allclose(x + x[::-1], 1.0, atol=1e-14)      # symmetric about 1/2
    with pytest.raises(ValueError):
        basis.gll_nodes(1)


def test_gauss_worked_values_and_exactness():
    x, w = basis.gauss(1)
    assert np.allclose(x, [0.5]) and np.allclose(w, [1.0])
    x, w = basis.gauss(2)
    assert np.allclose(x, _spec("gauss2_points"), atol=1e-15)
    assert np.allclose(w, _spec("gauss2_weights"), atol=1e-15)
    for n in range(1, 9):
        x, w = basis.gauss(n)
        for p in range(2 * n):
            assert abs(np.sum(w * x ** p) - 1.0 / (p + 1)) < 1e-14


def test_lagrange_delta_unity_and_derivative():
    rng = np.random.default_rng(1)
    for k in range(1, 8):
        nodes = basis.gll_nodes(k + 1)
        V, _ = basis.lagrange(nodes, nodes)
        assert np.allclose(V, np.eye(k + 1), atol=1e-13)
        xs = rng.uniform(0, 1, 30)
        V, D = basis.lagrange(nodes, xs)
        assert np.allclose(V.sum(axis=1), 1.0, atol=1e-12)    # partition of unity
        assert np.allclose(D.sum(axis=1), 0.0, atol=1e-9)
        # derivative vs central difference of the values (independent check)
        eps = 1e-6
        Vp, _ = basis.lagrange(nodes, xs + eps)
        Vm, _ = basis.lagrange(nodes, xs - eps)
        assert np.allclose(D, (Vp - Vm) / (2 * eps), atol=1e-5 * max(1, np.abs(D).max()))


def test_penalty_and_mass_worked_values():
    assert basis.penalty(2, 0.25, 0.25) == _spec("penalty_k2_h0.25")[0]
    ref = assemble.Reference(1, 1)
    _, M = ref.cell_matrices(1.0)
    assert np.allclose(M.ravel(), _spec("mass_k1_h1"), atol=1e-15)
    for k in range(1, 8):
        ref = assemble.Reference(1, k)
        for h in (1.0, 0.125):
            _, M = ref.cell_matrices(h)
            assert abs(M.sum() - h) < 1e-13                     # partition of unity


def _golden_1d():
    rows = read_golden("sipg_1d_k1.txt")
    out, cur = {}, None
    for r in rows:
        if len(r) == 1:
            cur = r[0]
            out[cur] = []
        else:
            out[cur].append([float(v) for v in r])
    return {k: np.array(v) for k, v in out.items()}


def test_sipg_1d_hand_derived():
    g = _golden_1d()
    A = assemble.assemble(mesh.Level(1, [1], 1.0), 1).toarray()
    assert np.allclose(A, g["one_cell_h1"], atol=1e-14)
    A = assemble.assemble(mesh.Level(1, [2], 0.5), 1).toarray()
    assert np.allclose(A, g["two_cells_h0.5"], atol=1e-13)


def _cellwise_to_global_lex(n, k):
    """Permutation p with A_cellwise = A_globallex[p][:, p] for a Cartesian box."""
    d = len(n)
    nc = k + 1
    perm = []
    cells = np.ndindex(*reversed(n))
    for cz in cells:
        c = tuple(reversed(cz))
        for lz in np.ndindex(*([nc] * d)):
            l = tuple(reversed(lz))
            g, stride = 0, 1
            for i in range(d):
                g += (c[i] * nc + l[i]) * stride
                stride *= n[i] * nc
            perm.append(g)
    return np.array(perm)


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2)])
def test_kronecker_separability(dim, k):
    """P2: A = sum_a M x..x L_a^glob x..x M (PAPER.md:118-126 generalised to the
    global matrix) with L^glob, M^glob the *1D* assembled SIPG and mass
    matrices -- the d-dim quadrature assembly must agree."""
    n = (4, 3, 2)[:dim]
    h = 0.25
    A = assemble.assemble(mesh.Level(dim, n, h), k).toarray()
    L1 = [assemble.assemble(mesh.Level(1, [n[i]], h), k).toarray() for i in range(dim)]
    _, M = assemble.Reference(1, k).cell_matrices(h)
    Mg = [np.kron(np.eye(n[i]), M) for i in range(dim)]
    Ak = 0
    for a in range(dim):
        t = np.ones((1, 1))
        for i in range(dim):
            t = np.kron(L1[i] if i == a else Mg[i], t)     # x fastest
        Ak = Ak + t
    p = _cellwise_to_global_lex(n, k)
    Ak = Ak[np.ix_(p, p)]
    assert np.abs(A - Ak).max() <= 1e-13 * np.abs(A).max()


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 4), (3, 2)])
def test_symmetric_positive_definite(dim, k):
    lv = mesh.hierarchy(dim, 2)[-1]
    A = assemble.assemble(lv, k).toarray()
    assert np.abs(A - A.T).max() <= 1e-14 * np.abs(A).max()
    sla.cholesky(A)                       # raises if not SPD


@pytest.mark.parametrize("dim,k", [(2, 2), (2, 3), (3, 2)])
def test_polynomial_exactness(dim, k):
    """P4: SIPG is consistent, so for u = prod x_i(1-x_i) in Q_k (k >= 2, u = 0
    on the boundary) the discrete solution is I_h u exactly: A I_h u = b(-lap u)."""
    lv = mesh.hierarchy(dim, 2)[-1]

    def u(X):
        return np.prod(X * (1 - X), axis=1)

    def f(X):
        s = 0.0
        for a in range(dim):
            others = np.prod([X[:, i] * (1 - X[:, i]) for i in range(dim) if i != a], axis=0)
            s = s + 2.0 * others
        return s

    A = assemble.assemble(lv, k)
    ui = assemble.interpolate(lv, k, u)
    b = assemble.rhs(lv, k, f)
    assert np.linalg.norm(A @ ui - b) <= 1e-12 * np.linalg.norm(b)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_l2_convergence_rate(k):
    """P5: u = sin(pi x) sin(pi y), f = 2 pi^2 u: L2 error O(h^{k+1})."""
    def u(X):
        return np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1])

    def f(X):
        return 2 * np.pi ** 2 * u(X)

    errs = []
    for lv in mesh.hierarchy(2, 4)[1:]:
        A = assemble.assemble(lv, k).tocsc()
        uh = spla.spsolve(A, assemble.rhs(lv, k, f))
        errs.append(assemble.l2_error(lv, k, uh, u))
    rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert rates[-1] >= k + 0.8, (errs, rates)


def test_patch_and_colour_counts():
    """P9: patches = prod(n_i - 1); colour sizes;
    C1 8x8: 49 patches in colours 16/12/12/9; every cell in at most one patch
    per colour."""
    assert len(mesh.patches(mesh.Level(2, [4, 4], 0.25))) == int(_spec("patches_2d_l1")[0])
    assert len(mesh.patches(mesh.Level(3, [8, 8, 8], 0.125))) == int(_spec("patches_3d_l2")[0])
    cl = mesh.coloured_patches(mesh.Level(2, [4, 4], 0.25))
    assert sorted([len(c) for c in cl], reverse=True) == list(_spec("colour_sizes_2d_4x4").astype(int))
    assert [len(c) for c in cl] == [4, 2, 2, 1]
    lv = mesh.Level(2, [8, 8], 0.125)
    cl = mesh.coloured_patches(lv)
    assert [len(c) for c in cl] == [16, 12, 12, 9]
    for cls in mesh.coloured_patches(mesh.Level(3, [4, 6, 4], 0.25)):
        cells = [c for _, cs in cls for c in cs]
        assert len(cells) == len(set(cells))
    # full-kernel local space: 2(k+1) per direction, 8 at k=3
    lv = mesh.Level(3, [4, 4, 4], 0.25)
    c0, cells = mesh.patches(lv)[0]
    assert len(mesh.patch_dofs(lv, cells, 3)) == int(_spec("local_space_full_k3")[0]) ** 3


def test_footnote_cell_order():
    """PAPER.md:384 footnote: first the cell whose top-right vertex is the shared
    vertex (bottom-left cell), then bottom-right, top-left, top-right."""
    lv = mesh.Level(2, [4, 4], 0.25)
    c0, cells = mesh.patches(lv)[5]
    assert c0 == (2, 1)
    assert cells == [lv.cell_lin((2, 1)), lv.cell_lin((3, 1)), lv.cell_lin((2, 2)), lv.cell_lin((3, 2))]
