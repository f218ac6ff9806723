"""Pins of the oracle's transfers, smoother, V-cycle and Krylov solvers
(DESIGN.md pins P6, P8, P10-P15)."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from conftest import read_golden
from oracle import assemble, basis, krylov, mesh, multigrid, smoother, transfer
from synth_inputs import uniform


# ---------------------------------------------------------------- transfers
@pytest.mark.parametrize("dim,k", [(2, 1), (2, 3), (3, 2)])
def test_prolongation_is_embedding(dim, k):
    """P8: the prolongated function equals the coarse function at random points
    (SPEC.md:386), evaluated with the basis directly."""
    levels = mesh.hierarchy(dim, 2)
    P = transfer.prolongation(levels[0], levels[1], k)
    xc = uniform(P.shape[1], seed=3)
    xf = P @ xc
    nodes = basis.gll_nodes(k + 1)
    rng = np.random.default_rng(4)

    def evaluate(level, vec, X):
        out = np.zeros(len(X))
        for p, pt in enumerate(X):
            c = tuple(min(int(pt[i] / level.h), level.n[i] - 1) for i in range(dim))
            loc = [pt[i] / level.h - c[i] for i in range(dim)]
            vals = [basis.lagrange(nodes, [loc[i]])[0][0] for i in range(dim)]
            base = level.cell_lin(c) * (k + 1) ** dim
            for l in range((k + 1) ** dim):
                w = 1.0
                for i in range(dim):
                    w *= vals[i][(l // (k + 1) ** i) % (k + 1)]
                out[p] += w * vec[base + l]
        return out

    X = rng.uniform(0, 1, (50, dim))
    assert np.allclose(evaluate(levels[0], xc, X), evaluate(levels[1], xf, X), atol=1e-12)
    assert np.allclose(P @ np.ones(P.shape[1]), 1.0, atol=1e-14)


@pytest.mark.parametrize("dim,k", [(2, 1), (2, 2), (3, 1)])
def test_coarse_operator_identity(dim, k):
    """P8 / reading A4: with re-discretised coarse operators,
    P^T A_f P = A_c + gamma_c J_c, i.e. the coarse SIPG matrix assembled with a
    doubled penalty (the fine penalty is 2k(k+1)/(h/2) on coarse faces; fine
    faces inside coarse cells carry no jump).  SPEC.md:408's Galerkin identity
    P^T A_f P = A_c is false."""
    levels = mesh.hierarchy(dim, 2)
    P = transfer.prolongation(levels[0], levels[1], k)
    Af = assemble.assemble(levels[1], k)
    G = (P.T @ Af @ P).toarray()
    Ac2 = assemble.assemble(levels[0], k, penalty_scale=2.0).toarray()
    Ac = assemble.assemble(levels[0], k).toarray()
    assert np.abs(G - Ac2).max() <= 1e-12 * np.abs(G).max()
    assert np.abs(G - Ac).max() > 0.1 * np.abs(G).max()


# ---------------------------------------------------------------- smoother
def _setup(dim, k, nl):
    lv = mesh.hierarchy(dim, nl)[-1]
    A = assemble.assemble(lv, k)
    return lv, A


@pytest.mark.parametrize("dim,k", [(2, 2), (3, 1)])
def test_signature_cache_is_exact(dim, k):
    lv, A = _setup(dim, k, 3 if dim == 2 else 2)
    S1 = smoother.PatchSmoother(lv, k, A, cache_by_signature=True)
    S2 = smoother.PatchSmoother(lv, k, A, cache_by_signature=False)
    x = uniform(A.shape[0], seed=1)
    b = uniform(A.shape[0], seed=2)
    assert np.abs(S1.smooth(x, b) - S2.smooth(x, b)).max() <= 1e-13 * np.abs(x).max()


@pytest.mark.parametrize("dim,k", [(2, 3), (3, 2)])
def test_smoother_fixed_point_and_energy_decrease(dim, k):
    """P10: x* = A^{-1} b is a fixed point; each colour step
    decreases the A-norm error (SPEC.md:334, PAPER.md:191-197 exact residual)."""
    lv, A = _setup(dim, k, 3 if dim == 2 else 2)
    b = assemble.rhs(lv, k)
    xs = spla.spsolve(A.tocsc(), b)
    S = smoother.PatchSmoother(lv, k, A)
    assert np.linalg.norm(S.smooth(xs, b) - xs) <= 1e-10 * np.linalg.norm(xs)
    x = uniform(A.shape[0], seed=5)

    def en(v):
        e = v - xs
        return e @ (A @ e)

    e_prev = en(x)
    for c in range(S.ncolours):
        r = b - A @ x
        for idx, delta in S.local_solves(c, r):
            x[idx] += delta
        e = en(x)
        assert e < e_prev
        e_prev = e


def test_smoother_local_solve_is_exact_patch_inverse():
    """Each correction solves the extracted patch system A_j delta_j = R_j r
    exactly (checked by re-multiplying with the patch block of A)."""
    lv, A = _setup(2, 2, 3)
    b = uniform(A.shape[0], seed=8)
    x = uniform(A.shape[0], seed=9)
    S = smoother.PatchSmoother(lv, 2, A)
    Ad = A.toarray()
    for c in range(S.ncolours):
        r = b - A @ x
        for idx, delta in S.local_solves(c, r):
            for j in range(idx.shape[0]):
                Aj = Ad[np.ix_(idx[j], idx[j])]
                assert np.abs(Aj @ delta[j] - r[idx[j]]).max() <= 1e-12 * np.abs(r).max()


def test_additive_smoother_reduces_energy():
    lv, A = _setup(2, 2, 3)
    b = assemble.rhs(lv, 2)
    xs = spla.spsolve(A.tocsc(), b)
    S = smoother.PatchSmoother(lv, 2, A)
    x = uniform(A.shape[0], seed=6)
    e0 = (x - xs) @ (A @ (x - xs))
    x1 = S.smooth_additive(x, b)
    e1 = (x1 - xs) @ (A @ (x1 - xs))
    assert e1 < e0


# ---------------------------------------------------------------- V-cycle
def test_single_level_vcycle_is_coarse_inverse():
    V = multigrid.VCycle(2, 3, 1)
    b = uniform(V.A64[0].shape[0], seed=7)
    assert np.linalg.norm(V.A64[0] @ V(b) - b) <= 1e-12 * np.linalg.norm(b)


@pytest.mark.parametrize("dim,k,nl,kind", [(2, 2, 3, "multiplicative"), (2, 3, 3, "additive"),
                                           (3, 1, 3, "multiplicative")])
def test_vcycle_linear_symmetric_convergent(dim, k, nl, kind):
    """P11/P12: V is linear, symmetric (forward pre / reverse post smoothing),
    positive, and rho(I - V A) < 1 (power iteration)."""
    V = multigrid.VCycle(dim, k, nl, smoother=kind)
    A = V.A64[-1]
    n = A.shape[0]
    b1, b2 = uniform(n, seed=11), uniform(n, seed=12)
    v1, v2 = V(b1), V(b2)
    assert np.linalg.norm(V(2.0 * b1 - 3.0 * b2) - (2.0 * v1 - 3.0 * v2)) <= 1e-12 * np.linalg.norm(v1)
    assert abs(v1 @ b2 - b1 @ v2) <= 1e-12 * abs(v1 @ b2)
    assert v1 @ b1 > 0
    if kind == "multiplicative":
        e = uniform(n, seed=13)
        for _ in range(12):
            e = e - V(A @ e)
            rho = np.linalg.norm(e)
            e /= rho
        assert rho < 1.0
    else:
        # additive with omega = 1/2^d: the non-Galerkin coarse correction
        # over-corrects (P^T A_f P >= A_c, test_coarse_operator_identity), so the
        # stationary iteration need not contract; V is SPD and CG converges.
        _, h, c = krylov.pcg(A, b1, V)
        assert c and len(h) - 1 <= 30


def test_mixed_vcycle_close_to_double():
    """P15: fp32 V-cycle vs fp64 V-cycle <= 1e-5 relative."""
    V = multigrid.VCycle(2, 3, 4)
    Vm = multigrid.VCycle(2, 3, 4, dtype=np.float32, operators=V.A64)
    b = uniform(V.A64[-1].shape[0], seed=14)
    z, zm = V(b), Vm(b)
    assert np.linalg.norm(z - zm) <= 1e-5 * np.linalg.norm(z)


# ---------------------------------------------------------------- Krylov
def test_nu_worked_values():
    """P14: SPEC.md:461-462."""
    rows = {r[0]: float(r[1]) for r in read_golden("spec_worked_examples.txt") if r[0].startswith("nu_")}
    assert abs(krylov.nu([1.0, 0.1, 1e-3, 1e-5, 1e-8]) - rows["nu_n4_ratio1e-8"]) < 1e-12
    assert abs(krylov.nu([1.0, 1e-2, 1e-5, 1e-9]) - rows["nu_n3_ratio1e-9"]) < 1e-12


def test_krylov_on_dense_spd():
    rng = np.random.default_rng(0)
    Q = rng.standard_normal((50, 50))
    A = Q @ Q.T + 50 * np.eye(50)
    b = rng.standard_normal(50)
    xs = np.linalg.solve(A, b)
    I = np.eye(50)
    for solve in (krylov.pcg, krylov.gmres):
        x, h, c = solve(A, b, I, rtol=1e-12)
        assert c and np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs)
        x, h, c = solve(I, b, I)
        assert c and len(h) == 2
        x, h, c = solve(A, b, np.linalg.inv(A))
        assert c and len(h) == 2
    x, h, c = krylov.pcg(A, np.zeros(50), I)
    assert c and len(h) == 1


@pytest.mark.parametrize("dim,k,nl", [(2, 2, 3), (3, 2, 2)])
def test_pcg_solution_matches_direct(dim, k, nl):
    """P6: GMG-PCG at rtol 1e-13 equals a sparse direct solve."""
    V = multigrid.VCycle(dim, k, nl)
    A = V.A64[-1]
    b = assemble.rhs(V.levels[-1], k)
    x, h, c = krylov.pcg(A, b, V, rtol=1e-13)
    xs = spla.spsolve(A.tocsc(), b)
    assert c and np.linalg.norm(x - xs) <= 1e-11 * np.linalg.norm(xs)
    # residual norms of CG are the true residuals
    assert np.linalg.norm(b - A @ x) <= 1.01e-13 * h[0]


def test_iterations_h_independent_2d():
    """P13: GMG-CG iteration counts are flat in h."""
    its = []
    for nl in (3, 4, 5, 6):
        V = multigrid.VCycle(2, 2, nl)
        A = V.A64[-1]
        _, h, c = krylov.pcg(A, assemble.rhs(V.levels[-1], 2), V)
        assert c
        its.append(len(h) - 1)
    assert max(its) - min(its) <= 1, its


def _table1():
    t = {}
    for r in read_golden("table1_full_kernel.txt"):
        L = int(r[0])
        for j, v in enumerate(r[1:]):
            if v != "---":
                t[(L, 3 + j)] = float(v)
    return t


# Table 1 under reading A22: the paper's nu is the one a left-preconditioned
# GMRES reports (preconditioned residual norm), the symmetric V-cycle (A7) and the paper's
# penalty (A2), row L = 2^L cells per direction (A5).  The block is every cell the oracle
# reaches in about a minute: L = 2 for Q3..Q7, L = 3 for Q3..Q5, L = 4 for Q3 -- no cell of
# it is left out.  Oracle values (tools/oracle_table1.py, fp64):
#   L=2: 3.10 2.97 2.98 2.98 2.99   (paper 3.4 2.9 2.8 2.6 2.4)
#   L=3: 3.65 3.39 3.47             (paper 3.7 3.2 2.8)
#   L=4: 3.55                       (paper 3.6)
# Expected deviation per cell: +-0.5 for k <= 4.  For k >= 5 the paper's nu
# falls with the degree and ours stays flat near 3.0-3.5 (also on the GPU up to L = 6,
# profiles/r02_table1_study.md): no reading tried (penalty scale, one-sided boundary
# penalty, level index, post-smoothing order, left/right preconditioning) reproduces that
# degree trend, so those cells carry the stated band [-0.5, +0.8] (A22).
TABLE1_BLOCK = [(2, 3), (2, 4), (2, 5), (2, 6), (2, 7), (3, 3), (3, 4), (3, 5), (4, 3)]
_NU_CACHE = {}


def _nu_left(L, k):
    if (L, k) not in _NU_CACHE:
        V = multigrid.VCycle(3, k, L)
        A = V.A64[-1]
        b = assemble.rhs(V.levels[-1], k)
        _, h, c = krylov.gmres_left(A, b, V)
        assert c
        _NU_CACHE[(L, k)] = krylov.nu(h)
    return _NU_CACHE[(L, k)]


@pytest.mark.parametrize("L,k", TABLE1_BLOCK)
def test_table1_full_kernel_gmres(L, k):
    """P13: the paper's Table 1, 3D, full kernel, GMRES to 1e-8
    preconditioned by one V-cycle, f == 1, under readings A2/A5/A7/A22."""
    d = _nu_left(L, k) - _table1()[(L, k)]
    lo, hi = (-0.5, 0.5) if k <= 4 else (-0.5, 0.8)
    assert lo <= d <= hi, (L, k, _nu_left(L, k), d)


def test_table1_level_trend_q3():
    """P13: Table 1's level pattern for Q3: nu rises from L = 2 to 3
    (3.4 -> 3.7) and falls from L = 3 to 4 (3.7 -> 3.6).  Under the right-preconditioned
    true-residual reading it rises monotonically (3.22, 3.97, 4.07), which is what led to
    reading A22."""
    n2, n3, n4 = _nu_left(2, 3), _nu_left(3, 3), _nu_left(4, 3)
    assert n3 > n2 + 0.2 and n4 < n3, (n2, n3, n4)


def test_gmres_left_minimises_preconditioned_residual():
    """The left-preconditioned GMRES of reading A22 is pinned against its definition:
    iterate x_j minimises ||M^{-1}(b - A x)|| over the Krylov space, so the reported
    history equals the preconditioned residual norm of the iterate it returns after j
    steps, the norms do not increase, and the converged x solves A x = b."""
    V = multigrid.VCycle(2, 2, 4)
    A = V.A64[-1]
    b = assemble.rhs(V.levels[-1], 2)
    x, h, c = krylov.gmres_left(A, b, V, rtol=1e-12)
    assert c and all(h[i + 1] <= h[i] * (1 + 1e-12) for i in range(len(h) - 1))
    for j in range(1, len(h)):
        xj, hj, _ = krylov.gmres_left(A, b, V, rtol=0.0, max_it=j)
        pr = np.linalg.norm(V(b - A @ xj))
        assert abs(pr - hj[-1]) <= 1e-9 * h[0], (j, pr, hj[-1])
    xs = spla.spsolve(A.tocsc(), b)
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs)
