"""1D building blocks of the oracle (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

PAPER.md:599-604 (Appendix A): the 1D shape functions phi_nu of Q_k are the
Lagrange polynomials on the k+1 Gauss-Lobatto points xi_mu of [0,1],
phi_nu(xi_mu) = delta_{mu nu}.  Quadrature is exact Gauss-Legendre (reading A3
of DESIGN.md: the paper names GLL points as *nodes* only; integrals are exact).
"""
import numpy as np
from numpy.polynomial import legendre as npleg


def gll_nodes(n):
    """The n Gauss-Lobatto points on [0,1]: 0, 1 and the n-2 roots
    of P'_{n-1} mapped from [-1,1].  SPEC.md:125 worked example n=4:
    {0, (1-1/sqrt5)/2, (1+1/sqrt5)/2, 1}."""
    if n < 2:
        raise ValueError("gll_nodes needs n >= 2")
    m = n - 1                                   # polynomial degree k
    cm = np.zeros(m + 1)
    cm[m] = 1.0                                 # P_m in Legendre coefficients
    inner = np.sort(npleg.legroots(npleg.legder(cm))) if m >= 2 else np.array([])
    x = np.concatenate([[-1.0], np.real(inner), [1.0]])
    return (x + 1.0) / 2.0


def gauss(n):
    """n-point Gauss-Legendre rule on [0,1] (library primitive leggauss, mapped).
    SPEC.md:133 worked example n=2: points (1-+1/sqrt3)/2, weights 1/2."""
    x, w = npleg.leggauss(n)
    return (x + 1.0) / 2.0, w / 2.0


def lagrange(nodes, x):
    """Values V[q, j] = phi_j(x_q) and derivatives D[q, j] = phi_j'(x_q) of the
    Lagrange basis on ``nodes``, by the product formula
    phi_j(x) = prod_{m != j} (x - xi_m) / (xi_j - xi_m) and its product-rule
    derivative.  Pure definition, O(n^3) per point."""
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    V = np.ones((len(x), n))
    D = np.zeros((len(x), n))
    for j in range(n):
        others = [m for m in range(n) if m != j]
        denom = np.prod([nodes[j] - nodes[m] for m in others])
        for q, xq in enumerate(x):
            V[q, j] = np.prod([xq - nodes[m] for m in others]) / denom
            s = 0.0
            for a in others:
                s += np.prod([xq - nodes[m] for m in others if m != a])
            D[q, j] = s / denom
    return V, D


def penalty(k, h_minus, h_plus, scale=1.0):
    """gamma_e = k(k+1)(1/h+ + 1/h-).  On a boundary face both
    sides take the cell's own h (reading A2).  SPEC.md:159 worked
    example: k=2, h=1/4 -> 48."""
    return scale * k * (k + 1) * (1.0 / h_plus + 1.0 / h_minus)


# ---------------------------------------------------------------- Hermite-type basis
# (clamped kernel, Fig. 3 right; reading A19)
def hermite_points(k):
    """Interior interpolation points of the Hermite-type basis: the k-3 Gauss
    points on (0,1)."""
    return gauss(k - 3)[0] if k > 3 else np.zeros(0)


def hermite(k, x):
    """Values V[q, j] and derivatives D[q, j] of the Hermite-type basis of Q_k
    (k >= 3): the dual basis of the functionals
        l_0 = v(0), l_1 = v'(0), l_{1+m} = v(eta_m) (m < k-3), l_{k-1} = -v'(1), l_k = v(1)
    (value and derivative at both ends, Lagrange at the interior Gauss points;
    the sign of v'(1) makes the reflection x -> 1-x map psi_j to psi_{k-j}).
    Built by inverting the functional matrix in the shifted Legendre basis."""
    if k < 3:
        raise ValueError("the Hermite-type basis needs k >= 3")
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    eta = hermite_points(k)
    n = k + 1
    F = np.zeros((n, n))
    for m in range(n):
        c = np.zeros(m + 1)
        c[m] = 1.0
        dc = npleg.legder(c) if m > 0 else np.zeros(1)
        F[0, m] = npleg.legval(-1.0, c)
        F[1, m] = 2.0 * npleg.legval(-1.0, dc)
        for i, e in enumerate(eta):
            F[2 + i, m] = npleg.legval(2.0 * e - 1.0, c)
        F[k - 1, m] = -2.0 * npleg.legval(1.0, dc)
        F[k, m] = npleg.legval(1.0, c)
    C = np.linalg.inv(F)                      # psi_j = sum_m C[m, j] P_m(2x - 1)
    V = np.zeros((len(x), n))
    D = np.zeros((len(x), n))
    for m in range(n):
        c = np.zeros(m + 1)
        c[m] = 1.0
        pm = npleg.legval(2.0 * x - 1.0, c)
        dpm = 2.0 * npleg.legval(2.0 * x - 1.0, npleg.legder(c)) if m > 0 else np.zeros_like(x)
        V += np.outer(pm, C[m])
        D += np.outer(dpm, C[m])
    return V, D


def evaluate(kind, k, x):
    """(V, D) of the 1D basis `kind` ('lagrange': GLL Lagrange, 'hermite')."""
    if kind == "hermite":
        return hermite(k, x)
    return lagrange(gll_nodes(k + 1), x)


def child_matrix(kind, k, q):
    """1D embedding of the coarse basis into child q in {0, 1}: B[i, j] = l_i(psi_j
    restricted to the child), l_i the child's defining functionals (nodal values
    for Lagrange; values/derivatives as in `hermite` for Hermite; a child
    derivative is 1/2 of the coarse one)."""
    if kind == "lagrange":
        nodes = gll_nodes(k + 1)
        return lagrange(nodes, (nodes + q) / 2.0)[0]
    eta = hermite_points(k)
    V0, D0 = hermite(k, [q / 2.0])
    V1, D1 = hermite(k, [(1.0 + q) / 2.0])
    Vi = hermite(k, (eta + q) / 2.0)[0] if k > 3 else np.zeros((0, k + 1))
    return np.vstack([V0, 0.5 * D0, Vi, -0.5 * D1, V1])
