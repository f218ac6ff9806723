"""Outer Krylov solvers and the fractional iteration count (TEST INFRASTRUCTURE
ONLY, see oracle/__init__.py).

* PCG (the north star's outer solver; reading A8): x0 = 0 (reading A11), stop
  when ||r_n||_2 <= rtol ||r_0||_2 with the true (unpreconditioned) residual,
  rtol = 1e-8.  n counts A-applications.
* GMRES: right-preconditioned, no restart, modified Gram-Schmidt (the paper's
  outer solver).
* nu = -8 / log10(rbar), rbar = (||r_n|| / ||r_0||)^(1/n) (PAPER.md:333-335,
  printed garbled as "-8 log10 rbar"; reading A6).
"""
import numpy as np


def nu(history):
    """Fractional iteration count from a residual-norm history r_0..r_n."""
    n = len(history) - 1
    if n < 1 or history[0] == 0:
        return 0.0
    return -8.0 * n / np.log10(history[-1] / history[0])


def pcg(A, b, M, rtol=1e-8, max_it=200):
    """Preconditioned CG; A, M: callables (or matrices).  Returns
    (x, history, converged)."""
    Aop = A if callable(A) else (lambda v: A @ v)
    Mop = M if callable(M) else (lambda v: M @ v)
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    r0 = np.linalg.norm(r)
    hist = [r0]
    if r0 == 0.0:
        return x, hist, True
    z = Mop(r)
    p = z.copy()
    rz = r @ z
    for _ in range(max_it):
        q = Aop(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        rn = np.linalg.norm(r)
        hist.append(rn)
        if rn <= rtol * r0:
            return x, hist, True
        z = Mop(r)
        rz_new = r @ z
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    return x, hist, False


def gmres(A, b, M, rtol=1e-8, max_it=200):
    """Right-preconditioned GMRES without restart (MGS).  Returns
    (x, history, converged); history holds the least-squares residual norms,
    equal to ||b - A x_j|| in exact arithmetic."""
    Aop = A if callable(A) else (lambda v: A @ v)
    Mop = M if callable(M) else (lambda v: M @ v)
    b = np.asarray(b, dtype=np.float64)
    beta0 = np.linalg.norm(b)
    hist = [beta0]
    if beta0 == 0.0:
        return np.zeros_like(b), hist, True
    V = [b / beta0]
    Z = []
    H = np.zeros((max_it + 1, max_it))
    cs, sn = np.zeros(max_it), np.zeros(max_it)
    g = np.zeros(max_it + 1)
    g[0] = beta0
    conv = False
    j = 0
    for j in range(max_it):
        z = Mop(V[j])
        Z.append(z)
        w = Aop(z)
        for i in range(j + 1):
            H[i, j] = w @ V[i]
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        V.append(w / H[j + 1, j] if H[j + 1, j] != 0 else w)
        for i in range(j):                      # apply previous rotations
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        den = np.hypot(H[j, j], H[j + 1, j])
        cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        hist.append(abs(g[j + 1]))
        if abs(g[j + 1]) <= rtol * beta0:
            conv = True
            break
    m = j + 1
    y = np.linalg.solve(np.triu(H[:m, :m]), g[:m])
    x = sum(y[i] * Z[i] for i in range(m))
    return x, hist, conv


def gmres_left(A, b, M, rtol=1e-8, max_it=200):
    """Left-preconditioned GMRES without restart (MGS) on M^{-1} A x = M^{-1} b,
    x0 = 0, stopping on the PRECONDITIONED residual |g_{j+1}| <= rtol ||M^{-1} b||.
    This is a probe of how the paper's nu may have been measured (DESIGN.md
    "Table 1 readings", reading A22: a solver whose default is left
    preconditioning reports the preconditioned residual norm)
    itself says "Euclidean norm of the residual".  Returns (x, history,
    converged); history = ||M^{-1} b||, |g_1|, .., |g_n|."""
    Aop = A if callable(A) else (lambda v: A @ v)
    Mop = M if callable(M) else (lambda v: M @ v)
    r0 = Mop(np.asarray(b, dtype=np.float64))
    beta0 = np.linalg.norm(r0)
    hist = [beta0]
    if beta0 == 0.0:
        return np.zeros_like(r0), hist, True
    V = [r0 / beta0]
    H = np.zeros((max_it + 1, max_it))
    cs, sn = np.zeros(max_it), np.zeros(max_it)
    g = np.zeros(max_it + 1)
    g[0] = beta0
    conv = False
    j = 0
    for j in range(max_it):
        w = Mop(Aop(V[j]))
        for i in range(j + 1):
            H[i, j] = w @ V[i]
            w = w - H[i, j] * V[i]
        H[j + 1, j] = np.linalg.norm(w)
        V.append(w / H[j + 1, j] if H[j + 1, j] != 0 else w)
        for i in range(j):
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        den = np.hypot(H[j, j], H[j + 1, j])
        cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
        H[j, j] = den
        H[j + 1, j] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        hist.append(abs(g[j + 1]))
        if abs(g[j + 1]) <= rtol * beta0:
            conv = True
            break
    m = j + 1
    y = np.linalg.solve(np.triu(H[:m, :m]), g[:m])
    x = sum(y[i] * V[i] for i in range(m))
    return x, hist, conv
