"""Element-by-element quadrature assembly of the SIPG matrix (TEST INFRASTRUCTURE
ONLY, see oracle/__init__.py).

a_h(u,v) = sum_K int_K grad u . grad v
         + sum_F int_F ( gamma [[u]].[[v]] - {grad u}.[[v]] - [[u]].{grad v} )
(eq. bilinear_form) with {u} = (u+ + u-)/2 and the jump read as
[[u]] = u+ n+ + u- n- (reading A1: PAPER.md:82 prints "(u+ + u-) n+", garbled),
and on boundary faces {u} = u, [[u]] = u n (eq. jump_boundary).
gamma = k(k+1)(1/h+ + 1/h-), boundary faces take h+ = h- = h
(reading A2).

Every cell and face matrix is computed by tensor Gauss quadrature of the full
d-dimensional basis functions phi_{alpha beta gamma}(x) = prod phi(x_i)
 -- *not* from the Kronecker formulas of PAPER.md:118-126, so
the separable structure the GPU path exploits is checked, not assumed.
"""
import numpy as np
import scipy.sparse as sp

from . import basis
from .mesh import Level


def _kron_all(mats):
    """Tensor-product evaluation table: mats[0] is the x factor (fastest)."""
    out = np.ones((1, 1))
    for m in mats:                   # x first, so later factors are slower
        out = np.kron(m, out)
    return out


class Reference:
    """Reference-cell tables for degree k in dimension d (unit cell [0,1]^d)."""

    def __init__(self, dim, k, nq=None, kind="lagrange"):
        self.dim, self.k = dim, k
        self.nc = k + 1
        self.nodes = basis.gll_nodes(self.nc)
        nq = nq if nq is not None else k + 1         # exact for degree 2k (A3)
        self.qx, self.qw = basis.gauss(nq)
        self.V, self.D = basis.evaluate(kind, k, self.qx)        # (nq, nc)
        self.V0, self.D0 = basis.evaluate(kind, k, [0.0])        # (1, nc)
        self.V1, self.D1 = basis.evaluate(kind, k, [1.0])

    def cell_matrices(self, h):
        """Cell stiffness K_ij = int_K grad phi_i . grad phi_j and mass, by
        quadrature at the tensor Gauss points."""
        d = self.dim
        W = _kron_all([np.diag(self.qw)] * d) * h ** d
        Phi = _kron_all([self.V] * d)
        K = np.zeros((self.nc ** d,) * 2)
        for a in range(d):
            G = _kron_all([self.D if i == a else self.V for i in range(d)]) / h
            K += G.T @ W @ G
        M = Phi.T @ W @ Phi
        return K, M

    def face_tables(self, a, side, h):
        """Values and d/dx_a-derivatives of all cell basis functions at the face
        quadrature points of the face x_a = side (0 or 1); weights include the
        h^(d-1) face measure."""
        d = self.dim
        Vn, Dn = (self.V0, self.D0) if side == 0 else (self.V1, self.D1)
        val = _kron_all([Vn if i == a else self.V for i in range(d)])
        der = _kron_all([Dn if i == a else self.V for i in range(d)]) / h
        wt = _kron_all([np.ones((1, 1)) if i == a else np.diag(self.qw) for i in range(d)])
        return val, der, np.diag(wt) * h ** (d - 1)

    def interior_face_blocks(self, a, h, gamma):
        """Blocks B[s][t] (test side s, trial side t, side 0 = K- at x_a=1 of
        its cell, side 1 = K+ at x_a=0) of
        int_F gamma (u- - u+)(v- - v+) - 1/2(d_a u- + d_a u+)(v- - v+)
                                      - 1/2(u- - u+)(d_a v- + d_a v+)."""
        vm, dm, w = self.face_tables(a, 1, h)
        vp, dp, _ = self.face_tables(a, 0, h)
        vals, ders, sig = (vm, vp), (dm, dp), (1.0, -1.0)
        W = np.diag(w)
        B = [[None, None], [None, None]]
        for s in range(2):
            for t in range(2):
                B[s][t] = (gamma * sig[s] * sig[t] * vals[s].T @ W @ vals[t]
                           - 0.5 * sig[s] * vals[s].T @ W @ ders[t]
                           - 0.5 * sig[t] * ders[s].T @ W @ vals[t])
        return B

    def boundary_face_block(self, a, side, h, gamma):
        """int_F gamma u v - d_n u v - u d_n v, d_n = -d_a on the low face
        (side 0) and +d_a on the high face (side 1)."""
        v, dd, w = self.face_tables(a, side, h)
        sgn = -1.0 if side == 0 else 1.0
        W = np.diag(w)
        return gamma * v.T @ W @ v - sgn * (v.T @ W @ dd + dd.T @ W @ v)


def _place(rows, cols, vals, block, row_cells, col_cells, nloc):
    ii, jj = np.nonzero(block)
    if len(ii) == 0 or len(row_cells) == 0:
        return
    rows.append((np.asarray(row_cells)[:, None] * nloc + ii[None, :]).ravel())
    cols.append((np.asarray(col_cells)[:, None] * nloc + jj[None, :]).ravel())
    vals.append(np.broadcast_to(block[ii, jj][None, :], (len(row_cells), len(ii))).ravel())


def _cell_grid(level):
    """coords[i] = array of cell coordinate i for every cell, in lex order."""
    grids = np.meshgrid(*[np.arange(n) for n in level.n], indexing="ij")
    lin = np.zeros(level.n, dtype=np.int64)
    stride = 1
    for i in range(level.dim):
        lin = lin + grids[i] * stride
        stride *= level.n[i]
    return grids, lin


def assemble(level: Level, k, penalty_scale=1.0, kind="lagrange", boundary_penalty_scale=1.0):
    """Global SIPG matrix of ``level`` in cell-wise lexicographic numbering, CSR.
    Exact zeros (e.g. phi_i(0) = 0 for i != 0 on GLL nodes) are not stored.
    kind: 1D basis ('lagrange' GLL, or 'hermite' for the clamped kernel).
    boundary_penalty_scale: the boundary-face penalty relative to the interior
    one (reading A2: 1, both sides take the cell's h; 0.5 is the one-sided
    k(k+1)/h, the probe of DESIGN.md "Table 1 readings")."""
    d, h = level.dim, level.h
    ref = Reference(d, k, kind=kind)
    nloc = ref.nc ** d
    gamma = basis.penalty(k, h, h, penalty_scale)
    gamma_b = boundary_penalty_scale * gamma
    rows, cols, vals = [], [], []
    grids, lin = _cell_grid(level)
    K, _ = ref.cell_matrices(h)
    allc = lin.ravel()
    _place(rows, cols, vals, K, allc, allc, nloc)
    for a in range(d):
        B = ref.interior_face_blocks(a, h, gamma)
        sl_m = [slice(None)] * d
        sl_p = [slice(None)] * d
        sl_m[a] = slice(0, level.n[a] - 1)
        sl_p[a] = slice(1, level.n[a])
        cm = lin[tuple(sl_m)].ravel()
        cp = lin[tuple(sl_p)].ravel()
        for s, cs in ((0, cm), (1, cp)):
            for t, ct in ((0, cm), (1, cp)):
                _place(rows, cols, vals, B[s][t], cs, ct, nloc)
        for side in (0, 1):
            Bb = ref.boundary_face_block(a, side, h, gamma_b)
            sl = [slice(None)] * d
            sl[a] = 0 if side == 0 else level.n[a] - 1
            cb = lin[tuple(sl)].ravel()
            _place(rows, cols, vals, Bb, cb, cb, nloc)
    n = level.ncells * nloc
    A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(n, n)).tocsr()
    A.sum_duplicates()
    A.eliminate_zeros()
    return A


def cell_nodes(level: Level, k):
    """Physical coordinates of every dof (cell-wise lexicographic order):
    array (ndofs, d)."""
    d, h = level.dim, level.h
    nodes = basis.gll_nodes(k + 1)
    nc = k + 1
    out = np.zeros((level.ncells * nc ** d, d))
    loc = np.array([[nodes[(l // nc ** i) % nc] for i in range(d)] for l in range(nc ** d)])
    for c in range(level.ncells):
        cc = np.array(level.cell_coords(c), dtype=np.float64)
        out[c * nc ** d:(c + 1) * nc ** d] = (cc[None, :] + loc) * h
    return out


def interpolate(level: Level, k, u):
    """Nodal interpolant I_h u (u: callable on an (n, d) coordinate array)."""
    return u(cell_nodes(level, k))


def rhs(level: Level, k, f=None, nq=None, kind="lagrange"):
    """b_i = int f phi_i (eq. weak_form) by tensor Gauss
    quadrature with k+3 points per direction; f=None means f == 1
    (PAPER.md:331)."""
    d, h = level.dim, level.h
    ref = Reference(d, k, nq=nq if nq is not None else k + 3, kind=kind)
    Phi = _kron_all([ref.V] * d)
    w = np.diag(_kron_all([np.diag(ref.qw)] * d)) * h ** d
    nq1 = len(ref.qx)
    qloc = np.array([[ref.qx[(l // nq1 ** i) % nq1] for i in range(d)] for l in range(nq1 ** d)])
    nloc = ref.nc ** d
    b = np.zeros(level.ncells * nloc)
    for c in range(level.ncells):
        cc = np.array(level.cell_coords(c), dtype=np.float64)
        fq = np.ones(len(qloc)) if f is None else f((cc[None, :] + qloc) * h)
        b[c * nloc:(c + 1) * nloc] = Phi.T @ (w * fq)
    return b


def l2_error(level: Level, k, uh, u, nq=None):
    """|| u_h - u ||_{L2} by Gauss quadrature with k+3 points per direction."""
    d, h = level.dim, level.h
    ref = Reference(d, k, nq=nq if nq is not None else k + 3)
    Phi = _kron_all([ref.V] * d)
    w = np.diag(_kron_all([np.diag(ref.qw)] * d)) * h ** d
    nq1 = len(ref.qx)
    qloc = np.array([[ref.qx[(l // nq1 ** i) % nq1] for i in range(d)] for l in range(nq1 ** d)])
    nloc = ref.nc ** d
    err2 = 0.0
    for c in range(level.ncells):
        cc = np.array(level.cell_coords(c), dtype=np.float64)
        e = Phi @ uh[c * nloc:(c + 1) * nloc] - u((cc[None, :] + qloc) * h)
        err2 += np.sum(w * e * e)
    return np.sqrt(err2)
