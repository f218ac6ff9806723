"""Grid transfer (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

PAPER.md:152: prolongation I^up is the canonical embedding V_l -> V_{l+1};
restriction of residuals is its transpose P^T (reading A4 of DESIGN.md; the
paper's "L2-projection" acting on dual vectors).  The embedding of a Lagrange
function is its nodal interpolant on the fine cell: fine nodal value = coarse
function evaluated at the fine node.
"""
import itertools
import numpy as np
import scipy.sparse as sp

from . import basis
from .mesh import Level


def prolongation(coarse: Level, fine: Level, k, kind="lagrange"):
    """Sparse P (fine ndofs x coarse ndofs), cell-wise lexicographic numbering on
    both levels.  Built by evaluating every coarse basis function at every
    fine-child node (definition of the embedding)."""
    d = coarse.dim
    nc = k + 1
    nodes = basis.gll_nodes(nc)
    nloc = nc ** d
    blocks = {}
    if kind == "hermite":   # tensor product of the 1D child embeddings (basis.child_matrix)
        B1 = [basis.child_matrix(kind, k, q) for q in (0, 1)]
        for q in itertools.product((0, 1), repeat=d):
            B = np.ones((1, 1))
            for i in range(d):              # x fastest: later factors are slower
                B = np.kron(B1[q[i]], B)
            blocks[q] = B
    for q in ([] if kind == "hermite" else itertools.product((0, 1), repeat=d)):
        # fine node coordinates (in the coarse reference cell) of child q
        pts = np.array([[(nodes[(l // nc ** i) % nc] + q[i]) / 2.0 for i in range(d)]
                        for l in range(nloc)])
        B = np.ones((nloc, nloc))
        for i in range(d):
            V, _ = basis.lagrange(nodes, pts[:, i])        # (nloc, nc)
            jl = np.array([(j // nc ** i) % nc for j in range(nloc)])
            B *= V[:, jl]
        blocks[q] = B
    rows, cols, vals = [], [], []
    for cc in range(coarse.ncells):
        C = coarse.cell_coords(cc)
        for q, B in blocks.items():
            F = tuple(2 * C[i] + q[i] for i in range(d))
            fl = fine.cell_lin(F)
            ii, jj = np.nonzero(B)
            rows.append(fl * nloc + ii)
            cols.append(cc * nloc + jj)
            vals.append(B[ii, jj])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(fine.ncells * nloc, coarse.ncells * nloc))
