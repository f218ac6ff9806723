"""Cartesian mesh hierarchy, cell-wise lexicographic numbering, vertex patches and
colours (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

* Hierarchy T_0 < T_1 < ... by 2^d refinement; T_0 is one cell refined once
  (PAPER.md:142-147).  The oracle allows a general T_0 box ``n0`` of cubic
  cells of size ``h0`` (reading A12 of DESIGN.md); default n0 = (2,)*d, h0=1/2
  (unit cube).
* Numbering: cell-wise lexicographic (Fig. 5 right):
  dof = cell_lin * (k+1)^d + local_lex, x fastest in both.
* Vertex patch: the 2^d cells sharing an interior vertex, ordered
  by the footnote of PAPER.md:384 (the cell whose top-right vertex is the shared
  vertex first, then lexicographic, x fastest).
* Colour of a patch with lowest cell c: sum_i (c_i mod 2) 2^i (Fig. 4,
  PAPER.md:236-240).
"""
import itertools
import numpy as np


class Level:
    def __init__(self, dim, n, h):
        self.dim = dim
        self.n = tuple(int(v) for v in n)       # cells per direction
        self.h = float(h)
        self.ncells = int(np.prod(self.n))

    def cell_lin(self, c):
        """lexicographic cell index, x fastest."""
        lin, stride = 0, 1
        for i in range(self.dim):
            lin += c[i] * stride
            stride *= self.n[i]
        return lin

    def cell_coords(self, lin):
        c = []
        for i in range(self.dim):
            c.append(lin % self.n[i])
            lin //= self.n[i]
        return tuple(c)

    def ndofs(self, k):
        return self.ncells * (k + 1) ** self.dim


def hierarchy(dim, n_levels, n0=None, h0=0.5):
    """Levels 0..n_levels-1; level l has n0*2^l cells per direction, h = h0/2^l
    (PAPER.md:142-147)."""
    if dim not in (1, 2, 3):
        raise ValueError("dim must be 1, 2 or 3")
    if n0 is None:
        n0 = (2,) * dim
    return [Level(dim, [c * 2 ** l for c in n0], h0 / 2 ** l) for l in range(n_levels)]


def patches(level):
    """All vertex patches of a level: list of (lowest_cell, [2^d cell_lin in
    footnote order]) -- one per interior vertex."""
    d = level.dim
    out = []
    ranges = [range(level.n[i] - 1) for i in range(d)]
    # iterate lowest-cell coordinates with x fastest
    for cz in itertools.product(*reversed(ranges)):
        c0 = tuple(reversed(cz))
        cells = []
        for q in itertools.product(*([(0, 1)] * d)):
            q = tuple(reversed(q))              # x fastest inside the patch
            cells.append(level.cell_lin(tuple(c0[i] + q[i] for i in range(d))))
        out.append((c0, cells))
    return out


def colour(c0):
    """Fig. 4 / SPEC.md:65: colour = sum_i (c_i mod 2) 2^i."""
    return sum((c0[i] % 2) << i for i in range(len(c0)))


def coloured_patches(level):
    """2^d colour classes, each a list of patches."""
    classes = [[] for _ in range(2 ** level.dim)]
    for c0, cells in patches(level):
        classes[colour(c0)].append((c0, cells))
    return classes


def patch_dofs(level, cells, k):
    """Global dof indices of a patch in *patch-lexicographic* order (the local
    tensor ordering of PAPER.md:383-384: x fastest over the 2(k+1)-wide patch)."""
    d = level.dim
    nc = k + 1
    npatch = 2 * nc
    idx = np.empty(npatch ** d, dtype=np.int64)
    for lex in range(npatch ** d):
        rem = lex
        p = []
        for _ in range(d):
            p.append(rem % npatch)
            rem //= npatch
        q = [pi // nc for pi in p]               # which cell of the patch
        loc = [pi % nc for pi in p]              # node inside the cell
        cell_in_patch = sum(q[i] << i for i in range(d))
        local_lex = sum(loc[i] * nc ** i for i in range(d))
        idx[lex] = cells[cell_in_patch] * nc ** d + local_lex
    return idx


def boundary_signature(level, c0):
    """Per direction: (low face on the domain boundary, high face on the domain
    boundary) -- patches sharing this signature have identical local matrices
    on a uniform Cartesian level."""
    return tuple((c0[i] == 0, c0[i] + 2 == level.n[i]) for i in range(level.dim))
