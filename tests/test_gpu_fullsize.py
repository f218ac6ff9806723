"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (C2: 2D k=7, 1024^2 cells, 10 levels, 67M dofs; C3 k=4: 3D 128x128x64
cells, 131M dofs), on SAMPLED outputs the oracle computes one by one.

The operator and the smoother are local: a cell's output depends on its face
neighbours, a patch's on the ring of cells around it.  The oracle assembles
the SIPG matrix element by element on the small window of cells around each
sample (the window edge coincides with the domain boundary where the sample
touches it, and is at least one cell away from the sampled rows otherwise) and
evaluates the sampled rows exactly.  Vectors are gathered with the documented
library layout (include/ipmg.h).  Plus whole-vector properties of the full-size
CG solve: convergence in the paper's iteration count, the true residual, and
the mirror symmetry of the discrete solution of f == 1 on the unit square.
"""
import functools

import numpy as np
import pytest
import scipy.linalg as sla

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import assemble, mesh  # noqa: E402

C2 = dict(dim=2, k=7, nl=10, coarse=(2, 2))
C3K4 = dict(dim=3, k=4, nl=7, coarse=(2, 2, 1))


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@functools.lru_cache(maxsize=None)
def handle(dim, k, nl, coarse):
    from paper_2405_18982_b200 import ipmg
    return ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=ipmg.FP32)


def lib_offsets(n, c, k, dim):
    """Library-order dof range of cell c on a parent-grouped level with n cells."""
    cell = (k + 1) ** dim
    parent = (c[0] // 2) + (n[0] // 2) * ((c[1] // 2) + ((n[1] // 2) * (c[2] // 2) if dim == 3 else 0))
    child = (c[0] & 1) + 2 * (c[1] & 1) + (4 * (c[2] & 1) if dim == 3 else 0)
    base = (parent * 2 ** dim + child) * cell
    return np.arange(base, base + cell)


def window_dofs(n, lo, hi, k, dim):
    """Library offsets of the window cells [lo, hi) in the window's cell-wise
    lexicographic order (the oracle's numbering)."""
    ranges = [range(lo[a], hi[a]) for a in range(dim)]
    out = []
    if dim == 2:
        for cy in ranges[1]:
            for cx in ranges[0]:
                out.append(lib_offsets(n, (cx, cy), k, dim))
    else:
        for cz in ranges[2]:
            for cy in ranges[1]:
                for cx in ranges[0]:
                    out.append(lib_offsets(n, (cx, cy, cz), k, dim))
    return np.concatenate(out)


def samples(n, dim, count, seed, margin=0):
    rng = np.random.default_rng(seed)
    pts = [tuple(0 for _ in range(dim)), tuple(v - 1 - margin for v in n)]      # corners
    pts += [tuple(int(rng.integers(0, v - margin)) for v in n) for _ in range(count)]
    return pts


def _fetch(t, idx):
    return t[torch.as_tensor(idx, device=t.device)].double().cpu().numpy()


@pytest.mark.parametrize("cfg", [C2, C3K4], ids=["C2", "C3k4"])
def test_fullsize_vmult_sampled(cfg):
    _need_gpu()
    dim, k, nl = cfg["dim"], cfg["k"], cfg["nl"]
    h = handle(dim, k, nl, cfg["coarse"])
    L = nl - 1
    n_dofs, cells, hs = h.level_info(L)
    n = cells[:dim]
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand(n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y = torch.empty_like(x)
    h.vmult(L, x, y)
    torch.cuda.synchronize()
    worst = 0.0
    for c in samples(n, dim, 24, seed=11):
        lo = [max(c[a] - 1, 0) for a in range(dim)]
        hi = [min(c[a] + 2, n[a]) for a in range(dim)]
        wl = mesh.Level(dim, [hi[a] - lo[a] for a in range(dim)], hs)
        A = assemble.assemble(wl, k)
        idx = window_dofs(n, lo, hi, k, dim)
        ref_all = A @ _fetch(x, idx)
        center = wl.cell_lin(tuple(c[a] - lo[a] for a in range(dim)))
        cell = (k + 1) ** dim
        ref = ref_all[center * cell:(center + 1) * cell]
        got = _fetch(y, lib_offsets(n, c, k, dim))
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    assert worst <= 1e-12, worst


@pytest.mark.parametrize("cfg", [C2, C3K4], ids=["C2", "C3k4"])
def test_fullsize_smoother_colour_sampled(cfg):
    """One fp32 colour pass of Algorithm 1 at full size; sampled patches against
    the oracle's dense local solve x_j = A_jj^{-1} (b_j - A_{j,ring} x_ring)
    (fp64 on the same fp32-rounded inputs, reading A18), 1e-5."""
    _need_gpu()
    dim, k, nl = cfg["dim"], cfg["k"], cfg["nl"]
    h = handle(dim, k, nl, cfg["coarse"])
    L = nl - 1
    n_dofs, cells, hs = h.level_info(L)
    n = cells[:dim]
    g = torch.Generator(device="cuda").manual_seed(8)
    x = (torch.rand(n_dofs, device="cuda", generator=g) * 2 - 1).float()
    b = (torch.rand(n_dofs, device="cuda", generator=g) * 2 - 1).float()
    colour = (1 << dim) - 1                       # shifted in every direction
    out = torch.empty_like(x)
    h.smooth_colour(L, x, b, out, colour)
    torch.cuda.synchronize()
    worst = 0.0
    for c in samples(n, dim, 12, seed=12, margin=2):
        c0 = tuple(min(max(((v >> 1) << 1) + 1, 1), n[a] - 3) for a, v in enumerate(c))   # odd: this colour
        lo = [max(c0[a] - 1, 0) for a in range(dim)]
        hi = [min(c0[a] + 3, n[a]) for a in range(dim)]
        wl = mesh.Level(dim, [hi[a] - lo[a] for a in range(dim)], hs)
        A = assemble.assemble(wl, k).toarray()
        idx = window_dofs(n, lo, hi, k, dim)
        xw, bw = _fetch(x, idx), _fetch(b, idx)
        cells_local = []
        for q in range(2 ** dim):
            cq = tuple(c0[a] + ((q >> a) & 1) - lo[a] for a in range(dim))
            cells_local.append(wl.cell_lin(cq))
        P = mesh.patch_dofs(wl, cells_local, k)
        ring = np.setdiff1d(np.arange(A.shape[0]), P)
        ref = sla.solve(A[np.ix_(P, P)], bw[P] - A[np.ix_(P, ring)] @ xw[ring])
        refmap = dict(zip(P.tolist(), ref.tolist()))
        cell = (k + 1) ** dim
        ref_cells, got = [], []
        for q in range(2 ** dim):
            cg = tuple(c0[a] + ((q >> a) & 1) for a in range(dim))
            got.append(_fetch(out, lib_offsets(n, cg, k, dim)))
            ref_cells.extend(refmap[cells_local[q] * cell + l] for l in range(cell))
        got, ref_cells = np.concatenate(got), np.array(ref_cells)
        worst = max(worst, np.abs(got - ref_cells).max() / np.abs(ref_cells).max())
    assert worst <= 1e-5, worst


def test_fullsize_cg_C2():
    """The bench solve itself: 5 CG iterations (oracle and B200 agree at every
    smaller size), true residual <= 1e-8 ||b|| with the (sample-checked) fp64
    operator, and the solution's mirror symmetry x <-> 1-x, x <-> y on the unit
    square (f == 1)."""
    _need_gpu()
    dim, k, nl = C2["dim"], C2["k"], C2["nl"]
    h = handle(dim, k, nl, C2["coarse"])
    L = nl - 1
    n_dofs, cells, _ = h.level_info(L)
    b = torch.empty(n_dofs, dtype=torch.float64, device="cuda")
    h.rhs(L, b)
    x = torch.empty_like(b)
    res = h.cg_solve(b, x, rtol=1e-8, max_it=50)
    assert res["converged"] and res["iterations"] == 5, res["iterations"]
    ax = torch.empty_like(x)
    h.vmult(L, x, ax)
    assert float(torch.linalg.norm(b - ax) / torch.linalg.norm(b)) <= 1e-8 * (1 + 1e-6)
    n = cells[:dim]
    nc = k + 1
    xmax = float(x.abs().max())
    for c in samples(n, dim, 16, seed=13):
        v = _fetch(x, lib_offsets(n, c, k, dim)).reshape(nc, nc)            # [iy, ix]
        mx = _fetch(x, lib_offsets(n, (n[0] - 1 - c[0], c[1]), k, dim)).reshape(nc, nc)[:, ::-1]
        tr = _fetch(x, lib_offsets(n, (c[1], c[0]), k, dim)).reshape(nc, nc).T
        assert np.abs(v - mx).max() <= 1e-6 * xmax
        assert np.abs(v - tr).max() <= 1e-6 * xmax
