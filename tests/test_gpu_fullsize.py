"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (C4, the headline: 3D k=4, 256x256x128 cells, 8 levels, 1.05B dofs; C2: 2D
k=7, 1024^2 cells, 10 levels, 67M dofs; C3 k=4: 3D 128x128x64 cells, 131M dofs),
on SAMPLED outputs the oracle computes one by one.

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
C4 = dict(dim=3, k=4, nl=8, coarse=(2, 2, 1))
CFGS, CFG_IDS = [C2, C3K4, C4], ["C2", "C3k4", "C4"]


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@functools.lru_cache(maxsize=1)   # one full-size handle at a time (C4 alone holds ~40 GB)
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


@pytest.mark.parametrize("cfg", CFGS, ids=CFG_IDS)
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


# (colour, x given?, dtype, tolerance): the shifted-everywhere colour in fp32 (the
# bench's V-cycle precision) and fp64, colour 1 in fp32, and the zero-start colour 0
SMOOTH_CASES = [("all", True, "fp32"), ("all", True, "fp64"), ("c1", True, "fp32"), ("zero", False, "fp32")]


@pytest.mark.parametrize("case", SMOOTH_CASES, ids=["shifted-fp32", "shifted-fp64", "c1-fp32", "zero-fp32"])
@pytest.mark.parametrize("cfg", CFGS, ids=CFG_IDS)
def test_fullsize_smoother_colour_sampled(cfg, case):
    """One colour pass of Algorithm 1 at full size; sampled patches against the
    oracle's dense local solve x_j = A_jj^{-1} (b_j - A_{j,ring} x_ring) (fp64 on the
    same fp32-rounded inputs, reading A18): 1e-5 in fp32, 1e-12 in fp64."""
    _need_gpu()
    which, with_x, prec = case
    dim, k, nl = cfg["dim"], cfg["k"], cfg["nl"]
    h = handle(dim, k, nl, cfg["coarse"])
    L = nl - 1
    n_dofs, cells, hs = h.level_info(L)
    n = cells[:dim]
    dt, tol = (torch.float32, 1e-5) if prec == "fp32" else (torch.float64, 1e-12)
    g = torch.Generator(device="cuda").manual_seed(8)
    x = (torch.rand(n_dofs, device="cuda", generator=g) * 2 - 1).to(dt)
    b = (torch.rand(n_dofs, device="cuda", generator=g) * 2 - 1).to(dt)
    colour = (1 << dim) - 1 if which == "all" else (1 if which == "c1" else 0)
    out = torch.empty_like(x)
    h.smooth_colour(L, x if with_x else None, b, out, colour)
    torch.cuda.synchronize()
    if not with_x:
        x.zero_()
    worst = 0.0
    for c in samples(n, dim, 12, seed=12, margin=2):
        # lowest patch cell of this colour: parity (colour >> a) & 1 in direction a
        c0 = []
        for a, v in enumerate(c):
            par = (colour >> a) & 1
            lo_c = 1 if par else 0
            c0.append(min(max(((v >> 1) << 1) + par, lo_c), n[a] - 2 - (1 if par else 0)))
        c0 = tuple(c0)
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
    assert worst <= tol, worst


def _child_prolongation(dim, k):
    """P of one coarse cell onto its 2^d children (children in the 2^d-cell level's
    lexicographic order), from the oracle's definition of the embedding."""
    from oracle import transfer
    return transfer.prolongation(mesh.Level(dim, [1] * dim, 1.0), mesh.Level(dim, [2] * dim, 0.5), k).toarray()


@pytest.mark.parametrize("cfg", CFGS, ids=CFG_IDS)
def test_fullsize_residual_restrict_sampled(cfg):
    """r_c = P^T (b - A x) (fp32) at sampled coarse cells: the oracle forms the fine
    residual on the children from the window operator, then applies P^T (reading A4)."""
    _need_gpu()
    dim, k, nl = cfg["dim"], cfg["k"], cfg["nl"]
    h = handle(dim, k, nl, cfg["coarse"])
    L = nl - 1
    n_dofs, cells, hs = h.level_info(L)
    nc_dofs, ccells, _ = h.level_info(L - 1)
    n, nco = cells[:dim], ccells[:dim]
    g = torch.Generator(device="cuda").manual_seed(9)
    x = (torch.rand(n_dofs, device="cuda", generator=g) * 2 - 1).float()
    b = (torch.rand(n_dofs, device="cuda", generator=g) * 2 - 1).float()
    rc = torch.empty(nc_dofs, device="cuda")
    h.residual_restrict(L, x, b, rc)
    torch.cuda.synchronize()
    Pc = _child_prolongation(dim, k)
    two = mesh.Level(dim, [2] * dim, 0.5)
    cell = (k + 1) ** dim
    worst = 0.0
    for C in samples(nco, dim, 10, seed=14):
        F0 = [2 * C[a] for a in range(dim)]
        lo = [max(F0[a] - 1, 0) for a in range(dim)]
        hi = [min(F0[a] + 3, n[a]) for a in range(dim)]
        wl = mesh.Level(dim, [hi[a] - lo[a] for a in range(dim)], hs)
        A = assemble.assemble(wl, k)
        idx = window_dofs(n, lo, hi, k, dim)
        rw = _fetch(b, idx) - A @ _fetch(x, idx)
        rch = np.zeros(two.ncells * cell)
        for q in range(2 ** dim):
            qq = tuple((q >> a) & 1 for a in range(dim))
            wlin = wl.cell_lin(tuple(F0[a] + qq[a] - lo[a] for a in range(dim)))
            tlin = two.cell_lin(qq)
            rch[tlin * cell:(tlin + 1) * cell] = rw[wlin * cell:(wlin + 1) * cell]
        ref = Pc.T @ rch
        got = _fetch(rc, lib_offsets(nco, C, k, dim))
        worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
    assert worst <= 1e-5, worst


@pytest.mark.parametrize("cfg", CFGS, ids=CFG_IDS)
def test_fullsize_prolongate_add_sampled(cfg):
    """x_f += P e_c (fp32) at sampled coarse cells: the fine children of a coarse
    cell against the oracle's embedding of that cell's function."""
    _need_gpu()
    dim, k, nl = cfg["dim"], cfg["k"], cfg["nl"]
    h = handle(dim, k, nl, cfg["coarse"])
    L = nl - 1
    n_dofs, cells, _ = h.level_info(L)
    nc_dofs, ccells, _ = h.level_info(L - 1)
    n, nco = cells[:dim], ccells[:dim]
    g = torch.Generator(device="cuda").manual_seed(10)
    xf = (torch.rand(n_dofs, device="cuda", generator=g) * 2 - 1).float()
    ec = (torch.rand(nc_dofs, device="cuda", generator=g) * 2 - 1).float()
    Cs = samples(nco, dim, 10, seed=15)
    cell = (k + 1) ** dim
    before = {C: [_fetch(xf, lib_offsets(n, tuple(2 * C[a] + ((q >> a) & 1) for a in range(dim)), k, dim))
                  for q in range(2 ** dim)] for C in Cs}
    h.prolongate_add(L, ec, xf)
    torch.cuda.synchronize()
    Pc = _child_prolongation(dim, k)
    two = mesh.Level(dim, [2] * dim, 0.5)
    worst = 0.0
    for C in Cs:
        pe = Pc @ _fetch(ec, lib_offsets(nco, C, k, dim))
        for q in range(2 ** dim):
            qq = tuple((q >> a) & 1 for a in range(dim))
            tlin = two.cell_lin(qq)
            ref = before[C][q] + pe[tlin * cell:(tlin + 1) * cell]
            got = _fetch(xf, lib_offsets(n, tuple(2 * C[a] + qq[a] for a in range(dim)), k, dim))
            worst = max(worst, np.abs(got - ref).max() / np.abs(ref).max())
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


def test_fullsize_cg_C4():
    """The headline solve (C4, 1.05B dofs): converged in 5 iterations (the level-
    independent count of every smaller C4-shaped hierarchy, profiles/), true residual
    <= 1e-8 ||b|| with the sample-checked fp64 operator, and the symmetries of the
    discrete solution of f == 1 on (0,1)^2 x (0,1/2): x <-> 1-x, x <-> y, z <-> 1/2-z."""
    _need_gpu()
    dim, k, nl = C4["dim"], C4["k"], C4["nl"]
    h = handle(dim, k, nl, C4["coarse"])
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
    del ax
    n = cells[:dim]
    nc = k + 1
    xmax = float(x.abs().max())
    for c in samples(n, dim, 16, seed=16):
        v = _fetch(x, lib_offsets(n, c, k, dim)).reshape(nc, nc, nc)             # [iz, iy, ix]
        mx = _fetch(x, lib_offsets(n, (n[0] - 1 - c[0], c[1], c[2]), k, dim)).reshape(nc, nc, nc)[:, :, ::-1]
        tr = _fetch(x, lib_offsets(n, (c[1], c[0], c[2]), k, dim)).reshape(nc, nc, nc).transpose(0, 2, 1)
        mz = _fetch(x, lib_offsets(n, (c[0], c[1], n[2] - 1 - c[2]), k, dim)).reshape(nc, nc, nc)[::-1, :, :]
        for other in (mx, tr, mz):
            assert np.abs(v - other).max() <= 1e-6 * xmax
