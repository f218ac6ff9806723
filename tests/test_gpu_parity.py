"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle, element
by element on the same seeded inputs.

Tolerances (north star, BASELINE.json): fp64 operator / smoother / V-cycle /
CG solution 1e-12 relative; fp32 kernels 1e-5 relative against the fp64 oracle
evaluated on the same fp32-rounded inputs (reading A18); CG iteration counts
+-1.  Vectors are compared in cell-wise lexicographic order through the
library's ipmg_to_cellwise (itself checked against the documented layout).
"""
import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import assemble, krylov, mesh, multigrid, smoother, transfer  # noqa: E402
from synth_inputs import uniform  # noqa: E402


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@functools.lru_cache(maxsize=None)
def handle(dim, k, nl, coarse=None, vprec=1, smoother_kind=0):
    from paper_2405_18982_b200 import ipmg
    return ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=vprec, smoother=smoother_kind)


@functools.lru_cache(maxsize=None)
def oracle_levels(dim, k, nl, coarse=None):
    levels = mesh.hierarchy(dim, nl, coarse)
    ops = [assemble.assemble(lv, k) for lv in levels]
    return levels, ops


def dev(a, dtype=torch.float64):
    return torch.tensor(np.asarray(a), dtype=dtype, device="cuda")


def to_lib(h, level, v_cw, dtype=torch.float64):
    """oracle (cell-wise) numpy vector -> library-order device tensor"""
    src = dev(v_cw, dtype)
    out = torch.empty_like(src)
    h.from_cellwise(level, src, out)
    return out


def to_cw(h, level, t):
    out = torch.empty_like(t)
    h.to_cellwise(level, t, out)
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


def rel(a, b):
    """Relative error: the larger of the norm-wise ||a-b|| / ||b|| and the element-wise
    max|a-b| / max|b| (a few wrong entries of a long vector fail the second)."""
    nrm = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    ele = np.abs(a - b).max() / max(np.abs(b).max(), 1e-300) if np.size(b) else 0.0
    return max(nrm, ele)


# (dim, k, n_levels, coarse) -- several CTAs, ragged last CTA, every boundary variant
CASES = [(2, 1, 4, None), (2, 2, 4, None), (2, 3, 4, None), (2, 4, 3, None), (2, 5, 3, None),
         (2, 6, 3, None), (2, 7, 3, None), (2, 3, 3, (2, 1)), (3, 1, 3, None), (3, 2, 3, None),
         (3, 3, 2, None), (3, 4, 2, None), (3, 5, 2, None), (3, 6, 2, None), (3, 7, 2, None),
         (3, 2, 3, (2, 1, 2)), (3, 4, 3, None)]
IDS = ["d%dk%dL%d%s" % (c[0], c[1], c[2], "" if c[3] is None else "c" + "".join(map(str, c[3]))) for c in CASES]


def test_layout_permutation_matches_documented_formula():
    _need_gpu()
    dim, k, nl = 3, 2, 3
    h = handle(dim, k, nl)
    L = nl - 1
    n, cells, _ = h.level_info(L)
    nc = k + 1
    cell = nc ** dim
    x = dev(np.arange(n, dtype=np.float64))
    y = torch.empty_like(x)
    h.to_cellwise(L, x, y)
    got = y.cpu().numpy()
    # documented layout (include/ipmg.h): ((parent_lex*2^d + child_lex)*cell + node)
    exp = np.empty(n)
    for c in range(cells[0] * cells[1] * cells[2]):
        cx, cy, cz = c % cells[0], (c // cells[0]) % cells[1], c // (cells[0] * cells[1])
        plin = (cx // 2) + (cells[0] // 2) * ((cy // 2) + (cells[1] // 2) * (cz // 2))
        lib = (plin * 8 + (cx & 1) + 2 * (cy & 1) + 4 * (cz & 1)) * cell
        exp[c * cell:(c + 1) * cell] = np.arange(lib, lib + cell)
    assert np.array_equal(got, exp)
    z = torch.empty_like(x)
    h.from_cellwise(L, y, z)
    assert torch.equal(z, x)


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_vmult(case):
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle(dim, k, nl, coarse)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    for L in range(1, nl):
        A = ops[L]
        x = uniform(A.shape[0], seed=10 + L)
        y_ref = A @ x
        for dtype, tol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
            xr = np.asarray(torch.tensor(x, dtype=dtype).double())
            xl = to_lib(h, L, x, dtype)
            yl = torch.empty_like(xl)
            h.vmult(L, xl, yl)
            got = to_cw(h, L, yl)
            ref = A @ xr
            assert rel(got, ref) <= tol, (L, dtype, rel(got, ref))
    assert y_ref is not None


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_smoother_colours_and_step(case):
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle(dim, k, nl, coarse)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    L = nl - 1
    A = ops[L]
    S = smoother.PatchSmoother(levels[L], k, A)
    x = uniform(A.shape[0], seed=21)
    b = uniform(A.shape[0], seed=22)
    for dtype, tol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
        xr = np.asarray(torch.tensor(x, dtype=dtype).double())
        br = np.asarray(torch.tensor(b, dtype=dtype).double())
        xl, bl = to_lib(h, L, x, dtype), to_lib(h, L, b, dtype)
        for c in range(2 ** dim):
            out = torch.empty_like(xl)
            h.smooth_colour(L, xl, bl, out, c)
            ref = xr.copy()
            for idx, delta in S.local_solves(c, br - A @ xr):
                ref[idx] += delta
            assert rel(to_cw(h, L, out), ref) <= tol, (c, dtype)
        # x_in = NULL (zero start)
        out = torch.empty_like(xl)
        h.smooth_colour(L, None, bl, out, 0)
        ref = np.zeros_like(xr)
        for idx, delta in S.local_solves(0, br):
            ref[idx] += delta
        assert rel(to_cw(h, L, out), ref) <= tol
        for rev in (False, True):
            xs = xl.clone()
            h.smooth(L, xs, bl, reverse=rev)
            ref = S.smooth(xr, br, reverse=rev)
            assert rel(to_cw(h, L, xs), ref) <= tol, (rev, dtype)


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_transfers_and_coarse(case):
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle(dim, k, nl, coarse)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    for L in range(1, nl):
        P = transfer.prolongation(levels[L - 1], levels[L], k)
        A = ops[L]
        x = uniform(A.shape[0], seed=31)
        b = uniform(A.shape[0], seed=32)
        e = uniform(P.shape[1], seed=33)
        for dtype, tol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
            xr = np.asarray(torch.tensor(x, dtype=dtype).double())
            br = np.asarray(torch.tensor(b, dtype=dtype).double())
            er = np.asarray(torch.tensor(e, dtype=dtype).double())
            xl, bl = to_lib(h, L, x, dtype), to_lib(h, L, b, dtype)
            rc = torch.empty(P.shape[1], dtype=dtype, device="cuda")
            h.residual_restrict(L, xl, bl, rc)
            assert rel(to_cw(h, L - 1, rc), P.T @ (br - A @ xr)) <= tol, (L, dtype)
            h.residual_restrict(L, None, bl, rc)
            assert rel(to_cw(h, L - 1, rc), P.T @ br) <= tol
            xf = xl.clone()
            h.prolongate_add(L, to_lib(h, L - 1, e, dtype), xf)
            assert rel(to_cw(h, L, xf), xr + P @ er) <= tol, (L, dtype)
    A0 = ops[0].toarray()
    b0 = uniform(A0.shape[0], seed=34)
    for dtype, tol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
        b0r = np.asarray(torch.tensor(b0, dtype=dtype).double())
        x0 = torch.empty(A0.shape[0], dtype=dtype, device="cuda")
        h.coarse_solve(to_lib(h, 0, b0, dtype), x0)
        ref = np.linalg.solve(A0, b0r)
        # fp32: the solve is exact up to rounding, so its relative error is bounded by
        # cond(A_0) times the unit roundoff (first-order perturbation bound); 1e-5 where
        # that is smaller (cond(A_0): 12 for 2D k=1 ... 870 for 3D k=7)
        if dtype == torch.float32:
            tol = max(1e-5, np.linalg.cond(A0) * 2.0 ** -24)
        assert rel(to_cw(h, 0, x0), ref) <= tol, dtype


@pytest.mark.parametrize("case", [(2, 2, 4, None), (2, 7, 3, None), (3, 3, 3, None), (3, 2, 3, (2, 1, 2))],
                         ids=["d2k2", "d2k7", "d3k3", "d3k2c212"])
@pytest.mark.parametrize("vprec", [0, 1], ids=["fp64", "fp32"])
def test_vcycle(case, vprec):
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle(dim, k, nl, coarse, vprec)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    V = multigrid.VCycle(dim, k, nl, n0=coarse, operators=ops)
    L = nl - 1
    r = uniform(ops[L].shape[0], seed=41)
    z = torch.empty(len(r), dtype=torch.float64, device="cuda")
    h.vcycle(to_lib(h, L, r), z)
    tol = 1e-12 if vprec == 0 else 1e-5
    assert rel(to_cw(h, L, z), V(r)) <= tol


@pytest.mark.parametrize("case", [(2, 3, 4), (3, 3, 3)], ids=["d2k3", "d3k3"])
@pytest.mark.parametrize("vprec", [0, 1], ids=["fp64", "fp32"])
@pytest.mark.parametrize("smk", [0, 1], ids=["mult", "add"])
def test_vcycle_additive_and_multiplicative(smk, vprec, case):
    """Both smoother kinds (C5: additive vs multiplicative), fp64 V-cycle at 1e-12 and
    the fp32 V-cycle at 1e-5 against the fp64 oracle."""
    _need_gpu()
    dim, k, nl = case
    h = handle(dim, k, nl, None, vprec, smk)
    levels, ops = oracle_levels(dim, k, nl)
    V = multigrid.VCycle(dim, k, nl, operators=ops, smoother="additive" if smk else "multiplicative")
    r = uniform(ops[-1].shape[0], seed=42)
    z = torch.empty(len(r), dtype=torch.float64, device="cuda")
    h.vcycle(to_lib(h, nl - 1, r), z)
    assert rel(to_cw(h, nl - 1, z), V(r)) <= (1e-12 if vprec == 0 else 1e-5)


@pytest.mark.parametrize("case", [(2, 2, 3, None), (2, 5, 4, None), (3, 2, 3, None), (3, 4, 2, None)],
                         ids=["C1_d2k2", "d2k5", "d3k2", "d3k4"])
@pytest.mark.parametrize("vprec", [0, 1], ids=["fp64", "mixed"])
def test_cg_solve(case, vprec):
    """GMG-CG on f == 1: iterations +-1, solution vs the oracle."""
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle(dim, k, nl, coarse, vprec)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    V = multigrid.VCycle(dim, k, nl, n0=coarse, operators=ops,
                         dtype=np.float64 if vprec == 0 else np.float32)
    L = nl - 1
    b = assemble.rhs(levels[L], k)
    xo, hist, conv = krylov.pcg(ops[L], b, V, rtol=1e-8)
    bl = torch.empty(len(b), dtype=torch.float64, device="cuda")
    h.rhs(L, bl)
    assert rel(to_cw(h, L, bl), b) <= 1e-14            # rhs kernel vs oracle quadrature
    x = torch.empty_like(bl)
    res = h.cg_solve(bl, x, rtol=1e-8, max_it=50)
    assert res["converged"] and conv
    assert abs(res["iterations"] - (len(hist) - 1)) <= 1
    tol = 1e-12 if vprec == 0 else 1e-6
    if res["iterations"] == len(hist) - 1:
        assert rel(to_cw(h, L, x), xo) <= tol
    # true residual of the GPU solution, evaluated by the oracle
    xg = to_cw(h, L, x)
    assert np.linalg.norm(b - ops[L] @ xg) <= 1.5e-8 * np.linalg.norm(b)


@pytest.mark.parametrize("case", [(2, 2, 3, None), (2, 5, 4, None), (3, 2, 3, None), (3, 3, 3, None)],
                         ids=["C1_d2k2", "d2k5", "d3k2", "d3k3"])
@pytest.mark.parametrize("vprec", [0, 1], ids=["fp64", "mixed"])
def test_gmres_solve(case, vprec):
    """NEXT-2: right-preconditioned GMRES (MGS, no restart) against the oracle's
    GMRES (oracle/krylov.py) on f == 1: same iteration count (+-1), the
    least-squares residual history, the solution, and nu."""
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle(dim, k, nl, coarse, vprec)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    V = multigrid.VCycle(dim, k, nl, n0=coarse, operators=ops,
                         dtype=np.float64 if vprec == 0 else np.float32)
    L = nl - 1
    b = assemble.rhs(levels[L], k)
    xo, hist, conv = krylov.gmres(ops[L], b, V, rtol=1e-8)
    bl = torch.empty(len(b), dtype=torch.float64, device="cuda")
    h.rhs(L, bl)
    x = torch.empty_like(bl)
    res = h.gmres_solve(bl, x, rtol=1e-8, max_it=60)
    assert res["converged"] and conv
    assert abs(res["iterations"] - (len(hist) - 1)) <= 1
    m = min(len(hist), len(res["history"]))
    # fp32 V-cycle rounding (~1e-7 relative) enters the Krylov basis in mixed mode
    htol, hatol = (1e-9, 1e-12) if vprec == 0 else (5e-2, 1e-7)
    assert np.allclose(res["history"][:m], hist[:m], rtol=htol, atol=hatol * hist[0])
    assert abs(res["nu"] - krylov.nu(hist)) <= (1e-6 if vprec == 0 else 0.3)
    xg = to_cw(h, L, x)
    if res["iterations"] == len(hist) - 1:
        assert rel(xg, xo) <= (1e-12 if vprec == 0 else 1e-6)
    assert np.linalg.norm(b - ops[L] @ xg) <= 1.5e-8 * np.linalg.norm(b)
    # a second solve reuses the library-owned Krylov basis
    res2 = h.gmres_solve(bl, x, rtol=1e-8, max_it=60)
    assert res2["iterations"] == res["iterations"]


# ---------------------------------------------------------------- Dirichlet kernel (NEXT-1)
@functools.lru_cache(maxsize=None)
def handle_dir(dim, k, nl, coarse=None, vprec=1, post_reverse=1):
    from paper_2405_18982_b200 import ipmg
    return ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=vprec, kernel=ipmg.KERNEL_DIRICHLET,
                       post_smooth_reverse=post_reverse)


DIR_CASES = [(2, 1, 4, None), (2, 2, 4, None), (2, 3, 4, None), (2, 5, 3, None), (2, 7, 3, None),
             (2, 3, 3, (2, 1)), (3, 1, 3, None), (3, 2, 3, None), (3, 3, 2, None), (3, 4, 2, None),
             (3, 7, 2, None), (3, 2, 3, (2, 1, 2))]
DIR_IDS = ["d%dk%dL%d%s" % (c[0], c[1], c[2], "" if c[3] is None else "c" + "".join(map(str, c[3]))) for c in DIR_CASES]


@pytest.mark.parametrize("case", DIR_CASES, ids=DIR_IDS)
def test_dirichlet_smoother_colours_and_step(case):
    """Every colour of Algorithm 1 with the Dirichlet kernel (patch-only residual,
    reduced local space) against the oracle's dense local solves of the
    extracted A[V_j, V_j]; fp64 1e-12, fp32 1e-5 (on fp32-rounded inputs)."""
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle_dir(dim, k, nl, coarse)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    L = nl - 1
    S = smoother.PatchSmoother(levels[L], k, ops[L], kernel="dirichlet")
    x = uniform(ops[L].shape[0], seed=31)
    b = uniform(ops[L].shape[0], seed=32)
    for dtype, tol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
        xr = np.asarray(torch.tensor(x, dtype=dtype).double())
        br = np.asarray(torch.tensor(b, dtype=dtype).double())
        xl, bl = to_lib(h, L, x, dtype), to_lib(h, L, b, dtype)
        for c in range(2 ** dim):
            out = torch.empty_like(xl)
            h.smooth_colour(L, xl, bl, out, c)
            assert rel(to_cw(h, L, out), S.colour_step_dirichlet(c, xr, br)) <= tol, (c, dtype)
        out = torch.empty_like(xl)
        h.smooth_colour(L, None, bl, out, 0)
        assert rel(to_cw(h, L, out), S.colour_step_dirichlet(0, np.zeros_like(xr), br)) <= tol
        for rev in (False, True):
            xs = xl.clone()
            h.smooth(L, xs, bl, reverse=rev)
            assert rel(to_cw(h, L, xs), S.smooth(xr, br, reverse=rev)) <= tol, (rev, dtype)


@pytest.mark.parametrize("case", [(2, 3, 4, None), (3, 2, 3, None), (3, 4, 2, None)], ids=["d2k3", "d3k2", "d3k4"])
@pytest.mark.parametrize("vprec", [0, 1], ids=["fp64", "fp32"])
def test_dirichlet_vcycle_and_gmres(case, vprec):
    _need_gpu()
    dim, k, nl, coarse = case
    h = handle_dir(dim, k, nl, coarse, vprec)
    levels, ops = oracle_levels(dim, k, nl, coarse)
    L = nl - 1
    V = multigrid.VCycle(dim, k, nl, n0=coarse, operators=ops, kernel="dirichlet",
                         dtype=np.float64 if vprec == 0 else np.float32)
    r = uniform(ops[L].shape[0], seed=33)
    z = torch.empty(len(r), dtype=torch.float64, device="cuda")
    h.vcycle(to_lib(h, L, r), z)
    assert rel(to_cw(h, L, z), V(r)) <= (1e-12 if vprec == 0 else 1e-5)
    b = assemble.rhs(levels[L], k)
    xo, hist, conv = krylov.gmres(ops[L], b, V, rtol=1e-8)
    bl = torch.empty(len(b), dtype=torch.float64, device="cuda")
    h.rhs(L, bl)
    x = torch.empty_like(bl)
    res = h.gmres_solve(bl, x, rtol=1e-8, max_it=80)
    assert res["converged"] and conv
    assert abs(res["iterations"] - (len(hist) - 1)) <= 1
    xg = to_cw(h, L, x)
    assert np.linalg.norm(b - ops[L] @ xg) <= 1.5e-8 * np.linalg.norm(b)


# ---------------------------------------------------------------- Hermite basis / clamped kernel (NEXT-3)
@functools.lru_cache(maxsize=None)
def handle_herm(dim, k, nl, kernel, vprec=1, post_reverse=1):
    from paper_2405_18982_b200 import ipmg
    return ipmg.Handle(dim, k, nl, vcycle_precision=vprec, kernel=kernel, basis=ipmg.BASIS_HERMITE,
                       post_smooth_reverse=post_reverse)


@functools.lru_cache(maxsize=None)
def oracle_herm(dim, k, nl):
    levels = mesh.hierarchy(dim, nl)
    return levels, [assemble.assemble(lv, k, kind="hermite") for lv in levels]


HERM_CASES = [(2, 3, 4), (2, 5, 3), (2, 7, 3), (3, 3, 3), (3, 4, 2), (3, 6, 2)]
HERM_IDS = ["d%dk%dL%d" % c for c in HERM_CASES]


@pytest.mark.parametrize("case", HERM_CASES, ids=HERM_IDS)
def test_hermite_vmult_and_rhs(case):
    """The Hermite-type basis through the same kernels: operator (1e-12 fp64,
    1e-5 fp32) and f == 1 right-hand side against the oracle's Hermite assembly."""
    _need_gpu()
    from paper_2405_18982_b200 import ipmg
    dim, k, nl = case
    h = handle_herm(dim, k, nl, ipmg.KERNEL_FULL)
    levels, ops = oracle_herm(dim, k, nl)
    for level in range(1, nl):
        A = ops[level]
        x = uniform(A.shape[0], seed=41 + level)
        for dtype, tol in ((torch.float64, 1e-12), (torch.float32, 1e-5)):
            xr = np.asarray(torch.tensor(x, dtype=dtype).double())
            y = torch.empty(len(x), dtype=dtype, device="cuda")
            h.vmult(level, to_lib(h, level, x, dtype), y)
            assert rel(to_cw(h, level, y), A @ xr) <= tol, (level, dtype)
    L = nl - 1
    b = torch.empty(ops[L].shape[0], dtype=torch.float64, device="cuda")
    h.rhs(L, b)
    assert rel(to_cw(h, L, b), assemble.rhs(levels[L], k, kind="hermite")) <= 1e-13


def _local_matrix(S, colour):
    """Dense local matrix of the first patch group of a colour (oracle)."""
    lu, iI, iP, AIP = S.groups[colour][0]
    mask = np.isin(iP[0], iI[0])
    return AIP[:, mask]


@pytest.mark.parametrize("case", HERM_CASES, ids=HERM_IDS)
def test_clamped_smoother_colours_and_step(case):
    _need_gpu()
    from paper_2405_18982_b200 import ipmg
    dim, k, nl = case
    h = handle_herm(dim, k, nl, ipmg.KERNEL_CLAMPED)
    levels, ops = oracle_herm(dim, k, nl)
    L = nl - 1
    S = smoother.PatchSmoother(levels[L], k, ops[L], kernel="clamped")
    x = uniform(ops[L].shape[0], seed=51)
    b = uniform(ops[L].shape[0], seed=52)
    # The Hermite-type basis is far worse conditioned than GLL Lagrange (cond(A_j)
    # ~7e4 at k=3, ~2e9 at k=7, vs 70 / 580): the two independent basis
    # constructions agree to 1e-12 in the operator (test above) and the local
    # solves amplify that by cond(A_j), so the bars scale with it.
    cnd = np.linalg.cond(_local_matrix(S, 0))
    tols = ((torch.float64, max(1e-12, 1e-19 * cnd)), (torch.float32, max(1e-5, 1e-11 * cnd)))
    for dtype, tol in tols:
        xr = np.asarray(torch.tensor(x, dtype=dtype).double())
        br = np.asarray(torch.tensor(b, dtype=dtype).double())
        xl, bl = to_lib(h, L, x, dtype), to_lib(h, L, b, dtype)
        for c in range(2 ** dim):
            out = torch.empty_like(xl)
            h.smooth_colour(L, xl, bl, out, c)
            assert rel(to_cw(h, L, out), S.colour_step_dirichlet(c, xr, br)) <= tol, (c, dtype)
        for rev in (False, True):
            xs = xl.clone()
            h.smooth(L, xs, bl, reverse=rev)
            assert rel(to_cw(h, L, xs), S.smooth(xr, br, reverse=rev)) <= tol, (rev, dtype)


@pytest.mark.parametrize("kernel", ["full", "clamped"])
@pytest.mark.parametrize("case", [(2, 3, 4), (3, 3, 3), (3, 5, 2)], ids=["d2k3", "d3k3", "d3k5"])
def test_hermite_vcycle_and_solvers(case, kernel):
    """V-cycle (1e-12 fp64) and GMRES / CG iteration counts against the oracle
    on the Hermite-type basis, for the full and the clamped kernel."""
    _need_gpu()
    from paper_2405_18982_b200 import ipmg
    dim, k, nl = case
    kern = ipmg.KERNEL_CLAMPED if kernel == "clamped" else ipmg.KERNEL_FULL
    h = handle_herm(dim, k, nl, kern, 0, 0)
    levels, ops = oracle_herm(dim, k, nl)
    L = nl - 1
    V = multigrid.VCycle(dim, k, nl, operators=ops, kernel=kernel, basis_kind="hermite", post_reverse=False)
    r = uniform(ops[L].shape[0], seed=53)
    z = torch.empty(len(r), dtype=torch.float64, device="cuda")
    h.vcycle(to_lib(h, L, r), z)
    assert rel(to_cw(h, L, z), V(r)) <= 1e-10   # Hermite conditioning, see test_clamped_smoother_colours_and_step
    b = assemble.rhs(levels[L], k, kind="hermite")
    bl = torch.empty(len(b), dtype=torch.float64, device="cuda")
    h.rhs(L, bl)
    xo, hist, conv = krylov.gmres(ops[L], b, V, rtol=1e-8)
    x = torch.empty_like(bl)
    res = h.gmres_solve(bl, x, rtol=1e-8, max_it=100)
    assert res["converged"] and conv and abs(res["iterations"] - (len(hist) - 1)) <= 1
    assert np.linalg.norm(b - ops[L] @ to_cw(h, L, x)) <= 1.5e-8 * np.linalg.norm(b)
