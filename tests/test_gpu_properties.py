"""Property tests of the CUDA path at sizes the oracle cannot reach:
the manufactured-solution L2 rate k+1 in 3D, operator symmetry <Ax, y> = <x, Ay> at the
full headline size, and the CG solution against a sparse direct solve at rtol 1e-14.

The manufactured right-hand side (ipmg_rhs kind 1, include/ipmg.h) is pinned against the
oracle's quadrature first; the L2 error is the GLL-quadrature norm of u_h - u at the nodes
(the weights are the kind-0 moments b_i = int phi_i, exact for the GLL Lagrange basis).
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import assemble, basis, mesh  # noqa: E402


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _handle(dim, k, nl, coarse=None, vprec=0):
    from paper_2405_18982_b200 import ipmg
    return ipmg.Handle(dim, k, nl, coarse_cells=coarse, vcycle_precision=vprec)


def _to_cw(h, level, t):
    out = torch.empty_like(t)
    h.to_cellwise(level, t, out)
    torch.cuda.synchronize()
    return out


def _exact_at_nodes(dim, k, n, hcell, ell):
    """u = prod_a sin(pi x_a / ell_a) at the nodes of the cell-wise lexicographic order
    (cells x fastest, nodes x fastest), as a device tensor."""
    nc = k + 1
    xi = torch.tensor(basis.gll_nodes(nc), dtype=torch.float64, device="cuda")
    u = None
    for a in range(dim):
        # coordinate a of (cell, node): cell index along a times h plus the node offset
        ca = torch.arange(n[a], dtype=torch.float64, device="cuda")
        coord = (ca[:, None] + xi[None, :]) * hcell                      # [cell_a, node_a]
        f = torch.sin(np.pi * coord / ell[a])
        # broadcast into [cz, cy, cx, lz, ly, lx] (3D) / [cy, cx, ly, lx] (2D)
        view = [1] * (2 * dim)
        view[dim - 1 - a] = n[a]
        view[2 * dim - 1 - a] = nc
        fa = f.reshape(view)
        u = fa if u is None else u * fa
    return u.reshape(-1)


@pytest.mark.parametrize("case", [(2, 2, 3, None), (3, 2, 2, None), (3, 3, 2, (2, 2, 1))], ids=["d2k2", "d3k2", "d3k3box"])
def test_rhs_kind1_matches_oracle_quadrature(case):
    """ipmg_rhs kind 1 vs the oracle's moments of f = pi^2 (sum_a ell_a^-2) u (Gauss quadrature)."""
    _need_gpu()
    dim, k, nl, coarse = case
    h = _handle(dim, k, nl, coarse)
    L = nl - 1
    lv = mesh.hierarchy(dim, nl, coarse)[L]
    n0 = coarse or (2,) * dim
    ell = [n0[a] * 0.5 for a in range(dim)]
    lam = np.pi ** 2 * sum(1.0 / e ** 2 for e in ell)

    def f(X):   # X: (points, dim)
        v = np.full(X.shape[0], lam)
        for a in range(dim):
            v = v * np.sin(np.pi * X[:, a] / ell[a])
        return v
    ref = assemble.rhs(lv, k, f=f, nq=k + 7)
    b = torch.empty(len(ref), dtype=torch.float64, device="cuda")
    h.rhs(L, b, kind=1)
    got = _to_cw(h, L, b).cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("k,levels", [(2, (4, 5, 6)), (3, (4, 5, 6)), (4, (3, 4, 5))], ids=["k2", "k3", "k4"])
def test_manufactured_l2_rate_3d(k, levels):
    """-Delta u = f on the unit cube, u = prod sin(pi x_a): GMG-CG (fp64) to 1e-13, the
    L2 error converges at order k+1; 3D meshes up to 64^3 cells
    (up to 33M dofs), beyond the oracle's reach."""
    _need_gpu()
    dim = 3
    errs, hs = [], []
    for nl in levels:
        h = _handle(dim, k, nl, None, 0)
        L = nl - 1
        n_dofs, cells, _ = h.level_info(L)
        n = cells[:dim]
        hcell = 1.0 / n[0]
        b = torch.empty(n_dofs, dtype=torch.float64, device="cuda")
        h.rhs(L, b, kind=1)
        x = torch.empty_like(b)
        res = h.cg_solve(b, x, rtol=1e-13, max_it=60)
        assert res["converged"], res
        w = torch.empty_like(b)
        h.rhs(L, w, kind=0)                      # int phi_i: GLL weights times h^d
        xc, wc = _to_cw(h, L, x), _to_cw(h, L, w)
        u = _exact_at_nodes(dim, k, n, hcell, [1.0] * dim)
        errs.append(float(torch.sqrt((wc * (xc - u) ** 2).sum())))
        hs.append(hcell)
        h.close()
    rates = [np.log(errs[i] / errs[i + 1]) / np.log(hs[i] / hs[i + 1]) for i in range(len(errs) - 1)]
    assert rates[-1] >= k + 0.8, (errs, rates)
    assert rates[-1] <= k + 2.5, (errs, rates)


@pytest.mark.parametrize("cfg", [dict(dim=2, k=7, nl=10, coarse=(2, 2)), dict(dim=3, k=4, nl=8, coarse=(2, 2, 1))],
                         ids=["C2", "C4"])
def test_fullsize_operator_symmetry(cfg):
    """<A x, y> = <x, A y> for the fp64 operator at full size (the SIPG form is
    symmetric): relative to ||Ax|| ||y||, 1e-13."""
    _need_gpu()
    h = _handle(cfg["dim"], cfg["k"], cfg["nl"], cfg["coarse"], 1)
    L = cfg["nl"] - 1
    n_dofs, _, _ = h.level_info(L)
    g = torch.Generator(device="cuda").manual_seed(17)
    x = torch.rand(n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y = torch.rand(n_dofs, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    ax = torch.empty_like(x)
    h.vmult(L, x, ax)
    axy = float(torch.dot(ax, y))
    scale = float(torch.linalg.norm(ax)) * float(torch.linalg.norm(y))
    ay = ax
    h.vmult(L, y, ay)
    xay = float(torch.dot(x, ay))
    h.close()
    assert abs(axy - xay) <= 1e-13 * scale, (axy, xay, scale)


@pytest.mark.parametrize("case", [(2, 7, 4), (3, 2, 3)], ids=["d2k7", "d3k2"])
@pytest.mark.parametrize("vprec", [0, 1], ids=["fp64", "mixed"])
def test_cg_vs_sparse_direct(case, vprec):
    """GMG-CG to rtol 1e-13 against a sparse direct solve of the oracle's matrix: the
    difference is bounded by the residual times cond(A), so 1e-9."""
    _need_gpu()
    dim, k, nl = case
    h = _handle(dim, k, nl, None, vprec)
    L = nl - 1
    lv = mesh.hierarchy(dim, nl)[L]
    A = assemble.assemble(lv, k).tocsc()
    b = assemble.rhs(lv, k)
    ref = spla.spsolve(A, b)
    bl = torch.tensor(b, dtype=torch.float64, device="cuda")
    bl2 = torch.empty_like(bl)
    h.from_cellwise(L, bl, bl2)
    x = torch.empty_like(bl2)
    res = h.cg_solve(bl2, x, rtol=1e-13, max_it=200)
    got = _to_cw(h, L, x).cpu().numpy()
    h.close()
    assert res["converged"], res
    assert np.abs(got - ref).max() <= 1e-9 * np.abs(ref).max()
