"""CPU tests of the C-ABI library (no GPU): it loads, exports every symbol
include/ipmg.h declares, and its host-side 1D setup agrees with the oracle's
independent quadrature assembly."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT

ipmg = pytest.importorskip("paper_2405_18982_b200.ipmg")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(ipmg.LIB_PATH):
        pytest.fail("libipmg.so not built: run python -c 'import __graft_entry__ as g; g.build()'")
    return ipmg.load()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "ipmg.h")).read()
    declared = set(re.findall(r"\b(ipmg_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(ipmg.EXPORTS), declared ^ set(ipmg.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name


def test_create_rejects_bad_config_without_gpu(lib):
    import ctypes
    cfg = ipmg.Config()
    lib.ipmg_config_default(ctypes.byref(cfg))
    assert cfg.dim == 3 and cfg.degree == 4 and cfg.vcycle_precision == ipmg.FP32
    h = ctypes.c_void_p()
    cfg.dim = 4
    assert lib.ipmg_create(ctypes.byref(cfg), ctypes.byref(h)) == 1          # INVALID_ARG
    cfg.dim, cfg.degree = 2, 9
    assert lib.ipmg_create(ctypes.byref(cfg), ctypes.byref(h)) == 2          # UNSUPPORTED
    assert b"degree" in lib.ipmg_last_error(None)


def _oracle_1d(k, ncell, h=1.0):
    from oracle import assemble, mesh
    return assemble.assemble(mesh.Level(1, [ncell], h), k).toarray()


@pytest.mark.parametrize("k", range(1, 8))
def test_tables_match_oracle(k):
    from oracle import assemble, basis, transfer, mesh
    nc, np_ = k + 1, 2 * (k + 1)
    assert np.allclose(ipmg.tables_1d(k, 0), basis.gll_nodes(nc), atol=1e-14)
    K, M = assemble.Reference(1, k).cell_matrices(1.0)
    assert np.allclose(ipmg.tables_1d(k, 1).reshape(nc, nc), M, atol=1e-13)
    assert np.allclose(ipmg.tables_1d(k, 2).reshape(nc, nc), K, atol=1e-11 * np.abs(K).max())
    # patch matrices = 2-cell blocks of oracle 1D SIPG matrices (unit h):
    # v0 interior both sides: cells 1,2 of 4; v1 low boundary: cells 0,1 of 3;
    # v2 high boundary: cells 1,2 of 3; v3 both: the 2-cell mesh itself.
    blocks = {0: _oracle_1d(k, 4)[nc:3 * nc, nc:3 * nc], 1: _oracle_1d(k, 3)[:2 * nc, :2 * nc],
              2: _oracle_1d(k, 3)[nc:, nc:], 3: _oracle_1d(k, 2)}
    MP = np.kron(np.eye(2), M)
    for v in range(4):
        LP = ipmg.tables_1d(k, 3 + v).reshape(np_, np_)
        assert np.abs(LP - blocks[v]).max() <= 1e-12 * np.abs(blocks[v]).max(), v
        S = ipmg.tables_1d(k, 7 + v).reshape(np_, np_)
        lam = ipmg.tables_1d(k, 11 + v)
        if v == 0:
            # interior patch: reflection-symmetric problem; modes ordered [even | odd]
            h = np_ // 2
            assert np.all(np.diff(lam[:h]) >= 0) and np.all(np.diff(lam[h:]) >= 0)
            assert np.abs(S[::-1, :h] - S[:, :h]).max() <= 1e-14 * np.abs(S).max()
            assert np.abs(S[::-1, h:] + S[:, h:]).max() <= 1e-14 * np.abs(S).max()
        else:
            assert np.all(np.diff(lam) >= 0)
        assert lam.min() > 0
        # generalized eigenpairs of the *oracle's* matrices: L S = M S Lambda, S^T M S = I
        assert np.abs(blocks[v] @ S - MP @ S * lam[None, :]).max() <= 1e-10 * lam.max()
        assert np.abs(S.T @ MP @ S - np.eye(np_)).max() <= 1e-11
    P = transfer.prolongation(mesh.Level(1, [1], 1.0), mesh.Level(1, [2], 0.5), k).toarray()
    assert np.allclose(ipmg.tables_1d(k, 15).reshape(np_, nc), P, atol=1e-13)


def test_penalty_scale_changes_tables():
    a = ipmg.tables_1d(2, 6, 1.0)
    b = ipmg.tables_1d(2, 6, 2.0)
    assert np.abs(a - b).max() > 1.0


@pytest.mark.parametrize("k", [1, 3, 5, 7])
def test_dirichlet_tables_match_oracle(k):
    """Dirichlet kernel (reading A20): the residual patch matrix (outer
    mesh-interior faces dropped) equals the oracle's assembled patch operator
    minus its outer-face terms, and the padded eigenbasis solves the local
    generalized eigenproblem on the kept nodes."""
    from oracle import assemble, mesh
    from oracle.smoother import PatchSmoother
    np_ = 2 * (k + 1)
    lv = mesh.Level(1, [4], 1.0)
    A = assemble.assemble(lv, k)
    S = PatchSmoother(lv, k, A, kernel="dirichlet")
    P = mesh.patch_dofs(lv, [1, 2], k)
    ref = A[P][:, P].toarray() - S._outer_face_terms(((False, False),))
    LPR = ipmg.tables_1d(k, 16).reshape(np_, np_)
    assert np.abs(LPR - ref).max() <= 1e-10 * np.abs(ref).max()
    LP = ipmg.tables_1d(k, 3).reshape(np_, np_)
    SD = ipmg.tables_1d(k, 20).reshape(np_, np_)
    lam = ipmg.tables_1d(k, 24)
    act = ipmg.tables_1d(k, 28)
    assert act.sum() == np_ - 2
    keep = np.arange(1, np_ - 1)
    Mp = np.kron(np.eye(2), assemble.Reference(1, k).cell_matrices(1.0)[1])
    for m in range(np_):
        s = SD[:, m]
        if act[m]:
            assert abs(s[0]) + abs(s[-1]) == 0.0
            res = LP[np.ix_(keep, keep)] @ s[keep] - lam[m] * Mp[np.ix_(keep, keep)] @ s[keep]
            assert np.abs(res).max() <= 1e-9 * max(1.0, lam[m])
            assert abs(s[keep] @ Mp[np.ix_(keep, keep)] @ s[keep] - 1.0) <= 1e-10
    # [even | odd] ordering of the interior variant
    h = np_ // 2
    assert np.allclose(SD[::-1, :h], SD[:, :h], atol=1e-14) and np.allclose(SD[::-1, h:], -SD[:, h:], atol=1e-14)
