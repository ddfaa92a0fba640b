"""Pins for the oracle's LU + iterative refinement (§III, §IV-A).

Special cases with known answers (identity, permutation, textbook 2x2 pivoting), the
factorisation residual bound ||PA - LU|| = O(n u_w ||A||), and the FP64 solve accuracy on
diagonally dominant systems.  The convergence-versus-kappa statistics are *parity
unpinned*: the paper's IR table is for single-BF16/FP16 LU at n = 50, not for
bf16x3 trailing updates.
"""
import numpy as np
import pytest

import synthetic


def _perm_matrix(ipiv, n):
    p = np.arange(n)
    for j, q in enumerate(ipiv):
        p[[j, q]] = p[[q, j]]
    return p


def _factor_residual(A, LU, ipiv):
    n = A.shape[0]
    L = np.tril(LU.astype(np.float64), -1) + np.eye(n)
    U = np.triu(LU.astype(np.float64))
    p = _perm_matrix(ipiv, n)
    return np.linalg.norm(A.astype(np.float64)[p] - L @ U) / np.linalg.norm(A.astype(np.float64))


def test_identity_and_2x2_pivot(orc):
    """identity -> L = U = I, no swaps; [[0,1],[1,0]] -> one row swap."""
    I = np.eye(7, dtype=np.float32)
    LU, ipiv, info = orc.getrf(I, variant=3, nb=3)
    assert info == 0 and np.array_equal(LU, I) and list(ipiv) == list(range(7))
    S = np.array([[0, 1], [1, 0]], dtype=np.float32)
    LU, ipiv, info = orc.getrf(S, variant=6, nb=1)
    assert info == 0 and list(ipiv) == [1, 1] and np.array_equal(LU, np.eye(2, dtype=np.float32))
    r = orc.gesv_ir(I, np.arange(7.0), variant=3)
    assert r["converged"] and r["iterations"] == 0 and np.array_equal(r["x"], np.arange(7.0))


def test_singular_reports_column(orc):
    A = np.ones((4, 4), dtype=np.float32)
    _, _, info = orc.getrf(A, variant=6, nb=2)
    assert info == 2   # column 2 (1-based) has an exact zero pivot after one step


@pytest.mark.parametrize("variant,tol", [(0, 2.0 ** -24), (6, 2.0 ** -24), (9, 2.0 ** -24), (3, 2.0 ** -16)])
def test_factorisation_residual(orc, variant, tol):
    """||P A - L U||_F / ||A||_F = O(n u) with u the unit roundoff of the trailing-update
    arithmetic: FP32-like for SGETRF (0) and the 6/9-product splits, 2^-16 for bf16x3."""
    n = 96
    A = synthetic.uniform(n, n, seed=21)
    LU, ipiv, info = orc.getrf(A, variant=variant, nb=16)
    assert info == 0
    res = _factor_residual(A, LU, ipiv)
    assert res <= 4 * n * tol
    assert np.all(np.abs(np.tril(LU, -1)) <= 1.0)        # partial pivoting: |l_ij| <= 1


def test_fp64_solve_diag_dominant(orc):
    """diagonally dominant 50x50 with FP32 factors and FP64 refinement reaches an FP64
    residual ||b - A x|| / ||b|| < 1e-12."""
    n = 50
    A = synthetic.diagdom(n, seed=5)
    x_true = synthetic.rhs(n, seed=6)
    b = A.astype(np.float64) @ x_true
    for v in (0, 3, 6):
        r = orc.gesv_ir(A, b, variant=v, nb=16)
        assert r["converged"]
        assert np.linalg.norm(b - A.astype(np.float64) @ r["x"]) / np.linalg.norm(b) < 1e-12
        assert np.linalg.norm(r["x"] - x_true) / np.linalg.norm(x_true) < 1e-12


def test_ir_convergence_vs_kappa(orc):
    """Parity unpinned (see module doc).  Model expectation: bf16x3-LU + IR
    converges for kappa = 1e2 and the FP64 forward error approaches kappa * 2^-53; with
    kappa = 1e9 the bf16x3 factors are too inaccurate and IR must not claim convergence to a
    wrong answer."""
    n = 128
    A, _ = synthetic.conditioned(n, 1e2, seed=8)
    x_true = synthetic.rhs(n, seed=9)
    b = A.astype(np.float64) @ x_true
    r = orc.gesv_ir(A, b, variant=3, nb=32)
    assert r["converged"] and r["iterations"] <= 10
    assert np.linalg.norm(r["x"] - x_true) / np.linalg.norm(x_true) < 1e-11
    A, _ = synthetic.conditioned(n, 1e9, seed=10)
    b = A.astype(np.float64) @ x_true
    r = orc.gesv_ir(A, b, variant=3, nb=32)
    if r["converged"]:
        assert np.linalg.norm(b - A.astype(np.float64) @ r["x"]) <= 1e-9 * np.linalg.norm(b)
