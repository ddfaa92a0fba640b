"""Pins for the oracle's GMRES and GMRES-IR (N1; section III, section IV-B).

What fixes GMRES independently of its code:
  * the identity system is solved in one step, exactly;
  * Krylov theory: for A = diag(d) with exactly k distinct values (and M = I), the Krylov
    space has dimension k, so GMRES reaches the exact solution at step k and not before;
  * optimality: after j steps the preconditioned residual is the minimum of
    ||z - B K_j y||_2 over the Krylov space (B = M^-1 A, z = M^-1 b), computed here by brute
    force with a library least-squares solve on an explicitly built Krylov basis;
  * GMRES-IR converges where LU-IR with the same bf16x3 factors does not (the point of P:408)
    and its answer agrees with LAPACK's FP64 solve to the conditioning bound.
The paper's GMRES table is for single-BF16 / FP16 LU preconditioners on
diagonally dominant matrices whose generator and residual norm it does not state: its
iteration counts are *parity unpinned* (reading R25).
"""
import numpy as np
import pytest

import synthetic


def _ident(v):
    return v


def test_identity_one_step(orc):
    b = np.arange(1.0, 12.0)
    g = orc.gmres(_ident, _ident, b, restart=11, tol=1e-14)
    assert g["iterations"] == 1 and g["converged"]
    np.testing.assert_allclose(g["x"], b, rtol=4e-16, atol=0)   # x = V y = (b / beta) * beta


@pytest.mark.parametrize("k", [1, 2, 3, 4, 6])
def test_distinct_eigenvalues_terminate_at_k(orc, k):
    n = 40
    rng = np.random.Generator(np.random.PCG64(k))
    vals = np.linspace(1.0, 3.0, k) if k > 1 else np.array([2.0])
    d = vals[np.arange(n) % k]
    b = rng.standard_normal(n)
    g = orc.gmres(lambda v: d * v, _ident, b, restart=n, tol=1e-12)
    assert g["converged"] and g["iterations"] == k, (g["iterations"], g["history"])
    if k > 1:
        assert g["history"][k - 2] > 1e-6 * np.linalg.norm(b)
    np.testing.assert_allclose(g["x"], b / d, rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("j", [1, 2, 3, 5])
def test_residual_minimal_over_krylov_space(orc, j):
    n = 30
    rng = np.random.Generator(np.random.PCG64(100 + j))
    A = np.eye(n) + 0.4 * rng.standard_normal((n, n)) / np.sqrt(n)
    Mdiag = 1.0 + rng.uniform(0, 1, n)
    b = rng.standard_normal(n)
    matvec = lambda v: A @ v
    psolve = lambda v: v / Mdiag
    g = orc.gmres(matvec, psolve, b, restart=j, tol=0.0, max_cycles=1)
    assert g["iterations"] == j
    # brute force: min over y of || z - B K y ||, K = [z, Bz, ..., B^{j-1} z] (columns normalised)
    B = A / Mdiag[:, None]
    z = b / Mdiag
    K = np.empty((n, j))
    v = z.copy()
    for c in range(j):
        K[:, c] = v / np.linalg.norm(v)
        v = B @ K[:, c]
    y, *_ = np.linalg.lstsq(B @ K, z, rcond=None)
    rmin = np.linalg.norm(z - B @ (K @ y))
    ractual = np.linalg.norm(psolve(b - matvec(g["x"])))
    assert abs(ractual - rmin) <= 1e-9 * np.linalg.norm(z), (ractual, rmin)
    assert abs(g["history"][-1] - rmin) <= 1e-9 * np.linalg.norm(z)
    # the rotated estimates are non-increasing (minimisation over nested spaces)
    h = g["history"]
    assert all(h[i + 1] <= h[i] * (1 + 1e-12) for i in range(len(h) - 1))


def test_restart_continues_from_iterate(orc):
    """Restarted cycles: GMRES(2) with enough cycles solves a well-conditioned system."""
    n = 25
    rng = np.random.Generator(np.random.PCG64(7))
    A = np.eye(n) + 0.2 * rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    g = orc.gmres(lambda v: A @ v, _ident, b, restart=2, tol=1e-12, max_cycles=60)
    assert g["converged"]
    np.testing.assert_allclose(A @ g["x"], b, rtol=0, atol=1e-10 * np.linalg.norm(b))


def test_preconditioning_reduces_steps(orc):
    """unpreconditioned GMRES needs more steps than with the bf16x LU factors."""
    n = 100
    A = synthetic.diagdom(n, seed=3)
    b = synthetic.rhs(n, seed=4)
    A64 = A.astype(np.float64)
    LU, ipiv, info = orc.getrf(A, variant=3, nb=32)
    assert info == 0
    kw = dict(restart=n, tol=1e-12, max_cycles=1)
    plain = orc.gmres(lambda v: A64 @ v, _ident, b, **kw)
    pre = orc.gmres(lambda v: A64 @ v, lambda v: orc.lu_solve_f64(LU, ipiv, v), b, **kw)
    assert pre["converged"] and pre["iterations"] < plain["iterations"]


def test_gmres_ir_beats_lu_ir_at_high_kappa(orc):
    n = 200
    A, _ = synthetic.conditioned(n, 1e8, seed=3)
    xt = synthetic.rhs(n, seed=4)
    A64 = A.astype(np.float64)
    b = A64 @ xt
    ir = orc.gesv_ir(A, b, variant=3, nb=64)
    g = orc.gmres_ir(A, b, variant=3, nb=64, restart=200)
    assert not ir["converged"]
    assert g["converged"] and g["inner_iterations"] <= 400
    xref = np.linalg.solve(A64, b)
    kappa = np.linalg.cond(A64)
    assert np.max(np.abs(g["x"] - xref)) <= 50 * kappa * 2.0 ** -53 * np.max(np.abs(xref))
    # the stopping test was met on the true FP64 residual
    r = orc.residual_f64(A, b, g["x"])
    anrm = np.max(np.abs(A64).sum(axis=1))
    assert np.max(np.abs(r)) <= np.sqrt(n) * np.max(np.abs(g["x"])) * anrm * 2.0 ** -53


def test_gmres_ir_identity_and_zero_rhs(orc):
    I = np.eye(9, dtype=np.float32)
    g = orc.gmres_ir(I, np.arange(9.0), variant=3)
    assert g["converged"] and g["iterations"] == 1 and g["inner_iterations"] == 1
    np.testing.assert_allclose(g["x"], np.arange(9.0), rtol=4e-16, atol=0)
    z = orc.gmres_ir(I, np.zeros(9), variant=3)
    assert z["converged"] and z["iterations"] == 0 and np.array_equal(z["x"], np.zeros(9))
