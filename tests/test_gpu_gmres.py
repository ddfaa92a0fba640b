"""N1 parity: bf16x_gesv_gmres_ir (GMRES-IR, P:408 / P:491-493) and bf16x_getrf against the
oracle's gmres_ir / getrf on the same seeded inputs.  The GPU's factors and Krylov sums differ
from the oracle's in rounding order (R23, R25), so the comparison is: the same convergence
decision, outer iterations within 1, Arnoldi steps within a band, and forward errors at the
FP64 conditioning level; the factorisation is compared element by element (same pivots) and
by its backward error ||PA - LU|| / ||A||."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu


def _gmres(A, b, variant=3, nb=64, restart=200, inner_tol=1e-10, max_iter=30):
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    bd = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    x, rep, hist = bx.gesv_gmres_ir(Ad, bd, variant=variant, nb=nb, restart=restart, inner_tol=inner_tol,
                                    max_iter=max_iter)
    return x.cpu().numpy(), rep, hist


def _perm(ipiv, n):
    p = np.arange(n)
    for j, q in enumerate(ipiv):
        p[[j, q]] = p[[q, j]]
    return p


def _backward_error(A, LU, ipiv):
    n = A.shape[0]
    L = np.tril(LU.astype(np.float64), -1) + np.eye(n)
    U = np.triu(LU.astype(np.float64))
    return np.linalg.norm(A.astype(np.float64)[_perm(ipiv, n)] - L @ U) / np.linalg.norm(A.astype(np.float64))


def test_identity_one_step():
    n = 300
    A = np.eye(n, dtype=np.float32, order="F")
    b = synthetic.rhs(n, seed=1)
    x, rep, hist = _gmres(A, b)
    assert rep.converged == 1 and rep.iterations == 1 and rep.inner_iterations == 1
    np.testing.assert_allclose(x, b, rtol=4e-16, atol=0)


def test_zero_rhs():
    A = synthetic.diagdom(100, seed=2)
    x, rep, _ = _gmres(A, np.zeros(100))
    assert rep.converged == 1 and rep.iterations == 0 and np.array_equal(x, np.zeros(100))


@pytest.mark.parametrize("variant", [3, 6])
@pytest.mark.parametrize("kappa", [1e2, 1e4, 1e6, 1e8])
def test_conditioned_vs_oracle(orc, kappa, variant):
    n = 384
    A, _ = synthetic.conditioned(n, kappa, seed=int(np.log10(kappa)) + 60)
    x_true = synthetic.rhs(n, seed=8)
    b = A.astype(np.float64) @ x_true
    x, rep, hist = _gmres(A, b, variant=variant, nb=64)
    ro = orc.gmres_ir(A, b, variant=variant, nb=64)
    assert bool(rep.converged) == bool(ro["converged"]), (rep.converged, ro["converged"], list(hist), ro["history"])
    assert rep.converged == 1
    xref = np.linalg.solve(A.astype(np.float64), b)
    k2 = np.linalg.cond(A.astype(np.float64))
    bound = 50 * k2 * 2.0 ** -53 * np.max(np.abs(xref))
    assert np.max(np.abs(x - xref)) <= bound
    assert np.max(np.abs(ro["x"] - xref)) <= bound
    assert abs(rep.iterations - ro["iterations"]) <= 1
    # Arnoldi steps per GMRES cycle (R25: one cycle per outer correction): with equal outer counts
    # this is the total; when the outer counts differ by the allowed one, the extra cycle's steps
    # are not a difference in the Krylov convergence (kappa 1e6 x6: oracle 1 x 5 steps, GPU with
    # the short-k promote-every-MMA trailing updates 2 x 5)
    gi, oi = rep.inner_iterations / max(rep.iterations, 1), ro["inner_iterations"] / max(ro["iterations"], 1)
    assert abs(gi - oi) <= max(3, 0.25 * oi), (rep.iterations, rep.inner_iterations, ro["iterations"], ro["inner_iterations"])
    assert len(hist) == rep.iterations + 1 and hist[0] == np.max(np.abs(b))


def test_gmres_ir_converges_where_lu_ir_fails():
    n = 512
    A, _ = synthetic.conditioned(n, 1e8, seed=71)
    x_true = synthetic.rhs(n, seed=9)
    b = A.astype(np.float64) @ x_true
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    bd = torch.from_numpy(b).cuda()
    _, rir, _ = bx.gesv_ir(Ad, bd, variant=3, nb=64)
    x, rep, _ = _gmres(A, b, variant=3, nb=64, restart=512)
    assert rir.converged == 0 and rep.converged == 1
    r = A.astype(np.float64) @ x - b
    assert np.max(np.abs(r)) <= rep.tol * (1 + 1e-12)


@pytest.mark.parametrize("restart", [5, 20])
def test_short_restart_still_converges(orc, restart):
    """Short cycles: more outer corrections, same answer (diag dominant, well conditioned)."""
    n = 640
    A = synthetic.diagdom(n, seed=11)
    x_true = synthetic.rhs(n, seed=12)
    b = A.astype(np.float64) @ x_true
    x, rep, _ = _gmres(A, b, variant=3, nb=128, restart=restart)
    ro = orc.gmres_ir(A, b, variant=3, nb=128, restart=restart)
    assert rep.converged == 1 and ro["converged"]
    assert np.linalg.norm(x - x_true) / np.linalg.norm(x_true) < 1e-12
    assert abs(rep.iterations - ro["iterations"]) <= 1


# ------------------------------------------------------------------------------------
# bf16x_getrf
# ------------------------------------------------------------------------------------
@pytest.mark.parametrize("variant", [3, 6, 9])
@pytest.mark.parametrize("n,nb", [(300, 64), (700, 128)])
def test_getrf_vs_oracle(orc, n, nb, variant):
    A = synthetic.uniform(n, n, seed=n + variant)
    LU, ipiv, info = bx.getrf(torch.from_numpy(A).cuda(), variant=variant, nb=nb)
    LU = LU.cpu().numpy()
    ipiv = ipiv.cpu().numpy()
    LUo, ipo, info_o = orc.getrf(A, variant=variant, nb=nb)
    assert info == 0 and info_o == 0
    assert np.array_equal(ipiv, ipo)
    be_g = _backward_error(A, LU, ipiv)
    be_o = _backward_error(A, LUo, ipo)
    u = 2.0 ** -24
    assert be_g <= max(2 * be_o, n * u), (be_g, be_o)
    # same pivots: factors agree to the factorisation's own error level
    assert np.linalg.norm(LU.astype(np.float64) - LUo) / np.linalg.norm(LUo) <= 1e3 * be_o


def test_getrf_large_backward_error():
    n = 4096
    A = synthetic.uniform(n, n, seed=5)
    LU, ipiv, info = bx.getrf(torch.from_numpy(A).cuda(), variant=6, nb=256)
    assert info == 0
    # ||PA - LU||_F / ||A||_F on the GPU in FP64
    Ad = torch.from_numpy(A).cuda().double()
    L = torch.tril(LU.double(), -1) + torch.eye(n, device="cuda", dtype=torch.float64)
    U = torch.triu(LU.double())
    p = torch.from_numpy(_perm(ipiv.cpu().numpy(), n)).cuda()
    be = float(torch.linalg.norm(Ad[p] - L @ U) / torch.linalg.norm(Ad))
    # FP32-LU level: the oracle's x6 LU measures 0.024 n u at n = 2048 (FP32 SGETRF 0.045 n u)
    assert be < 0.05 * n * 2.0 ** -24, be


def test_getrf_singular_and_empty():
    n = 64
    A = synthetic.uniform(n, n, seed=3)
    A[:, 10] = 0.0
    _, _, info = bx.getrf(torch.from_numpy(A).cuda(), variant=3, nb=32)
    assert info == 11
    LU, ipiv, info = bx.getrf(torch.zeros(0, 0, device="cuda"), variant=3)
    assert info == 0 and LU.numel() == 0
