"""N4 pins: the fully 16-bit LU + refinement experiment (§IV-B; reading R28).

* binary16 conversion: exhaustive round trip of every finite pattern, the format's special
  values, ties to even, and agreement with numpy's float16 conversion (a library routine);
* the 16-bit elimination: identity, representability of every stored entry, exactness on
  integer factors whose elimination never leaves the format, FP32 backward error;
* the refinement loop: the identity system, and the precision ordering the paper reports
  (FP32 converges at least as often and in fewer iterations than FP16, FP16 than BF16).
The paper's percentages themselves are *parity unpinned* (its matrix generator and pivoting
are not stated; R28 lists the readings tried)."""
import numpy as np
import pytest

import synthetic


def test_fp16_exhaustive_roundtrip_and_specials(orc):
    for h in range(65536):
        f = orc.fp16_widen(h)
        if np.isnan(f):
            continue
        assert orc.fp16_round(f) == h, hex(h)
    assert orc.fp16_round(1.0) == 0x3C00
    assert orc.fp16_round(65504.0) == 0x7BFF
    assert orc.fp16_round(65520.0) == 0x7C00              # tie at the top rounds to even = Inf
    assert orc.fp16_round(2.0 ** -25) == 0x0000           # half of the smallest subnormal: to even
    assert orc.fp16_round(3 * 2.0 ** -26) == 0x0001
    assert orc.fp16_round(1 + 2.0 ** -11) == 0x3C00       # tie, even stays
    assert orc.fp16_round(1 + 3 * 2.0 ** -11) == 0x3C02   # tie, odd rounds up
    assert orc.fp16_round(-2.0) == 0xC000


def test_fp16_matches_numpy(orc):
    g = np.random.default_rng(7)
    x = (g.standard_normal(30000) * np.exp2(g.integers(-30, 18, 30000))).astype(np.float32)
    with np.errstate(over="ignore"):
        ref = x.astype(np.float16).view(np.uint16)
    got = np.array([orc.fp16_round(v) for v in x], dtype=np.uint16)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("fmt", ["fp32", "bf16", "fp16"])
def test_getrf16_identity_and_representable(orc, fmt):
    I = np.eye(9, dtype=np.float32)
    LU, ipiv, info = orc.getrf16(I, fmt=fmt)
    assert info == 0 and np.array_equal(LU, I) and list(ipiv) == list(range(9))
    A, _ = synthetic.conditioned(40, 100.0, seed=3)
    LU, ipiv, info = orc.getrf16(A, fmt=fmt)
    assert info == 0
    if fmt == "bf16":
        assert np.array_equal(LU, orc.widen(orc.split(LU)[0]))
    if fmt == "fp16":
        assert all(orc.fp16_widen(orc.fp16_round(v)) == v for v in LU.ravel())


@pytest.mark.parametrize("fmt", ["fp32", "bf16", "fp16"])
def test_getrf16_exact_integer_factors(orc, fmt):
    """A = L U with small integer entries (|.| <= 8) and L's multipliers in {-1, 0, 1}: without
    pivoting every intermediate value is an integer below 256, exact in all three formats."""
    g = np.random.default_rng(11)
    n = 12
    L = np.tril(g.integers(-1, 2, (n, n)), -1) + np.eye(n, dtype=np.int64)
    U = np.triu(g.integers(-3, 4, (n, n)))
    np.fill_diagonal(U, g.choice([1, 2], n))
    A = (L @ U).astype(np.float32)
    assert np.abs(A).max() < 256
    LU, ipiv, info = orc.getrf16(A, fmt=fmt, pivot=False)
    assert info == 0
    assert np.array_equal(np.tril(LU, -1), np.tril(L, -1).astype(np.float32))
    assert np.array_equal(np.triu(LU), U.astype(np.float32))


def test_getrf16_fp32_backward_error(orc):
    n = 50
    A, _ = synthetic.conditioned(n, 1e3, seed=4)
    LU, ipiv, info = orc.getrf16(A, fmt="fp32")
    p = orc.row_permutation(ipiv)
    L = np.tril(LU.astype(np.float64), -1) + np.eye(n)
    U = np.triu(LU.astype(np.float64))
    be = np.linalg.norm(A.astype(np.float64)[p] - L @ U) / np.linalg.norm(A.astype(np.float64))
    assert be < n * 2.0 ** -24


def test_gesv16_identity(orc):
    b = np.arange(1.0, 8.0)
    r = orc.gesv16_ir(np.eye(7, dtype=np.float32), b, fmt="bf16", tol=2.0 ** -53)
    assert r["converged"] and r["iterations"] == 0 and np.array_equal(r["x"], b)


def test_gesv16_precision_ordering(orc):
    """'the lower the precision, the more stringent conditioning is needed' and the
    table's ordering FP32 < FP16 < BF16 in iterations, FP32 >= FP16 >= BF16 in convergence."""
    n, trials = 50, 20
    for kappa in (10.0, 1e3):
        conv, its = {}, {}
        for fmt in ("fp32", "fp16", "bf16"):
            c, it = 0, []
            for s in range(trials):
                A, _ = synthetic.conditioned(n, kappa, seed=s)
                b = A.astype(np.float64) @ synthetic.rhs(n, seed=s + 1000)
                r = orc.gesv16_ir(A, b, fmt=fmt, tol=kappa * 2.0 ** -53, max_iter=100)
                c += r["converged"]
                if r["converged"]:
                    it.append(r["iterations"])
            conv[fmt], its[fmt] = c, (np.mean(it) if it else np.inf)
        assert conv["fp32"] >= conv["fp16"] >= conv["bf16"], conv
        assert its["fp32"] < its["fp16"] < its["bf16"], its


def _diagdom_rc(n, seed):
    """Row- and column-diagonally dominant unsymmetric matrix ("row and column
    diagonally dominant unsymmetric matrices"): off-diagonal U[-1, 1], diagonal +-(max of the
    row and column absolute sums + 1)."""
    g = np.random.Generator(np.random.PCG64([seed, 8]))
    A = g.uniform(-1.0, 1.0, (n, n))
    np.fill_diagonal(A, 0.0)
    d = np.maximum(np.abs(A).sum(axis=0), np.abs(A).sum(axis=1)) + 1.0
    A[np.arange(n), np.arange(n)] = d * np.where(g.uniform(-1.0, 1.0, n) < 0, -1.0, 1.0)
    return np.asfortranarray(A.astype(np.float32))


def test_gmres_with_16bit_preconditioner_table_ordering(orc):
    """P:491-506 second table: GMRES preconditioned by the single-16-bit LU converges on
    diagonally dominant systems for every preconditioner precision, in fewer iterations the
    more precise the factors (FP32 < FP16 < BF16).  Counts themselves: parity unpinned (the
    paper's 2.0 / 5.0 / 7.0 at n = 50 depend on its unstated residual norm; ours: ~4 / 8 / 11)."""
    for n in (10, 50):
        its = {}
        for fmt in ("fp32", "fp16", "bf16"):
            it = []
            for t in range(20):
                A = _diagdom_rc(n, t)
                A64 = A.astype(np.float64)
                b = np.random.Generator(np.random.PCG64([t, 9])).standard_normal(n)
                LU, ipiv, info = orc.getrf16(A, fmt=fmt)
                g = orc.gmres(lambda v: A64 @ v, lambda v: orc.lu_solve_f64(LU, ipiv, v), b, restart=n,
                              tol=np.linalg.cond(A64) * 2.0 ** -53, max_cycles=1)
                assert g["converged"] or fmt == "bf16"
                it.append(g["iterations"])
            its[fmt] = np.mean(it)
        assert its["fp32"] < its["fp16"] < its["bf16"], its
