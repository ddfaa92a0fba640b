"""Pins for the oracle's partial products, bin combination and scaling
(§II-D, §II-E, §II-G, §IV-A).

References used here are independent of the oracle's code: exact FP64 sums (math.fsum of
exactly-representable products), numpy's sequential float32 accumulation (np.add.accumulate),
integer arithmetic, and the paper's printed bounds, example and orderings.
"""
import math
import os

import numpy as np
import pytest

import synthetic

EPS_F = 2.0 ** -24
EPS_B = 2.0 ** -8
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def gam(k, eps=EPS_F):
    """gamma_k = k eps / (1 - k eps)."""
    return k * eps / (1 - k * eps)


def _golden_xy():
    vals = {}
    with open(os.path.join(GOLDEN, "paper_xy_example.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                k, v = line.split()
                vals[k] = v
    return vals


# ---------------------------------------------------------------------------------------
def test_partials_brute_force_small_k(orc):
    """Z^(i,j) is the FP32 FMA recursion over l.  Brute force: each BF16 x BF16
    product is exact in FP32, so the recursion equals numpy's *sequential* float32
    accumulation (np.add.accumulate) of the exact products; for k = 1 it is the exact
    product itself."""
    rng = np.random.default_rng(0)
    for k in (1, 2, 3, 7, 33):
        A = rng.uniform(-1, 1, size=(5, k)).astype(np.float32)
        B = rng.uniform(-1, 1, size=(k, 4)).astype(np.float32)
        Z = orc.partials(A, B)
        pa = [orc.widen(p) for p in orc.split(A)]
        pb = [orc.widen(p) for p in orc.split(B)]
        for i in range(3):
            for j in range(3):
                for r in range(5):
                    for c in range(4):
                        prods = (pa[i][r, :].astype(np.float64) * pb[j][:, c].astype(np.float64))
                        assert np.all(prods.astype(np.float32).astype(np.float64) == prods)  # exact in FP32
                        seq = np.add.accumulate(prods.astype(np.float32), dtype=np.float32)[-1]
                        assert Z[i, j, r, c] == seq


def test_multiply_sets_by_value(orc):
    """P:380-390 table: 2 BF16s -> 3 products {00,01,10}; 3 BF16s -> 6 products (adds the
    2^-16 bin {02,11,20}).  x = y = 1 + 2^-9 + 2^-18 splits into (1, 2^-9, 2^-18), so bin
    i+j is 2^-9(i+j) times the number of products in it:
      x3 = 1 + 2*2^-9          (exactly; Z11 = 2^-18 must be absent)
      x6 = 1 + 2*2^-9 + 3*2^-18  (exactly; all three bin-2 products present)
      x1 = 1."""
    x = np.array([[1 + 2 ** -9 + 2 ** -18]], dtype=np.float32)
    assert orc.widen(orc.split(x)[1])[0, 0] == 2 ** -9
    assert orc.widen(orc.split(x)[2])[0, 0] == 2 ** -18
    assert orc.gemm(x, x, variant=1)[0, 0] == 1.0
    assert orc.gemm(x, x, variant=3)[0, 0] == 1 + 2 * 2 ** -9
    assert orc.gemm(x, x, variant=6)[0, 0] == 1 + 2 * 2 ** -9 + 3 * 2 ** -18


def test_variant_product_sets_by_value(orc):
    """N2 product sets (reading R27), pinned by value with k = 2 and an exact
    cancellation of bin 0: x = y = (1 + 2^-9 + 2^-18, -1) . (1 + 2^-9 + 2^-18, 1) has pieces
    (1, 2^-9, 2^-18) and (-1, 0, 0) / (1, 0, 0), so Z00 = 0 and every other Z^(i,j) is
    2^-9(i+j) (each a single term), and the result is the sum of the products the variant
    takes, exactly (all spans <= 24 bits):
      x3 = 2*2^-9;  x5 = 2*2^-9 + 2*2^-18 (A has no third piece: Z20 absent);
      x6 = 2*2^-9 + 3*2^-18;  x7 = x6 + 2^-27 (Z12 only);  x8 = x6 + 2*2^-27."""
    t = 1 + 2 ** -9 + 2 ** -18
    A = np.array([[t, -1.0]], dtype=np.float32)
    B = np.array([[t], [1.0]], dtype=np.float32)
    want = {3: 2 * 2 ** -9, 5: 2 * 2 ** -9 + 2 * 2 ** -18, 6: 2 * 2 ** -9 + 3 * 2 ** -18,
            7: 2 * 2 ** -9 + 3 * 2 ** -18 + 2 ** -27, 8: 2 * 2 ** -9 + 3 * 2 ** -18 + 2 * 2 ** -27}
    for v, val in want.items():
        assert float(orc.gemm(A, B, variant=v)[0, 0]) == val, v
    # x5's asymmetry: with B = (1 + 2^-9, 1) (pieces 1, 2^-9, 0) only Z11 and Z20 are nonzero
    # in bin 2; x5 drops Z20 (A's third piece), x6 keeps both
    B2 = np.array([[1 + 2 ** -9], [1.0]], dtype=np.float32)
    assert float(orc.gemm(A, B2, variant=5)[0, 0]) == 2 ** -8 + 2 ** -18
    assert float(orc.gemm(A, B2, variant=6)[0, 0]) == 2 ** -8 + 2 * 2 ** -18


def test_x9_product_set_and_order_by_value(orc):
    """x9 = Z0 + (Z1 + (Z2 + (Z3 + Z4))) ("bins should be added from smallest to
    largest"; reading R9), pinned by value: Z^(2,2) must be present and the bins must be
    added smallest first.  u = 1 + 2^-8 + 2^-17 splits into (1 + 2^-7, -2^-8, 2^-17); with
    k = 6, A = (u, -u0, u, u0, 1, 2^-23), B = (u, u, -u0, u0, 1, 1) every Z^(0,j) and Z^(i,0)
    cancels exactly except Z00 = 1 + 2^-23 (each FP32 step exact), and Z11 = u1^2 = 2^-16,
    Z12 = Z21 = u1 u2 = -2^-25, Z22 = u2^2 = 2^-34.  Hence
      x9 (smallest first): 1 + 2^-23 + (2^-16 - 2^-24 + 2^-34) -> 1 + 2^-16 + 2^-23
          (the exact sum is 1 + 2^-16 + 2^-24 + 2^-34: above the half-ulp, rounds up);
      x8 (no Z22): 1 + 2^-16 + 2^-24 is a tie -> even -> 1 + 2^-16;
      largest first ((((Z0 + Z1) + Z2) + Z3) + Z4): the tie is met before Z22 -> 1 + 2^-16."""
    u = 1 + 2 ** -8 + 2 ** -17
    p = [float(orc.widen(q)[0, 0]) for q in orc.split(np.array([[u]], dtype=np.float32))]
    assert p == [1 + 2 ** -7, -2 ** -8, 2 ** -17]
    u0 = p[0]
    A = np.array([[u, -u0, u, u0, 1.0, 2 ** -23]], dtype=np.float32)
    B = np.array([[u], [u], [-u0], [u0], [1.0], [1.0]], dtype=np.float32)
    Z = orc.partials(A, B)[:, :, 0, 0].astype(np.float64)
    want_z = np.zeros((3, 3))
    want_z[0, 0], want_z[1, 1], want_z[1, 2], want_z[2, 1], want_z[2, 2] = 1 + 2 ** -23, 2 ** -16, -2 ** -25, -2 ** -25, 2 ** -34
    assert np.array_equal(Z, want_z)
    assert float(orc.gemm(A, B, variant=9)[0, 0]) == 1 + 2 ** -16 + 2 ** -23
    assert float(orc.gemm(A, B, variant=8)[0, 0]) == 1 + 2 ** -16
    f = np.float32
    largest_first = f(f(f(f(f(Z[0, 0]) + f(0)) + f(Z[1, 1])) + f(f(Z[1, 2]) + f(Z[2, 1]))) + f(Z[2, 2]))
    assert float(largest_first) == 1 + 2 ** -16          # the order is what the pin detects


def test_partial_sums_are_fused_multiply_adds(orc):
    """Z <- FMA(x_l, y_l, Z), one rounding per term.  A BF16 x BF16 product is exact
    in FP32 unless it is subnormal; there a multiply-then-add rounds twice.  With
    A = (2^-125, 2^-74, (1 + 2^-7) 2^-75) and B = (1, 2^-74, 2^-75) (all BF16), Z reaches
    2^-125 + 2^-148 (odd at its quantum 2^-148) and the third product is (1 + 2^-7) 2^-150:
    FMA: RN(Z + 0.252 quantum) = Z;  multiply first: RN(p) = 2^-149 = half a quantum, a tie
    that rounds Z up to 2^-125 + 2^-147."""
    A = np.array([[2.0 ** -125, 2.0 ** -74, (1 + 2 ** -7) * 2.0 ** -75]], dtype=np.float32)
    B = np.array([[1.0], [2.0 ** -74], [2.0 ** -75]], dtype=np.float32)
    for v in (1, 3, 6, 9):
        assert float(orc.gemm(A, B, variant=v)[0, 0]) == 2.0 ** -125 + 2.0 ** -148, v
    mul_add = np.float32(np.float32(2.0 ** -125 + 2.0 ** -148) + np.float32(A[0, 2] * B[2, 0]))
    assert float(mul_add) == 2.0 ** -125 + 2.0 ** -147


def test_x5_x7_identity_closed_forms(orc):
    """A*I under x5 (A in two pieces) is fl32(a0 + a1) -- the third piece is dropped -- and
    under x7 it is A exactly; I*B is B exactly under both (B keeps three pieces).  x5 equals
    x6 bit for bit when A's values carry <= 16 significant bits (a2 == 0)."""
    rng = np.random.default_rng(5)
    A = synthetic.uniform(19, 13, seed=int(rng.integers(1 << 30)))
    I = np.eye(13, dtype=np.float32)
    a0, a1, _ = (orc.widen(p) for p in orc.split(A))
    assert np.array_equal(orc.gemm(A, I, variant=5), (a0 + a1).astype(np.float32))
    assert np.array_equal(orc.gemm(A, I, variant=7), A)
    B = synthetic.uniform(13, 11, seed=int(rng.integers(1 << 30)))
    for v in (5, 7):
        assert np.array_equal(orc.gemm(I, B, variant=v), B)
    A16 = (a0 + a1).astype(np.float32)                       # exactly two BF16 pieces
    assert np.all(orc.widen(orc.split(A16)[2]) == 0)
    assert np.array_equal(orc.gemm(A16, B, variant=5), orc.gemm(A16, B, variant=6))


def test_paper_worked_example_xy(orc):
    """P:376 worked example (tests/golden/paper_xy_example.txt): with 6 products the result is
    less accurate than FP32 (the 2^-24-bin term a1*b2 matters); with all 9 products the FP32
    accuracy is reached."""
    g = _golden_xy()
    x = np.float32(float(g["x"]))
    y = np.float32(float(g["y"]))
    exact = float(x) * float(y)                      # exact in FP64 (24+24 bits)
    A = np.array([[x]], dtype=np.float32)
    B = np.array([[y]], dtype=np.float32)
    f32 = float(orc.sgemm_fma(A, B)[0, 0])
    x6 = float(orc.gemm(A, B, variant=6)[0, 0])
    x9 = float(orc.gemm(A, B, variant=9)[0, 0])
    x8 = float(orc.gemm(A, B, variant=8)[0, 0])
    x7 = float(orc.gemm(A, B, variant=7)[0, 0])
    assert f32 == float(np.float32(exact))           # one rounding
    assert abs(x7 - exact) <= abs(f32 - exact)       # "computing at least 7 products"
    assert abs(x6 - exact) > abs(f32 - exact)
    assert abs(x9 - exact) <= abs(f32 - exact)
    assert abs(x8 - exact) <= abs(f32 - exact)
    # the E term: |Z12 + Z21 + Z22| <= (513/512) 2^-23 |a0 b0|
    Z = orc.partials(A, B)[:, :, 0, 0].astype(np.float64)
    assert abs(Z[1, 2] + Z[2, 1] + Z[2, 2]) <= (513 / 512) * 2.0 ** -23 * abs(Z[0, 0])


def test_identity_and_permutation_exact(orc):
    """A*I and A*P: each output has one nonzero term per piece pair, so the bins recombine the
    split exactly (x6/x9 return A bit-exactly in the safe exponent range)."""
    rng = np.random.default_rng(1)
    for dist in ("uniform", "wide", "gauss"):
        A = synthetic.by_name(dist, 33, 17, seed=int(rng.integers(1 << 30)))
        I = np.eye(17, dtype=np.float32)
        P = I[:, rng.permutation(17)]
        for v in (6, 9):
            assert np.array_equal(orc.gemm(A, I, variant=v), A)
            assert np.array_equal(orc.gemm(A, P, variant=v), A @ P)
            assert np.array_equal(orc.gemm(P.T, A.T, variant=v), P.T @ A.T)


def test_small_integers_exact(orc):
    """10-bit integers need two BF16 pieces; with k <= 16 every product and partial sum is an
    integer below 2^24, so x6 and x9 must equal the exact integer product (int64 matmul),
    while x3 (no Z11 term) must not in general."""
    A = synthetic.small_ints(24, 16, seed=3, bound=1000)
    B = synthetic.small_ints(16, 20, seed=4, bound=1000)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    for v in (6, 9):
        assert np.array_equal(orc.gemm(A, B, variant=v).astype(np.float64), exact)
    assert not np.array_equal(orc.gemm(A, B, variant=3).astype(np.float64), exact)
    assert np.array_equal(orc.dgemm(A, B), exact)


def test_fp32_reference_bound_and_exact_case(orc):
    """|Z - z| <= gamma_n * z~ for the FP32 FMA recursion; (2^20, 1).(1, 1) =
    2^20 + 1 exactly."""
    A = np.array([[2.0 ** 20, 1.0]], dtype=np.float32)
    B = np.array([[1.0], [1.0]], dtype=np.float32)
    assert orc.sgemm_fma(A, B)[0, 0] == 2.0 ** 20 + 1
    rng = np.random.default_rng(2)
    for n in (1, 10, 100, 1000, 4096):
        x = rng.uniform(-1, 1, size=(1, n)).astype(np.float32)
        y = rng.uniform(-1, 1, size=(n, 1)).astype(np.float32)
        prods = x[0].astype(np.float64) * y[:, 0].astype(np.float64)
        z, zt = math.fsum(prods), math.fsum(np.abs(prods))
        Z = float(orc.sgemm_fma(x, y)[0, 0])
        assert abs(Z - z) <= gam(n) * zt
        # the FP64 reference is the exact sum to within FP64 rounding
        assert abs(float(orc.dgemm(x, y)[0, 0]) - z) <= n * 2.0 ** -53 * zt


@pytest.mark.parametrize("dist", ["uniform", "wide", "gauss"])
def test_z2_error_bound(orc, dist):
    """P:309-321 (§II-E): |Z_2 - z| <= 1.01 (gamma_{n+2} + eps^3) z~, with the eps_b^3 reading of
    the printed eps_f^3 (R11, the derivation's own truncation term P:313).  Zero violations
    over random dot products; the per-bin bound |Z^(i,j) - z^(i,j)| <= gamma_n eps_b^(i+j) z~
     is audited too."""
    rng = np.random.default_rng(hash(dist) & 0xFFFF)
    for trial in range(60):
        n = int(rng.choice([1, 2, 16, 100, 1000, 4096]))
        s = int(rng.integers(1 << 30))
        x = synthetic.by_name(dist, 1, n, seed=s)
        y = synthetic.by_name(dist, n, 1, seed=s + 1)
        prods = x[0].astype(np.float64) * y[:, 0].astype(np.float64)
        z, zt = math.fsum(prods), math.fsum(np.abs(prods))
        Z2 = float(orc.gemm(x, y, variant=6)[0, 0])
        assert abs(Z2 - z) <= 1.01 * (gam(n + 2) + EPS_B ** 3) * zt
        Z = orc.partials(x, y)[:, :, 0, 0].astype(np.float64)
        px = [orc.widen(p)[0].astype(np.float64) for p in orc.split(x)]
        py = [orc.widen(p)[:, 0].astype(np.float64) for p in orc.split(y)]
        for i in range(3):
            for j in range(3):
                zij = math.fsum(px[i] * py[j])
                assert abs(Z[i, j] - zij) <= gam(n) * EPS_B ** (i + j) * zt * 1.0000001 + 1e-300


def test_exact_accumulation_special_case(orc):
    """when ceil(log2(1.01 max|x y|)) - 23 <= ceil(log2(0.99 min|x y|)) - 15, the
    level-0 sum is exact (Z^(0,0) = z^(0,0)) and |Z_2 - z| <= 1.01 gamma_3 z~.  Inputs: |x|, |y|
    in [1, 2) with random signs, n = 64 (so the sum also stays inside 24 bits)."""
    rng = np.random.default_rng(9)
    for trial in range(200):
        n = 64
        x = (rng.uniform(1, 2, size=(1, n)) * rng.choice([-1, 1], size=(1, n))).astype(np.float32)
        y = (rng.uniform(1, 2, size=(n, 1)) * rng.choice([-1, 1], size=(n, 1))).astype(np.float32)
        p = np.abs(x[0].astype(np.float64) * y[:, 0].astype(np.float64))
        assert math.ceil(math.log2(1.01 * p.max())) - 23 <= math.ceil(math.log2(0.99 * p.min())) - 15
        px0 = orc.widen(orc.split(x)[0])[0].astype(np.float64)
        py0 = orc.widen(orc.split(y)[0])[:, 0].astype(np.float64)
        Z = orc.partials(x, y)[:, :, 0, 0]
        assert float(Z[0, 0]) == math.fsum(px0 * py0)
        prods = x[0].astype(np.float64) * y[:, 0].astype(np.float64)
        z, zt = math.fsum(prods), math.fsum(np.abs(prods))
        assert abs(float(orc.gemm(x, y, variant=6)[0, 0]) - z) <= 1.01 * gam(3) * zt


def _errs(orc, dist, seeds, n=64):
    out = {v: [] for v in ("f32", 3, 6, 9)}
    for s in seeds:
        A = synthetic.by_name(dist, n, n, seed=s)
        B = synthetic.by_name(dist, n, n, seed=s + 50_000)
        C64 = orc.dgemm(A, B)
        out["f32"].append(orc.normwise_error(orc.sgemm_fma(A, B), C64, A, B))
        for v in (3, 6, 9):
            out[v].append(orc.normwise_error(orc.gemm(A, B, variant=v), C64, A, B))
    return {k: np.array(v) for k, v in out.items()}


def test_error_ordering_small_range(orc):
    """for [-1,1] data the order of error is b2x3 > SGEMM > b3x6 (Fig. 2), and
    bf16x9 ~ bf16x6 (north star).  64^3, 20 seeds."""
    e = _errs(orc, "uniform", range(20))
    assert e[3].mean() > e["f32"].mean() > e[6].mean()
    assert np.count_nonzero(e[6] < e["f32"]) >= 18
    assert e[9].mean() <= e[6].mean() * 1.05
    assert np.all(e[3] > 10 * e[6])


def test_error_ordering_wide_and_gaussian(orc):
    """with a huge exponent range SGEMM is "marginally" better than b3x6 but
    "nearly identical"; Gaussian exponents, b3x6 on average worse than SGEMM with a
    smaller gap.  Checked as: f32 <= x6 <= 2 f32 on the mean, x3 much worse."""
    for dist in ("wide", "gauss"):
        e = _errs(orc, dist, range(100, 120))
        assert e["f32"].mean() <= e[6].mean() <= 2 * e["f32"].mean()
        assert e[3].mean() > 5 * e[6].mean()
        assert e[9].mean() <= e[6].mean() * 1.05


def test_alpha_beta_quick_returns(orc):
    """BLAS semantics (R19): beta == 0 never reads C (NaN-filled C must not leak);
    alpha == 0 or k == 0 gives beta*C; general case alpha*AB + beta*C."""
    rng = np.random.default_rng(4)
    A = rng.uniform(-1, 1, size=(9, 5)).astype(np.float32)
    B = rng.uniform(-1, 1, size=(5, 7)).astype(np.float32)
    Cnan = np.full((9, 7), np.nan, dtype=np.float32, order="F")
    out = orc.gemm(A, B, C=Cnan, alpha=1.0, beta=0.0, variant=6)
    assert np.all(np.isfinite(out))
    C = rng.uniform(-1, 1, size=(9, 7)).astype(np.float32)
    assert np.array_equal(orc.gemm(A, B, C=C, alpha=0.0, beta=2.0, variant=6), (2.0 * C).astype(np.float32))
    ab = orc.gemm(A, B, variant=6)
    full = orc.gemm(A, B, C=C, alpha=-1.5, beta=0.5, variant=6)
    want = (np.float32(-1.5) * ab.astype(np.float64) + (np.float32(0.5) * C).astype(np.float64))
    assert np.allclose(full, want, rtol=2 ** -23, atol=0)
    A0 = np.zeros((9, 0), dtype=np.float32)
    B0 = np.zeros((0, 7), dtype=np.float32)
    assert np.array_equal(orc.gemm(A0, B0, C=C, alpha=1.0, beta=3.0, variant=9), (3.0 * C).astype(np.float32))
