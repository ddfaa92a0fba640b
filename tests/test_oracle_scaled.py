"""Pins for the oracle's N2 rows: power-of-two scaled pieces (reading R29)
and the FP64 final combine, the paper's "d" variants (P:420, P:425 caption; reading R30).

The references are independent of the oracle's code: exact rational / FP64 sums of the
pieces, the correctly rounded FP32 product (the FP64 product of two FP32 values is exact),
integer matrix products, power-of-two homogeneity, and the already-pinned unscaled split and
FP32-combine oracle (test_oracle_split.py, test_oracle_gemm.py).
"""
from fractions import Fraction

import numpy as np
import pytest

import synthetic


def _f(bits):
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def _recon_scaled(orc, x):
    b0, b1, b2 = orc.split_scaled(x)
    w = [orc.widen(b).astype(np.float64) for b in (b0, b1, b2)]
    return (w[0] + w[1] * 2.0 ** -8) + w[2] * 2.0 ** -16, (b0, b1, b2)


# ---------------------------------------------------------------------------------------
# scaled split (R29)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("field", [0, 1, 2, 8, 15, 16, 17, 18, 60, 127, 200, 253, 254])
def test_scaled_exact_for_every_exponent(orc, field):
    """P:344-351 (§II-F): the unscaled split loses bits below exponent -110 (pinned in
    test_oracle_split.py: fields <= 16 fail).  Scaling the residuals by 2^8 keeps every
    piece at the magnitude of x, so x = b0 + 2^-8 b1' + 2^-16 b2' exactly for EVERY finite x,
    subnormals and the b0-saturation band included -- exhaustively over all 2^24 patterns of
    the field, both signs.  (Each FP64 sum below is exact: the pieces span < 53 bits.)"""
    mant = np.arange(1 << 23, dtype=np.uint32)
    pats = np.concatenate([(field << 23) | mant, 0x80000000 | (field << 23) | mant]).astype(np.uint32)
    x = pats.view(np.float32)
    rec, _ = _recon_scaled(orc, x)
    assert int(np.count_nonzero(rec != x.astype(np.float64))) == 0


def test_scaled_random_patterns_all_fields(orc):
    """Same identity on 4M random finite patterns from every exponent field."""
    g = np.random.default_rng(29)
    pats = g.integers(0, 1 << 32, size=1 << 22, dtype=np.uint64).astype(np.uint32)
    pats = pats[(pats & 0x7F800000) != 0x7F800000]
    x = pats.view(np.float32)
    rec, _ = _recon_scaled(orc, x)
    assert np.array_equal(rec, x.astype(np.float64))


def test_scaled_equals_unscaled_times_powers_in_normal_range(orc):
    """Where every unscaled piece is a normal BF16 (or zero), scaling commutes with the
    rounding: b1' = 2^8 b1 and b2' = 2^16 b2 bit for bit (the unscaled split is pinned by
    test_oracle_split.py).  Exhaustive for biased exponent fields 60, 127 and 254.  The
    exception is the b0-saturation band |x| >= 0x7F7F8000 (R3): there 2^8 b1 would be 2^128,
    so b1' saturates as well and the pieces differ (both still reconstruct x exactly)."""
    mant = np.arange(1 << 23, dtype=np.uint32)
    for field in (60, 127, 254):
        pats = np.concatenate([(field << 23) | mant, 0x80000000 | (field << 23) | mant]).astype(np.uint32)
        band = (pats & 0x7FFFFFFF) >= 0x7F7F8000
        assert int(band.sum()) == (2 * 0x8000 if field == 254 else 0)
        if band.any():   # b1' saturates for part of the band
            s1b = orc.split_scaled(pats[band].view(np.float32))[1]
            u1b = orc.split(pats[band].view(np.float32))[1]
            assert np.any((s1b & 0x7FFF) == 0x7F7F)
            assert not np.array_equal(orc.widen(u1b).astype(np.float64) * 256.0, orc.widen(s1b).astype(np.float64))
        x = pats[~band].view(np.float32)
        u0, u1, u2 = orc.split(x)
        s0, s1, s2 = orc.split_scaled(x)
        assert np.array_equal(u0, s0)
        assert np.array_equal(orc.widen(u1).astype(np.float64) * 256.0, orc.widen(s1).astype(np.float64))
        assert np.array_equal(orc.widen(u2).astype(np.float64) * 65536.0, orc.widen(s2).astype(np.float64))


def test_scaled_bad_numbers_of_section_II_F(orc):
    """P:346-348's "bad number" 0x0081FFFF and the RNE worst case 0x00817FFF (R2): the
    unscaled split loses bits 0-15 (b1 = b2 = 0 or subnormal-truncated); the scaled split
    reconstructs both exactly.  Non-finite values keep (bf16(x), +0, +0) (R4)."""
    x = _f([0x0081FFFF, 0x00817FFF, 0x80817FFF])
    b0, b1, b2 = orc.split(x)
    w = [orc.widen(b).astype(np.float64) for b in (b0, b1, b2)]
    assert np.any((w[0] + w[1]) + w[2] != x.astype(np.float64))
    rec, _ = _recon_scaled(orc, x)
    assert np.array_equal(rec, x.astype(np.float64))
    b0, b1, b2 = orc.split_scaled(np.array([np.inf, -np.inf, np.nan], dtype=np.float32))
    assert [hex(v) for v in b0] == ["0x7f80", "0xff80", "0x7fc0"]
    assert b1.tolist() == [0, 0, 0] and b2.tolist() == [0, 0, 0]


# ---------------------------------------------------------------------------------------
# GEMM with scaled pieces (R29)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("variant", [1, 3, 5, 6, 7, 8, 9])
def test_scaled_gemm_equals_unscaled_in_normal_range(orc, variant):
    """With U[-1,1] inputs and k = 48 no piece, product or partial sum leaves the normal
    range, so the Horner combine of the scaled bins (Z'_s = 2^(8s) Z_s, each brought down by
    an exact multiply by 2^-8) equals the pinned FP32 combine bit for bit, alpha/beta included."""
    A = synthetic.uniform(37, 48, seed=5)
    B = synthetic.uniform(48, 29, seed=6)
    C = synthetic.uniform(37, 29, seed=7)
    want = orc.gemm(A, B, C, alpha=0.75, beta=-1.25, variant=variant)
    got = orc.gemm(A, B, C, alpha=0.75, beta=-1.25, variant=variant, scaled=True)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("variant", [3, 6, 9])
def test_scaled_gemm_below_minus_110(orc, variant):
    """A scaled by 2^-115 and 2^-121 (below the paper's -110), B by 2^100.
    * At 2^-115 (almost) every scaled piece of A is still a normal BF16 and the scaled-piece
      GEMM is exactly homogeneous on these inputs: C(2^-115 A, 2^100 B) = 2^-15 C(A, B) bit
      for bit.  The
      unscaled pieces b2 are BF16 subnormals there: x6 / x9 lose a factor > 20 in accuracy.
    * At 2^-121 some scaled b1' are subnormal (the split stays exact, pinned above): the
      scaled GEMM keeps its normal-range accuracy (within 10 %); the unscaled one is > 1000x
      worse for x6 / x9, > 20x for x3 (b1 and b2 both subnormal)."""
    A = synthetic.uniform(40, 64, seed=11, lo=0.0625, hi=1.0)     # exponents -4..-1
    A[::3] = -A[::3]
    B = synthetic.uniform(64, 33, seed=12)
    C64 = orc.dgemm(A, B)
    base = orc.gemm(A, B, variant=variant, scaled=True)
    e_base = orc.normwise_error(base, C64, A, B)
    Bs = (B.astype(np.float64) * 2.0 ** 100).astype(np.float32)
    for sh in (-115, -121):
        As = (A.astype(np.float64) * 2.0 ** sh).astype(np.float32)
        assert np.array_equal(As.astype(np.float64) * 2.0 ** -sh, A.astype(np.float64))   # exact scaling
        got = orc.gemm(As, Bs, variant=variant, scaled=True).astype(np.float64) * 2.0 ** (-sh - 100)
        uns = orc.gemm(As, Bs, variant=variant).astype(np.float64) * 2.0 ** (-sh - 100)
        e_s = orc.normwise_error(got, C64, A, B)
        e_u = orc.normwise_error(uns, C64, A, B)
        pieces = orc.split_scaled(As)
        subn = sum(int(np.count_nonzero(((p & 0x7F80) == 0) & ((p & 0x7FFF) != 0))) for p in pieces)
        if sh == -115:
            assert subn <= 2
            assert np.array_equal(got, base.astype(np.float64))
            if variant >= 6:
                assert e_u > 20 * e_base
        else:
            assert subn > 0
            assert e_s <= 1.1 * e_base
            assert e_u > (1000 if variant >= 6 else 20) * e_base


def test_scaled_gemm_exact_on_subnormal_integers(orc):
    """A = integers x 2^-140 (FP32 subnormals), B = integers x 2^120: the exact product
    (A_int B_int) 2^-20 is an FP32 number (|entries| < 2^24).  With scaled pieces every
    piece and product is exact, so x3 / x6 / x9 reproduce it exactly; the unscaled split
    rounds A's residuals to BF16 subnormals (quantum 2^-133) and misses it."""
    g = np.random.default_rng(140)
    Ai = g.integers(-1000, 1001, size=(24, 16))
    Bi = g.integers(-200, 201, size=(16, 20))
    A = (Ai.astype(np.float64) * 2.0 ** -140).astype(np.float32)
    B = (Bi.astype(np.float64) * 2.0 ** 120).astype(np.float32)
    assert np.array_equal(A.astype(np.float64) * 2.0 ** 140, Ai.astype(np.float64))
    exact = (Ai @ Bi).astype(np.float64) * 2.0 ** -20
    assert np.abs(Ai @ Bi).max() < 2 ** 24
    for v in (3, 6, 9):
        assert np.array_equal(orc.gemm(A, B, variant=v, scaled=True).astype(np.float64), exact)
    assert not np.array_equal(orc.gemm(A, B, variant=6).astype(np.float64), exact)


# ---------------------------------------------------------------------------------------
# FP64 final combine, the "d" variants (R30)
# ---------------------------------------------------------------------------------------
def _exact_products_sum(orc, x, y, pairs, scaled=False):
    sp = orc.split_scaled if scaled else orc.split
    a = sp(np.array([x], dtype=np.float32))
    b = sp(np.array([y], dtype=np.float32))
    tot = Fraction(0)
    for i, j in pairs:
        ai = Fraction(float(orc.widen(a[i])[0])) * (Fraction(1, 256) ** i if scaled else 1)
        bj = Fraction(float(orc.widen(b[j])[0])) * (Fraction(1, 256) ** j if scaled else 1)
        tot += ai * bj
    return tot


def test_x9d_k1_is_the_correctly_rounded_product(orc):
    """k = 1: each Z^(i,j) is one exact product and the nine of them span < 53 bits, so the
    FP64 collection is exact and x9d = RN32(x*y) -- the correctly rounded FP32 product (the
    FP64 product of two FP32 numbers is exact).  Holds for the scaled pieces too, also at
    x's exponent -120 where the unscaled pieces are subnormal."""
    g = np.random.default_rng(9)
    x = synthetic.uniform(1, 400, seed=21).reshape(-1)
    y = synthetic.wide(1, 400, seed=22, E=20).reshape(-1)
    for t in range(400):
        xx, yy = x[t], y[t]
        want = np.float32(np.float64(xx) * np.float64(yy))
        got = orc.gemm(np.array([[xx]]), np.array([[yy]]), variant=9, fp64_combine=True)[0, 0]
        assert got == want, (t, xx, yy)
        got_s = orc.gemm(np.array([[xx]]), np.array([[yy]]), variant=9, fp64_combine=True, scaled=True)[0, 0]
        assert got_s == want
    xt = np.float32(np.float64(g.uniform(1, 2)) * 2.0 ** -120)
    yt = np.float32(g.uniform(1, 2) * 2.0 ** 100)
    want = np.float32(np.float64(xt) * np.float64(yt))
    assert orc.gemm(np.array([[xt]]), np.array([[yt]]), variant=9, fp64_combine=True, scaled=True)[0, 0] == want


@pytest.mark.parametrize("variant,pairs", [
    (3, [(0, 0), (0, 1), (1, 0)]),
    (6, [(0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0)]),
])
def test_xd_k1_rounds_the_exact_bin_sum_once(orc, variant, pairs):
    """k = 1 (an outer product: 300 x 300 pairs x*y at once): x3d / x6d = RN32 of the exact
    sum of the variant's piece products ("adding the final results together in FP64";
    one rounding).  The exact sum is formed in FP64 from the pinned split: every product and
    partial sum spans < 53 bits, so it is exact (confirmed with rationals on a sample).  The
    FP32 combine rounds each bin sum; for x6 it differs from the single rounding for some
    pairs (that difference is the "d"); for x3 the FP32 bin sum a0*b1 + a1*b0 is exact."""
    x = synthetic.uniform(300, 1, seed=31)
    y = synthetic.uniform(1, 300, seed=32)
    a = [orc.widen(p).astype(np.float64) for p in orc.split(x)]
    b = [orc.widen(p).astype(np.float64) for p in orc.split(y)]
    exact = np.zeros((300, 300))
    for i, j in pairs:
        exact += a[i] @ b[j]                     # k = 1: outer product, exact in FP64
    for t in range(0, 300, 37):                  # rational confirmation on a sample
        ex = _exact_products_sum(orc, x[t, 0], y[0, (7 * t) % 300], pairs)
        assert Fraction(float(exact[t, (7 * t) % 300])) == ex
    want = exact.astype(np.float32)
    got = orc.gemm(x, y, variant=variant, fp64_combine=True)
    assert np.array_equal(got, want)
    assert np.array_equal(orc.gemm(x, y, variant=variant, fp64_combine=True, scaled=True), want)
    differ = int(np.count_nonzero(orc.gemm(x, y, variant=variant) != want))
    assert (differ > 0) if variant == 6 else (differ == 0)


def test_x6d_ordering_over_seeds(orc):
    """P:420-425 (Fig. "smallgemm", [-1,1] data): "the order of accuracy was the order stated
    here": bx2_3, SGEMM, bx3_6, bx3_6d.  Mean normwise error over 20 seeds at 64^3: x6d is
    more accurate than SGEMM; x6d and x6 agree within 0.1 % (the partial sums' FP32
    accumulation over k dominates the error, the final combine's rounding is negligible), so
    the paper's strict x6 -> x6d step is not resolvable here (reading R30; x3 > SGEMM > x6 is
    pinned in test_oracle_gemm.py)."""
    e6, e6d, e32 = [], [], []
    for s in range(20):
        A = synthetic.uniform(64, 64, seed=2 * s + 400)
        B = synthetic.uniform(64, 64, seed=2 * s + 401)
        C64 = orc.dgemm(A, B)
        e6.append(orc.normwise_error(orc.gemm(A, B, variant=6), C64, A, B))
        e6d.append(orc.normwise_error(orc.gemm(A, B, variant=6, fp64_combine=True), C64, A, B))
        e32.append(orc.normwise_error(orc.sgemm_fma(A, B), C64, A, B))
    assert abs(np.mean(e6d) - np.mean(e6)) <= 1e-3 * np.mean(e6)
    assert np.mean(e6d) < 0.5 * np.mean(e32)
