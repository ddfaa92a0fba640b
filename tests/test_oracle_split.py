"""Pins for the oracle's 3-way split (§II-A) against the paper and exact arithmetic.

Reconstruction is checked in FP64 with plain numpy (independent of the oracle's FP32
residual arithmetic): b0 + b1 + b2 is exact in FP64 for any three BF16 values that
come from one FP32 number.
"""
import math

import numpy as np
import pytest


def _f(bits):
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def _recon(orc, x):
    b0, b1, b2 = orc.split(x)
    w = [orc.widen(b).astype(np.float64) for b in (b0, b1, b2)]
    return (w[0] + w[1]) + w[2], (b0, b1, b2)


def test_worked_values(orc):
    """S:121-122 worked values, plus hand-derived bit cases:
      1.5 = bf16 exactly -> (1.5, +0, +0);  1 + 2^-20 -> (1, 2^-20, +0);
      0x3F80FFFF = 1 + 2^-7 - 2^-23: b0 rounds up to 1 + 2^-7 (0x3F81), residual -2^-23
        is a BF16 (0xB400), b2 = +0;
      0x7F7FFFFF (max finite): b0 saturates to 0x7F7F (R3) and the residual pieces carry
        the rest exactly: (0x7F7F, 0x7B80, 0xF380)."""
    x = np.array([1.5, 1 + 2 ** -20], dtype=np.float32)
    b0, b1, b2 = orc.split(x)
    assert orc.widen(b0).tolist() == [1.5, 1.0]
    assert orc.widen(b1).tolist() == [0.0, 2 ** -20]
    assert b2.tolist() == [0, 0]
    b0, b1, b2 = orc.split(_f([0x3F80FFFF, 0x7F7FFFFF]))
    assert [hex(v) for v in b0] == ["0x3f81", "0x7f7f"]
    assert [hex(v) for v in b1] == ["0xb400", "0x7b80"]
    assert [hex(v) for v in b2] == ["0x0", "0xf380"]
    # (F32)(a - b0 - b1) is left to right: -0 -> (0x8000, +0, +0)  (R5)
    b0, b1, b2 = orc.split(np.array([-0.0], dtype=np.float32))
    assert (int(b0[0]), int(b1[0]), int(b2[0])) == (0x8000, 0, 0)


@pytest.mark.parametrize("field", [0, 1, 2, 8, 15, 16, 17, 18, 60, 127, 200, 253, 254])
def test_exact_reconstruction_threshold(orc, field):
    """P:348 (§II-F): "As long as the exponent of a is at least no smaller than -110, then we
    can form b1 and b2 within the FP32 threshold".  Exhaustively over all 2^24 patterns of a
    biased exponent field (both signs): fields >= 17 (unbiased >= -110) reconstruct exactly;
    fields <= 16 lose bits for some values (the paper's worst case)."""
    mant = np.arange(1 << 23, dtype=np.uint32)
    pats = np.concatenate([(field << 23) | mant, 0x80000000 | (field << 23) | mant]).astype(np.uint32)
    x = pats.view(np.float32)
    rec, _ = _recon(orc, x)
    bad = int(np.count_nonzero(rec != x.astype(np.float64)))
    if field >= 17:
        assert bad == 0
    else:
        assert bad > 0


def test_paper_bad_number_and_rne_worst_case(orc):
    """a value with exponent field 1 and mantissa bits 0-15 set loses those bits
    (b1 = b2 = 0).  Under RNE (R1, R2) the paper's 0x0081FFFF rounds b0 *up* and is nearly
    exact; the pattern with bit 15 clear, 0x00817FFF, is the RNE worst case: b1 = b2 = +0 and
    the relative error is 0x7FFF/0x817FFF ~ 3.86e-3 ~ 2^-8.  Value check: 0x0081FFFF ~ 1.1939e-38
    as printed."""
    x = _f([0x0081FFFF, 0x00817FFF])
    assert abs(float(x[0]) - 1.1939e-38) < 1e-42
    rec, (b0, b1, b2) = _recon(orc, x)
    assert int(b0[0]) == 0x0082
    assert abs(rec[0] - float(x[0])) / float(x[0]) < 2e-7
    assert (int(b0[1]), int(b1[1]), int(b2[1])) == (0x0081, 0, 0)
    rel = abs(rec[1] - float(x[1])) / float(x[1])
    assert abs(rel - 0x7FFF / 0x817FFF) < 1e-12
    assert 2.0 ** -9 < rel < 2.0 ** -7


def test_piece_magnitudes(orc):
    """P:358-359 (§II-G): |a1| <= 2^-8 |a0| and |a2| <= 2^-16 |a0| in the safe range."""
    rng = np.random.default_rng(11)
    n = 2_000_000
    e = rng.integers(17, 254, size=n).astype(np.uint32)
    pats = (rng.integers(0, 2, size=n).astype(np.uint32) << 31) | (e << 23) | rng.integers(0, 1 << 23, size=n).astype(np.uint32)
    x = pats.view(np.float32)
    b0, b1, b2 = orc.split(x)
    a0, a1, a2 = (np.abs(orc.widen(b).astype(np.float64)) for b in (b0, b1, b2))
    assert np.all(a1 <= 2.0 ** -8 * a0)
    assert np.all(a2 <= 2.0 ** -16 * a0)
    rec = orc.widen(b0).astype(np.float64) + orc.widen(b1).astype(np.float64) + orc.widen(b2).astype(np.float64)
    assert np.array_equal(rec, x.astype(np.float64))


def test_decay_statistics_1_over_768(orc):
    """P:372 (§II-G): "on average, |a1| ~ |a0/768|" and |a2| ~ |a0/768^2|.  For mantissas
    uniform in [1,2) the RNE residual |r1| is uniform on [0, 2^-8], so E|b1| / E|b0| is
    exactly 2^-9 / 1.5 = 1/768 (closed form); the mean of the ratio is ln2/512 (closed form).
    |a2| is checked within 25% of 1/768^2 (S:143 band)."""
    rng = np.random.default_rng(5)
    x = rng.uniform(1.0, 2.0, size=4_000_000).astype(np.float32)
    b0, b1, b2 = orc.split(x)
    a0, a1, a2 = (np.abs(orc.widen(b).astype(np.float64)) for b in (b0, b1, b2))
    assert abs(a1.mean() / a0.mean() * 768 - 1) < 0.01
    assert abs(np.mean(a1 / a0) * 512 / math.log(2) - 1) < 0.01
    assert abs(a2.mean() / a0.mean() * 768 ** 2 - 1) < 0.25


def test_x3_uses_first_two_pieces(orc):
    """S:150 / P:378-380: the pair-of-BF16 variant consumes b0, b1 of the same split:
    a GEMM with B = I returns fl32(b0 + b1) for x3 and exactly A for x6/x9."""
    rng = np.random.default_rng(3)
    A = rng.uniform(-1, 1, size=(16, 8)).astype(np.float32)
    I = np.eye(8, dtype=np.float32)
    b0, b1, _ = orc.split(A)
    want3 = (orc.widen(b0) + orc.widen(b1)).astype(np.float32)
    assert np.array_equal(orc.gemm(A, I, variant=3), want3)
    for v in (6, 9):
        assert np.array_equal(orc.gemm(A, I, variant=v), A)
