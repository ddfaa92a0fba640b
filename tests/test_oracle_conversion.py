"""Pins for the oracle's (B16)/(F32) operators (§II-A; R1, R3, R4).

Each test checks the oracle against something other than itself: the format
definition, an exhaustive 16-bit sweep, a library RNE routine
(torch's CPU float32->bfloat16 conversion), or hand-derived tie cases.
"""
import numpy as np
import pytest
import torch


def _f(bits):
    return np.asarray(bits, dtype=np.uint32).view(np.float32)


def test_widen_narrow_identity_all_65536(orc):
    """Every BF16 pattern widens exactly and rounds back to itself (BF16 is
    FP32 with 16 mantissa bits cut); NaN patterns canonicalise to 0x7FC0 (R4)."""
    pats = np.arange(1 << 16, dtype=np.uint32)
    x = (pats << 16).view(np.float32)
    b0, b1, b2 = orc.split(x)
    is_nan = ((pats & 0x7F80) == 0x7F80) & ((pats & 0x007F) != 0)
    assert np.array_equal(b0[~is_nan], pats[~is_nan].astype(np.uint16))
    assert np.all(b0[is_nan] == 0x7FC0)
    # an exactly representable value leaves no residual
    fin = ~((pats & 0x7F80) == 0x7F80)
    assert np.all((b1[fin] & 0x7FFF) == 0) and np.all((b2[fin] & 0x7FFF) == 0)
    # the widening operator is the exact bit shift
    for p in (0x3F80, 0xC000, 0x0001, 0x8001, 0x7F7F):
        assert orc.bf16_widen(p) == float(_f(p << 16))


def test_ties_to_even():
    """Hand-derived tie cases: 0x3F808000 (1 + 2^-8) is exactly half-way between 0x3F80 and
    0x3F81 and rounds to the even 0x3F80; 0x3F818000 rounds up to even 0x3F82."""
    import oracle
    assert oracle.bf16_round(_f(0x3F808000)) == 0x3F80
    assert oracle.bf16_round(_f(0x3F818000)) == 0x3F82
    assert oracle.bf16_round(_f(0x3F808001)) == 0x3F81
    assert oracle.bf16_round(_f(0x3F807FFF)) == 0x3F80
    assert oracle.bf16_round(_f(0xBF808000)) == 0xBF80
    assert oracle.bf16_round(1.0) == 0x3F80
    assert oracle.bf16_round(-2.0) == 0xC000


def test_matches_library_rne_routine(orc):
    """Outside the overflow band and NaNs, (B16) is IEEE RNE, so it must equal torch's CPU
    float32 -> bfloat16 conversion (a library RNE routine) bit for bit."""
    rng = np.random.default_rng(123)
    rnd = rng.integers(0, 1 << 32, size=4_000_000, dtype=np.uint64).astype(np.uint32)
    sub = np.concatenate([np.arange(0, 1 << 20, dtype=np.uint32),
                          np.arange(0x80000000, 0x80000000 + (1 << 20), dtype=np.uint32),
                          np.arange(0x007F0000, 0x00810000, dtype=np.uint32),
                          np.arange(0x7F7E0000, 0x7F7F8000, dtype=np.uint32)])
    pats = np.concatenate([rnd, sub])
    x = pats.view(np.float32)
    absbits = pats & 0x7FFFFFFF
    keep = (absbits < 0x7F7F8000)            # finite and RNE does not overflow
    x = x[keep]
    b0, _, _ = orc.split(x)
    ref = torch.from_numpy(x.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(b0, ref)


def test_saturation_and_specials(orc):
    """R3: finite values whose RNE rounding overflows saturate to +-0x7F7F; R4: NaN -> 0x7FC0;
    +-Inf stay +-Inf; signed zeros keep their sign."""
    cases = {0x7F7F8000: 0x7F7F, 0x7F7FFFFF: 0x7F7F, 0xFF7F8000: 0xFF7F, 0xFF7FFFFF: 0xFF7F,
             0x7F7F7FFF: 0x7F7F, 0x7F800000: 0x7F80, 0xFF800000: 0xFF80, 0x7FC00000: 0x7FC0,
             0x7F800001: 0x7FC0, 0xFFFFFFFF: 0x7FC0, 0x00000000: 0x0000, 0x80000000: 0x8000}
    x = _f(list(cases))
    b0, b1, b2 = orc.split(x)
    assert [int(v) for v in b0] == list(cases.values())
    nonfin = ~np.isfinite(x)
    assert np.all(b1[nonfin] == 0) and np.all(b2[nonfin] == 0)


def test_error_bound_and_monotone(orc):
    """For normal results |bf16(x) - x| <= 2^-8 |x| (half an ulp of an 8-significant-bit
    format, eps_b = 2^-8) and rounding is monotone."""
    rng = np.random.default_rng(7)
    x = rng.uniform(-1e30, 1e30, size=200_000).astype(np.float32)
    x = np.concatenate([x, rng.uniform(-1, 1, size=200_000).astype(np.float32)])
    b0, _, _ = orc.split(x)
    w = orc.widen(b0).astype(np.float64)
    xd = x.astype(np.float64)
    assert np.all(np.abs(w - xd) <= 2.0 ** -8 * np.abs(xd))
    order = np.argsort(xd, kind="stable")
    assert np.all(np.diff(w[order]) >= 0)
