"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic (no split, no products, no sums): only
random draws, so that both sides of a parity test see identical bytes.  Every
generator returns an FP32 matrix in column-major (Fortran) order, generated
column block by column block with a per-block counter-derived PCG64 stream so
that the bytes do not depend on how many blocks are requested at a time.

Distributions:
  uniform       FP64 U[lo,hi] rounded to FP32 ("[-1.0,1.0] range with
                drand48()"; reading R18)
  wide          sign uniform, unbiased exponent uniform integer in [-E, E],
                23 uniform mantissa bits ("exponents are randomly chosen
                bits"; reading R16, E = 48)
  gauss_exp     as wide but the exponent is round(N(0, sigma)) clamped to
                [-E, E] ("Gaussian distribution"; reading R17, sigma = 8)
  conditioned   U diag(s) V^T, U, V Haar-orthogonal (FP64 QR of Gaussians),
                s geometric from 1 to 1/kappa, rounded to FP32 (config 5;
                reading R15)
  diagdom       uniform off-diagonal, |a_ii| = row abs-sum + 1
"""
from __future__ import annotations

import numpy as np

_BLOCK = 256  # columns per independently-seeded block


def _block_rng(seed: int, tag: int, block: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([int(seed) & 0xFFFFFFFF, int(tag), int(block)]))


def _by_blocks(rows: int, cols: int, seed: int, tag: int, fill) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float32, order="F")
    for b0 in range(0, cols, _BLOCK):
        b1 = min(cols, b0 + _BLOCK)
        out[:, b0:b1] = fill(_block_rng(seed, tag, b0 // _BLOCK), rows, b1 - b0)
    return out


def uniform(rows: int, cols: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    return _by_blocks(rows, cols, seed, 1,
                      lambda g, r, c: g.uniform(lo, hi, size=(c, r)).T.astype(np.float32))


def _exp_mant(g: np.random.Generator, r: int, c: int, exps: np.ndarray) -> np.ndarray:
    sign = g.integers(0, 2, size=(c, r), dtype=np.uint32)
    mant = g.integers(0, 1 << 23, size=(c, r), dtype=np.uint32)
    field = (exps.astype(np.int64) + 127).astype(np.uint32)
    bits = (sign << 31) | (field << 23) | mant
    return bits.view(np.float32).T


def wide(rows: int, cols: int, seed: int, E: int = 48) -> np.ndarray:
    def fill(g, r, c):
        e = g.integers(-E, E + 1, size=(c, r))
        return _exp_mant(g, r, c, e)
    return _by_blocks(rows, cols, seed, 2, fill)


def gauss_exp(rows: int, cols: int, seed: int, sigma: float = 8.0, E: int = 48) -> np.ndarray:
    def fill(g, r, c):
        e = np.clip(np.rint(g.normal(0.0, sigma, size=(c, r))), -E, E).astype(np.int64)
        return _exp_mant(g, r, c, e)
    return _by_blocks(rows, cols, seed, 3, fill)


def small_ints(rows: int, cols: int, seed: int, bound: int) -> np.ndarray:
    """Integers uniform in [-bound, bound] (exact-arithmetic pins)."""
    return _by_blocks(rows, cols, seed, 4,
                      lambda g, r, c: g.integers(-bound, bound + 1, size=(c, r)).T.astype(np.float32))


def by_name(dist: str, rows: int, cols: int, seed: int) -> np.ndarray:
    if dist == "uniform":
        return uniform(rows, cols, seed)
    if dist == "wide":
        return wide(rows, cols, seed)
    if dist == "gauss":
        return gauss_exp(rows, cols, seed)
    raise ValueError(dist)


def _haar(g: np.random.Generator, n: int) -> np.ndarray:
    q, r = np.linalg.qr(g.standard_normal((n, n)))
    return q * np.sign(np.diag(r))[None, :]


def conditioned(n: int, kappa: float, seed: int):
    """Returns (A_fp32 column-major, sigma) with A = U diag(sigma) V^T rounded to FP32."""
    g = np.random.Generator(np.random.PCG64([int(seed) & 0xFFFFFFFF, 5]))
    U = _haar(g, n)
    V = _haar(g, n)
    s = np.geomspace(1.0, 1.0 / kappa, n) if n > 1 else np.ones(1)
    A = (U * s[None, :]) @ V.T
    return np.asfortranarray(A.astype(np.float32)), s


def diagdom(n: int, seed: int) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64([int(seed) & 0xFFFFFFFF, 6]))
    A = g.uniform(-1.0, 1.0, size=(n, n))
    np.fill_diagonal(A, 0.0)
    np.fill_diagonal(A, np.abs(A).sum(axis=1) + 1.0)
    return np.asfortranarray(A.astype(np.float32))


def rhs(n: int, seed: int) -> np.ndarray:
    """x_true ~ N(0,1) in FP64 (config 5)."""
    g = np.random.Generator(np.random.PCG64([int(seed) & 0xFFFFFFFF, 7]))
    return g.standard_normal(n)
