"""K2 on the device against exact constructions and against its own schedule.

1. Product sets by value (the product table): inputs whose
   bins are exactly representable make the result the exact sum of the products the variant
   takes -- on the tensor core as in the oracle (every addend is a multiple of the MMA's
   alignment quantum, so nothing is truncated).  The pattern is placed at scattered k inside
   a multi-tile, multi-interval problem with power-of-two row / column scalings (exact).
2. The elementwise error bound of section II-E (reading R11: the derivable
   1.01 (gamma_{k+2} + eps_b^3) |A||B| form) holds for every output of the 6-, 7-, 8- and
   9-product variants.
3. Schedule conformance: the kernel's output equals, bit for bit, tests/tc_model.py -- the
   schedule of DESIGN.md section 6 (bands smallest bin first, the variant's product set, the
   promotion interval, RN promotion) executed on a model of tcgen05's FP32 accumulation that
   was fitted on 196,608 single-interval MMA results (tools/tc_model_fit.py).  A dropped,
   duplicated or reordered product, band or interval changes bits here even where the
   normwise parity tests cannot see it.  (The model is not the oracle: parity stays with the
   paper-order oracle in test_gpu_gemm.py / test_gpu_configs.py.)
"""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic
import tc_model

pytestmark = pytest.mark.gpu

EPS_F = 2.0 ** -24
EPS_B = 2.0 ** -8


def _gpu(A, B, variant, cg=0, **kw):
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    Bd = torch.from_numpy(np.asfortranarray(B)).cuda()
    C = bx.gemm(Ad, Bd, variant=variant, cta_group=cg, **kw)
    torch.cuda.synchronize()
    return C.cpu().numpy()


@pytest.fixture(params=[1, 2], ids=["spi1", "spi2"])
def spi(request):
    bx.lib().bf16x_tune(0, 0, request.param)
    yield request.param
    bx.lib().bf16x_tune(0, 0, 0)


# ---------------------------------------------------------------------------------------
# 1. product sets by value
U = 1 + 2 ** -8 + 2 ** -17     # pieces (1 + 2^-7, -2^-8, 2^-17)
U0 = 1 + 2 ** -7
# with a = (U, -U0), b = (U, U0): Z00 = U0^2 - U0^2 = 0 and Z_ij = u_i u_j otherwise, so
#   bin 1 = 2 u0 u1 = -2^-7 - 2^-14;  Z02 = Z20 = u0 u2 = 2^-17 + 2^-24;  Z11 = 2^-16;
#   Z12 = Z21 = -2^-25;  Z22 = 2^-34
PAPER_VALUE = {
    3: -2 ** -7 - 2 ** -14,                                             # {00, 01, 10}
    5: -2 ** -7 - 2 ** -14 + 2 ** -16 + 2 ** -17 + 2 ** -24,           # + {02, 11} (no Z20: A has 2 pieces)
    6: -2 ** -7 - 2 ** -15 + 2 ** -23,                                  # + {02, 11, 20}
    7: -2 ** -7 - 2 ** -15 + 2 ** -23 - 2 ** -25,                       # + Z12
    8: -2 ** -7 - 2 ** -15 + 2 ** -24,                                  # + Z12 + Z21
    9: -2 ** -7 - 2 ** -15 + 2 ** -24,                                  # + Z22 = 2^-34: below FP32 of the sum
}


def _pattern(m, n, k, seed):
    """A (m x k), B (k x n) zero except one (U, -U0) . (U, U0) pair per output row block at a
    pseudo-random even k, scaled by 2^er (rows) and 2^ec (columns); returns A, B, expected
    scale matrix S with C = S * value(variant)."""
    rng = np.random.default_rng(seed)
    A = np.zeros((m, k), dtype=np.float32, order="F")
    B = np.zeros((k, n), dtype=np.float32, order="F")
    er = rng.integers(-20, 21, size=m)
    ec = rng.integers(-20, 21, size=n)
    kk = 2 * rng.integers(0, k // 2, size=m)                            # each row's pair position
    for r in range(m):
        A[r, kk[r]] = np.float32(U * 2.0 ** er[r])
        A[r, kk[r] + 1] = np.float32(-U0 * 2.0 ** er[r])
    for l in range(0, k, 2):
        B[l, :] = (U * 2.0 ** ec).astype(np.float32)
        B[l + 1, :] = (U0 * 2.0 ** ec).astype(np.float32)
    S = np.ldexp(1.0, er[:, None] + ec[None, :])
    return A, B, S


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("variant", [3, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("shape", [(300, 520, 200), (129, 257, 66)])
def test_product_sets_by_value(orc, shape, variant, cg, spi):
    m, n, k = shape
    A, B, S = _pattern(m, n, k, seed=m + variant)
    want = (S * PAPER_VALUE[variant]).astype(np.float32)
    assert np.array_equal(want.astype(np.float64), S * PAPER_VALUE[variant])      # exact in FP32
    O = orc.gemm(A, B, variant=variant)
    assert np.array_equal(O, want)                                                 # the paper's value
    G = _gpu(A, B, variant, cg=cg)
    assert np.array_equal(G, want), (variant, int(np.sum(G != want)))


# ---------------------------------------------------------------------------------------
# 2. elementwise bound of section II-E
def _gam(n):
    return n * EPS_F / (1 - n * EPS_F)


@pytest.mark.parametrize("dist", ["uniform", "wide", "gauss"])
@pytest.mark.parametrize("k", [64, 1000, 4096])
@pytest.mark.parametrize("variant", [6, 7, 8, 9])
def test_elementwise_error_bound_p321(dist, k, variant):
    """|C - A B| <= 1.01 (gamma_{k+2} + eps_b^3) (|A| |B|) elementwise (P:321 with R11)."""
    m, n = 192, 160
    A = synthetic.by_name(dist, m, k, seed=11 + k)
    B = synthetic.by_name(dist, k, n, seed=12 + k)
    G = _gpu(A, B, variant).astype(np.float64)
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    C64 = A64 @ B64
    bound = 1.01 * (_gam(k + 2) + EPS_B ** 3) * (np.abs(A64) @ np.abs(B64))
    viol = np.abs(G - C64) > bound
    assert not viol.any(), (int(viol.sum()), float(np.max(np.abs(G - C64) / bound)))


# ---------------------------------------------------------------------------------------
# 3. schedule conformance (bit for bit against tests/tc_model.py)
def _stages(variant, cg):
    """Piece-ring stages of the kernel (csrc/gemm_impl.cuh Cfg)."""
    pa, pb = tc_model.PIECES[variant]
    if cg == 1:
        stage = pa * 128 * 64 + pb * 256 * 64
    else:
        stage = pa * 128 * 64 + pb * 128 * 64
    base = 232448 - 1024 - 256 - 1024
    stages = (base - 32768) // stage                  # 32 KB: the C staging buffers ...
    if stages < 4:
        stages = base // stage                        # ... only where 4 stages remain with them
    return min(8, stages)


def _uses_pm(variant, cg, k, m=0, n=0):
    """The library's automatic schedule promotes every MMA at k <= 128 on outputs of at most
    2^20 elements when the tile's k fits the ring (gemm.cu use_pm, launch_s)."""
    return k <= 128 and m * n <= (1 << 20) and -(-k // 32) <= min(4, _stages(variant, cg))


def _interval(variant, cg, spi, k):
    """Promotion interval the dispatcher picks (csrc/gemm_impl.cuh launch_s): a forced spi of
    1 or 2 stages of 32 k, unless the 2-stage ring would have fewer than 4 stages (tile N 256
    per CTA with cta_group 1 and 3 pieces of B: 3 stages) -> 1."""
    stages = _stages(variant, cg)
    if spi == 0 and variant == 3 and cg == 2 and 64 < k <= 256:
        return 128                                    # x3 short k: 128-k intervals (callers exclude PM)
    s = spi if spi in (1, 2) else (2 if (cg == 2 and k > 128) else 1)
    if s == 2 and stages < 4:
        s = 1
    return 32 * s


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("variant", [1, 3, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("dist", ["uniform", "wide", "gauss"])
@pytest.mark.parametrize("shape", [(129, 257, 33), (200, 136, 260)])
def test_kernel_equals_schedule_model(shape, dist, variant, cg, spi):
    m, n, k = shape
    A = synthetic.by_name(dist, m, k, seed=7 * m + k)
    B = synthetic.by_name(dist, k, n, seed=5 * n + k)
    G = _gpu(A, B, variant, cg=cg)
    M = tc_model.simulate(A, B, variant, interval=_interval(variant, cg, spi, k))
    bad = G.view(np.uint32) != M.view(np.uint32)
    assert not bad.any(), (int(bad.sum()), _interval(variant, cg, spi, k))


@pytest.mark.parametrize("variant", [3, 6, 9])
def test_kernel_equals_schedule_model_default(variant):
    """The library's own choice of schedule (no tuning override) on configs[0]'s 64^3 arms, a
    k = 200 problem and a k = 1000 problem: every MMA promoted on its own at k <= 128 (PM),
    128-k intervals for bf16x3 at 128 < k <= 256, 64-k intervals otherwise (2-CTA pairs)."""
    for (m, n, k) in ((64, 64, 64), (96, 160, 1000), (300, 260, 200)):
        for dist in ("uniform", "wide", "gauss"):
            A = synthetic.by_name(dist, m, k, seed=3)
            B = synthetic.by_name(dist, k, n, seed=4)
            G = _gpu(A, B, variant)
            if k <= 128:
                M = tc_model.simulate(A, B, variant, interval=128, promote_every_mma=True)
            else:
                M = tc_model.simulate(A, B, variant, interval=_interval(variant, 2, 0, k))
            assert np.array_equal(G.view(np.uint32), M.view(np.uint32)), (m, n, k, dist)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("variant", [1, 3, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("shape", [(129, 257, 33), (300, 200, 128), (64, 600, 17)])
def test_promote_every_mma_equals_model(shape, variant, cg):
    """Short k (library schedule, k <= 128): each K=16 MMA of each product overwrites a TMEM
    buffer and is added into G with FP32 round-to-nearest in issue order -- bins smallest first
    over the whole k of the tile, then the halves, then the band's pairs -- bit for bit the
    model's promote_every_mma schedule with one group spanning k, ragged k included (a last
    K=16 half cut short)."""
    m, n, k = shape
    for dist in ("uniform", "gauss"):
        A = synthetic.by_name(dist, m, k, seed=m + k + variant)
        B = synthetic.by_name(dist, k, n, seed=n + k)
        G = _gpu(A, B, variant, cg=cg)
        if _uses_pm(variant, cg, k, m, n):
            M = tc_model.simulate(A, B, variant, interval=128, promote_every_mma=True)
        else:                                         # the tile's k does not fit the ring
            M = tc_model.simulate(A, B, variant, interval=_interval(variant, cg, 0, k))
        bad = G.view(np.uint32) != M.view(np.uint32)
        assert not bad.any(), (dist, int(bad.sum()))


def test_stream_k_equals_model():
    """Hybrid stream-K, bit for bit: with the grid capped at 4 CTA pairs (bf16x_max_ctas), a
    512 x 768 output (2 x 3 tiles of 256 x 256) and k = 768 (12 intervals of 64 k) runs every
    tile in stream-K mode: the 72 intervals are dealt 18 per cluster, so tiles 1 and 4 are cut
    in two.  An uncut tile is the RN promotion of its 12 interval partials; a cut tile is
    RN(G_owner + G_contributor), each the promotion of its own intervals (csrc/gemm_impl.cuh
    WorkIter and the fix-up)."""
    m, n, k, v = 512, 768, 768, 6
    A = synthetic.uniform(m, k, seed=21)
    B = synthetic.uniform(k, n, seed=22)
    L = bx.lib()
    L.bf16x_max_ctas(8)
    try:
        G = _gpu(A, B, v)
    finally:
        L.bf16x_max_ctas(0)
    parts = tc_model.interval_partials(A, B, v, interval=64)
    n_int, ncl, tiles_n = 12, 4, 3
    U = 6 * n_int
    bounds = [U * c // ncl for c in range(ncl + 1)]
    want = np.empty((m, n), dtype=np.float32)
    for t in range(6):
        tm, tn = t // tiles_n, t % tiles_n                 # raster: one tile row per group (tiles_n <= 16)
        rs, cs = slice(256 * tm, 256 * tm + 256), slice(256 * tn, 256 * tn + 256)
        lo, hi = t * n_int, (t + 1) * n_int
        cut = [b - lo for b in bounds if lo < b < hi]
        P = [p[rs, cs] for p in parts]
        if not cut:
            want[rs, cs] = tc_model.promote(P)
        else:
            assert len(cut) == 1
            want[rs, cs] = (tc_model.promote(P[:cut[0]]) + tc_model.promote(P[cut[0]:])).astype(np.float32)
    assert np.array_equal(G.view(np.uint32), want.view(np.uint32)), int(np.sum(G != want))
