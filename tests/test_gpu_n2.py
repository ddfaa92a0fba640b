"""N2 rows on the GPU: power-of-two scaled pieces (R29, the
split exact below the paper's exponent -110) and the FP64 final collection of the
bins, the paper's "d" variants (R30), against the oracle.

Acceptance as for the other variants: split bit-exact; GEMM normwise error <= 2x the
oracle's for the same variant and options; bit-exact where the arithmetic is exact.
"""
import ctypes

import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu

RATIO = 2.0
CHUNK = 1 << 27


def _gpu(A, B, C=None, alpha=1.0, beta=0.0, variant=6, **kw):
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    Bd = torch.from_numpy(np.asfortranarray(B)).cuda()
    Cd = None if C is None else torch.from_numpy(np.asfortranarray(C)).cuda()
    out = bx.gemm(Ad, Bd, Cd, alpha=alpha, beta=beta, variant=variant, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy()


# ---------------------------------------------------------------------------------------
# scaled split (R29)
# ---------------------------------------------------------------------------------------
def test_scaled_split_all_2_32_patterns(orc):
    """Every FP32 pattern through the scaled split (fast cvt.rn path and the integer path
    for NaN / Inf / the b0-overflow band), bit-exact against the oracle."""
    dev = torch.device("cuda")
    first_bad = None
    for c in range((1 << 32) // CHUNK):
        first = c * CHUNK
        x = torch.arange(first, first + CHUNK, dtype=torch.int64, device=dev).to(torch.int32).view(torch.float32)
        g = bx.split(x, scaled=True)
        want = orc.split_scaled_patterns(first, CHUNK)
        for q in range(3):
            got = g[q].cpu().numpy().view(np.uint16)
            if not np.array_equal(got, want[q]):
                i = int(np.flatnonzero(got != want[q])[0])
                first_bad = (hex(first + i), q, hex(int(got[i])), hex(int(want[q][i])))
                break
        if first_bad:
            break
    assert first_bad is None, f"pattern/piece/gpu/oracle: {first_bad}"


@pytest.mark.parametrize("rows,cols,ld", [(7, 3, 9), (129, 65, 130), (1000, 17, 1003)])
def test_scaled_split_transposed_layout(orc, rows, cols, ld):
    X = synthetic.wide(ld, cols, seed=rows + cols, E=120)
    Xd = torch.from_numpy(np.asfortranarray(X)).cuda()
    want = orc.split_scaled(np.asfortranarray(X[:rows, :]))
    ldt = cols + 3
    outs = [torch.zeros((rows * ldt,), dtype=torch.uint16, device="cuda") for _ in range(3)]
    L = bx.lib()
    rc = L.bf16x_split_ex(rows, cols, Xd.data_ptr(), ld, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(),
                          ldt, bx.SCALED_PIECES | bx.SPLIT_TRANSPOSED, None)
    assert rc == 0
    torch.cuda.synchronize()
    for q in range(3):
        got = outs[q].cpu().numpy().view(np.uint16).reshape(rows, ldt)[:, :cols]
        assert np.array_equal(got, want[q])


# ---------------------------------------------------------------------------------------
# GEMM with scaled pieces (R29)
# ---------------------------------------------------------------------------------------
@pytest.fixture(params=[0, 2], ids=["mc_auto", "mc2"])
def mc(request):
    """0: library default (no multicast at these sizes); 2: two CTA pairs per cluster sharing B."""
    bx.lib().bf16x_multicast(request.param)
    yield request.param
    bx.lib().bf16x_multicast(0)


@pytest.mark.parametrize("variant", [1, 3, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("shape", [(129, 257, 33), (333, 517, 77), (512, 384, 1000), (700, 300, 200)])
def test_scaled_equals_unscaled_on_normal_range_inputs(shape, variant, mc):
    """U[-1,1] inputs: nothing leaves the normal range, so scaling each band's accumulator by
    2^-8 (scale-input-d) on the tensor core reproduces the unscaled GEMM bit for bit (both
    promotion-interval lengths, alpha/beta included) -- the hardware check that the scale is
    applied exactly once per band, to the accumulator only."""
    m, n, k = shape
    A = synthetic.uniform(m, k, seed=m + k)
    B = synthetic.uniform(k, n, seed=n + 3 * k)
    C = synthetic.uniform(m, n, seed=5)
    for spi in (1, 2):
        bx.lib().bf16x_tune(0, 0, spi)
        try:
            u = _gpu(A, B, C, alpha=0.5, beta=-2.0, variant=variant)
            s = _gpu(A, B, C, alpha=0.5, beta=-2.0, variant=variant, scaled=True)
        finally:
            bx.lib().bf16x_tune(0, 0, 0)
        assert np.array_equal(u.view(np.uint32), s.view(np.uint32)), (spi, variant)


@pytest.mark.parametrize("variant", [3, 6, 9])
def test_scaled_below_minus_110_vs_oracle(orc, variant):
    """A scaled by 2^-115 and 2^-121, B by 2^100 (the oracle pins: near-homogeneous at -115, at
    normal-range accuracy at -121).  GPU scaled-piece GEMM within 2x of the oracle's scaled
    error; the unscaled GPU GEMM is > 20x worse for x6 / x9."""
    A = synthetic.uniform(300, 640, seed=11, lo=0.0625, hi=1.0)
    A[::3] = -A[::3]
    B = synthetic.uniform(640, 260, seed=12)
    C64 = orc.dgemm(A, B)
    Bs = (B.astype(np.float64) * 2.0 ** 100).astype(np.float32)
    for sh in (-115, -121):
        As = (A.astype(np.float64) * 2.0 ** sh).astype(np.float32)
        g = _gpu(As, Bs, variant=variant, scaled=True).astype(np.float64) * 2.0 ** (-sh - 100)
        o = orc.gemm(As, Bs, variant=variant, scaled=True).astype(np.float64) * 2.0 ** (-sh - 100)
        eg, eo = orc.normwise_error(g, C64, A, B), orc.normwise_error(o, C64, A, B)
        assert eg <= RATIO * eo, (sh, eg, eo)
        u = _gpu(As, Bs, variant=variant).astype(np.float64) * 2.0 ** (-sh - 100)
        if variant >= 6:
            assert orc.normwise_error(u, C64, A, B) > 20 * eg


def test_scaled_exact_on_subnormal_integers(orc):
    """A = integers x 2^-140 (FP32 subnormals), B = integers x 2^120: the scaled-piece GEMM
    is exact on the tensor core (BF16 subnormal inputs and products kept), like the oracle."""
    g = np.random.default_rng(140)
    Ai = g.integers(-1000, 1001, size=(200, 160))
    Bi = g.integers(-200, 201, size=(160, 130))
    A = (Ai.astype(np.float64) * 2.0 ** -140).astype(np.float32)
    B = (Bi.astype(np.float64) * 2.0 ** 120).astype(np.float32)
    exact = (Ai @ Bi).astype(np.float64) * 2.0 ** -20
    assert np.abs(Ai @ Bi).max() < 2 ** 24
    for v in (3, 6, 9):
        assert np.array_equal(orc.gemm(A, B, variant=v, scaled=True).astype(np.float64), exact)
        assert np.array_equal(_gpu(A, B, variant=v, scaled=True).astype(np.float64), exact), v


def test_scaled_pre_split_pieces_through_gemm_ex(orc):
    """Scaled pieces from bf16x_split_ex fed to bf16x_gemm_ex (K-major A via the transposed
    split, B in place) equal the library's own scaled path bit for bit."""
    m, n, k = 300, 200, 136
    A = synthetic.wide(m, k, seed=3, E=30)
    B = synthetic.wide(k, n, seed=4, E=30)
    Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
    Bd = torch.from_numpy(np.asfortranarray(B)).cuda()
    Ap = torch.zeros(3 * m * k, dtype=torch.uint16, device="cuda")
    Bp = torch.zeros(3 * n * k, dtype=torch.uint16, device="cuda")
    L = bx.lib()
    base = Ap.data_ptr()
    assert L.bf16x_split_ex(m, k, Ad.data_ptr(), m, base, base + 2 * m * k, base + 4 * m * k, k,
                            bx.SCALED_PIECES | bx.SPLIT_TRANSPOSED, None) == 0
    bb = Bp.data_ptr()
    assert L.bf16x_split_ex(k, n, Bd.data_ptr(), k, bb, bb + 2 * n * k, bb + 4 * n * k, k, bx.SCALED_PIECES,
                            None) == 0
    C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device="cuda")
    bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), m, variant=6, flags=bx.SCALED_PIECES,
                A_pieces=base, ldap=k, a_plane=m * k, B_pieces=bb, ldbp=k, b_plane=n * k)
    torch.cuda.synchronize()
    want = _gpu(A, B, variant=6, scaled=True)
    assert np.array_equal(C.cpu().numpy(), want)


# ---------------------------------------------------------------------------------------
# FP64 collection, "d" variants (R30)
# ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("scaled", [False, True])
@pytest.mark.parametrize("variant", [3, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("shape", [(129, 257, 33), (333, 517, 77), (256, 512, 1000), (700, 300, 2000)])
def test_fp64_combine_vs_oracle(orc, shape, variant, scaled):
    m, n, k = shape
    A = synthetic.uniform(m, k, seed=m + 5 * k)
    B = synthetic.uniform(k, n, seed=n + 9 * k)
    g = _gpu(A, B, variant=variant, fp64_combine=True, scaled=scaled)
    o = orc.gemm(A, B, variant=variant, fp64_combine=True, scaled=scaled)
    C64 = orc.dgemm(A, B)
    eg, eo = orc.normwise_error(g, C64, A, B), orc.normwise_error(o, C64, A, B)
    assert eg <= RATIO * eo, (eg, eo)


@pytest.mark.parametrize("dist", ["wide", "gauss"])
def test_fp64_combine_exponent_spread(orc, dist):
    """Wide / Gaussian-exponent inputs: mean ratio over 4 seeds <= 2."""
    r = []
    for s in range(4):
        A = synthetic.by_name(dist, 200, 300, seed=50 + s)
        B = synthetic.by_name(dist, 300, 260, seed=60 + s)
        g = _gpu(A, B, variant=6, fp64_combine=True)
        o = orc.gemm(A, B, variant=6, fp64_combine=True)
        C64 = orc.dgemm(A, B)
        r.append(orc.normwise_error(g, C64, A, B) / orc.normwise_error(o, C64, A, B))
    assert np.mean(r) <= RATIO, r


def test_fp64_combine_alpha_beta_ragged_and_stream_k(orc):
    """alpha/beta epilogue on the FP64-collected value (rounded once, then fmaf(alpha, z,
    beta*C)), ragged tiles, and a tile count that triggers the stream-K fix-up (FP64 partial
    accumulators exchanged between clusters)."""
    for (m, n, k) in [(333, 517, 77), (2304, 2560, 512), (4096, 1280, 640)]:
        A = synthetic.uniform(m, k, seed=m)
        B = synthetic.uniform(k, n, seed=n)
        C = synthetic.uniform(m, n, seed=k)
        g = _gpu(A, B, C, alpha=1.5, beta=-0.5, variant=6, fp64_combine=True)
        o = orc.gemm(A, B, C, alpha=1.5, beta=-0.5, variant=6, fp64_combine=True)
        ref = 1.5 * orc.dgemm(A, B) - 0.5 * C.astype(np.float64)
        eg = np.linalg.norm(g - ref) / np.linalg.norm(ref)
        eo = np.linalg.norm(o - ref) / np.linalg.norm(ref)
        assert eg <= RATIO * eo, (m, n, k, eg, eo)


def test_fp64_combine_large_k_sampled(orc):
    """configs[1]-like k = 4096 (m = n = 1024, sampled columns): x6d within 2x of the oracle's
    x6d and not worse than the GPU's own x6 (bin 0 is never rounded against the small bins in
    FP32; their sum is formed once, in FP64)."""
    m = n = 1024
    k = 4096
    A = synthetic.uniform(m, k, seed=1)
    B = synthetic.uniform(k, n, seed=2)
    cols = np.arange(0, n, 16)
    C64 = orc.dgemm(A, B, cols=cols)
    g6 = _gpu(A, B, variant=6)[:, cols]
    g6d = _gpu(A, B, variant=6, fp64_combine=True)[:, cols]
    o6d = orc.gemm(A, B, variant=6, fp64_combine=True, cols=cols)
    e6 = orc.normwise_error(g6, C64, A, B[:, cols])
    e6d = orc.normwise_error(g6d, C64, A, B[:, cols])
    eo = orc.normwise_error(o6d, C64, A, B[:, cols])
    assert e6d <= RATIO * eo, (e6d, eo)
    assert e6d <= 1.02 * e6, (e6d, e6)
