"""A's pieces in A's own layout (BF16X_A_PIECES_MN; the tensor cores read them MN-major).

bf16x_gemm splits A without a transpose and the K2 kernel loads it with the 128-byte swizzle and
tcgen05 a_major = MN.  The MMA products and their order are the same as with K-major pieces
(bf16x_split_t), so every output must be bit-identical between the two layouts -- for every
variant, CTA mode, promotion interval, multicast, stream-K, the promote-every-MMA short-k
schedule, scaled pieces and the FP64 collection, and at ragged m / k (TMA out-of-range rows and k
read as zero).  The host-buffer pipelines (MN pieces of row blocks of A) are compared with bf16x_gemm
in test_gpu_gemm.py.  The parity of the layout-independent arithmetic itself is covered by the oracle
comparisons (test_gpu_gemm.py, test_gpu_schedule.py), which now run on the MN path."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu


def _kmajor_gemm(A, B, variant, flags=0):
    """C from K-major pieces of A (bf16x_split_t) and B's pieces, through bf16x_gemm_ex."""
    m, k = A.shape
    n = B.shape[1]
    pa, pb = (2, 3) if variant == 5 else (bx.PIECES.get(variant, 3),) * 2
    kp = (k + 7) // 8 * 8
    scaled = bool(flags & bx.SCALED_PIECES)
    Ap = torch.zeros(3 * max(1, m * kp), dtype=torch.uint16, device="cuda")
    Bp = torch.zeros(3 * max(1, n * kp), dtype=torch.uint16, device="cuda")
    L = bx.lib()
    st = torch.cuda.current_stream().cuda_stream
    a = [Ap.data_ptr() + q * m * kp * 2 if q < pa else None for q in range(3)]
    b = [Bp.data_ptr() + q * n * kp * 2 if q < pb else None for q in range(3)]
    L.bf16x_split_ex.argtypes = [bx._i64, bx._i64, bx._vp, bx._i64, bx._vp, bx._vp, bx._vp, bx._i64, bx._u, bx._vp]
    fa = bx.SPLIT_TRANSPOSED | (bx.SCALED_PIECES if scaled else 0)
    if scaled:
        assert L.bf16x_split_ex(m, k, A.data_ptr(), m, a[0], a[1], a[2], kp, fa, st) == 0
        assert L.bf16x_split_ex(k, n, B.data_ptr(), k, b[0], b[1], b[2], kp, bx.SCALED_PIECES, st) == 0
    else:
        assert L.bf16x_split_t(m, k, A.data_ptr(), m, a[0], a[1], a[2], kp, st) == 0
        assert L.bf16x_split(k, n, B.data_ptr(), k, b[0], b[1], b[2], kp, st) == 0
    C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device="cuda")
    bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), m, variant=variant, flags=flags,
                A_pieces=Ap.data_ptr(), ldap=kp, a_plane=m * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp)
    return C


def _internal_gemm(A, B, variant, flags=0):
    """bf16x_gemm_ex without pieces: the library splits A in its own layout (MN pieces)."""
    m, k = A.shape
    n = B.shape[1]
    C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device="cuda")
    bx.gemm_raw(m, n, k, 1.0, A.data_ptr(), m, B.data_ptr(), k, 0.0, C.data_ptr(), m, variant=variant, flags=flags)
    return C


def _operands(m, n, k, seed, dist="uniform"):
    if dist == "wide":
        A, B = synthetic.wide(m, k, seed=seed), synthetic.wide(k, n, seed=seed + 1)
    else:
        A, B = synthetic.uniform(m, k, seed=seed), synthetic.uniform(k, n, seed=seed + 1)
    return (torch.from_numpy(np.asfortranarray(A)).cuda(), torch.from_numpy(np.asfortranarray(B)).cuda())


def _same(X, Y):
    torch.cuda.synchronize()
    assert torch.equal(X.view(torch.int32), Y.view(torch.int32)), \
        f"{(X.view(torch.int32) != Y.view(torch.int32)).sum().item()} elements differ"


@pytest.fixture
def tune():
    yield bx.lib().bf16x_tune
    bx.lib().bf16x_tune(0, 0, 0)
    bx.lib().bf16x_multicast(0)
    bx.lib().bf16x_fused_a(-1)


SHAPES = [(64, 64, 64), (129, 257, 33), (333, 517, 77), (20, 600, 48), (1000, 300, 1000), (1, 5, 7), (130, 70, 200),
          (777, 129, 300)]


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("variant", [1, 3, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_mn_pieces_bit_identical_to_kmajor(tune, shape, variant, cg):
    tune(cg, 0, 0)
    bx.lib().bf16x_fused_a(0)     # x9: the pre-pass path on both sides
    A, B = _operands(*shape, seed=sum(shape) + variant)
    _same(_internal_gemm(A, B, variant), _kmajor_gemm(A, B, variant))


@pytest.mark.parametrize("spi", [1, 2, 4])
@pytest.mark.parametrize("variant", [3, 6, 9])
def test_mn_promotion_intervals(tune, spi, variant):
    if spi == 4 and variant != 3:
        pytest.skip("128-k intervals: x1 / x3 only")
    tune(0, 0, spi)
    bx.lib().bf16x_fused_a(0)
    A, B = _operands(300, 700, 1500, seed=spi + variant, dist="wide")
    _same(_internal_gemm(A, B, variant), _kmajor_gemm(A, B, variant))


@pytest.mark.parametrize("variant", [3, 6])
def test_mn_multicast_and_stream_k(tune, variant):
    """Two CTA pairs sharing B (multicast) and a stream-K tail (tiles > 74, not a multiple)."""
    bx.lib().bf16x_multicast(2)
    A, B = _operands(2304, 2560, 1024, seed=variant)
    _same(_internal_gemm(A, B, variant), _kmajor_gemm(A, B, variant))
    bx.lib().bf16x_multicast(1)
    _same(_internal_gemm(A, B, variant), _kmajor_gemm(A, B, variant))


MC4_SHAPES = [(2304, 2560, 1024), (1000, 1300, 520), (300, 700, 200), (513, 257, 160), (4096, 512, 256)]


@pytest.mark.parametrize("variant", [1, 3, 5, 6, 7, 8, 9])
@pytest.mark.parametrize("shape", MC4_SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_mn_multicast_2x2(tune, shape, variant):
    """2 x 2 CTA pairs per cluster (bf16x_multicast(4)): A's 64-row boxes shared along each row of
    the cluster block, B's halves down each column.  Each tile's MMAs are the same, so with
    BF16X_NO_STREAM_K the output equals the one-pair schedule's bit for bit (ragged m, n, k:
    partial super-tiles whose out-of-range pairs read zeros); the default schedule (a stream-K
    tail where the super-tile count is not a multiple of the cluster count) is repeatable and
    equals the K-major path, which falls back to B-only multicast."""
    A, B = _operands(*shape, seed=7 * variant + shape[2], dist="wide")
    bx.lib().bf16x_fused_a(0)
    bx.lib().bf16x_multicast(1)
    want = _internal_gemm(A, B, variant, flags=bx.NO_STREAM_K)
    bx.lib().bf16x_multicast(4)
    _same(_internal_gemm(A, B, variant, flags=bx.NO_STREAM_K), want)
    _same(_kmajor_gemm(A, B, variant, flags=bx.NO_STREAM_K), want)
    first = _internal_gemm(A, B, variant)
    _same(_internal_gemm(A, B, variant), first)
    if variant == 9:
        bx.lib().bf16x_fused_a(-1)    # fused A is not taken with multicast: same bits
        _same(_internal_gemm(A, B, variant, flags=bx.NO_STREAM_K), want)


@pytest.mark.parametrize("variant", [3, 6, 9])
def test_mn_short_k_promote_every_mma(tune, variant):
    bx.lib().bf16x_fused_a(0)
    for shape in [(200, 300, 16), (512, 512, 100), (96, 1000, 128)]:
        A, B = _operands(*shape, seed=variant, dist="wide")
        _same(_internal_gemm(A, B, variant), _kmajor_gemm(A, B, variant))


@pytest.mark.parametrize("flag", ["scaled", "fp64"])
@pytest.mark.parametrize("variant", [3, 6, 9])
def test_mn_n2_options(tune, flag, variant):
    f = bx.SCALED_PIECES if flag == "scaled" else bx.FP64_COMBINE
    bx.lib().bf16x_fused_a(0)
    A, B = _operands(333, 400, 500, seed=variant, dist="wide")
    _same(_internal_gemm(A, B, variant, f), _kmajor_gemm(A, B, variant, f))


def test_split_operands_ex_mn_equals_split():
    """bf16x_split_operands_ex(BF16X_A_PIECES_MN) writes exactly bf16x_split's pieces of A and B."""
    m, n, k = 333, 250, 129
    A, B = _operands(m, n, k, seed=5, dist="wide")
    mp, kp = (m + 7) // 8 * 8, (k + 7) // 8 * 8
    Ap = torch.zeros(3 * mp * k, dtype=torch.uint16, device="cuda")
    Bp = torch.zeros(3 * n * kp, dtype=torch.uint16, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    assert bx.lib().bf16x_split_operands_ex(m, n, k, A.data_ptr(), m, B.data_ptr(), k, 3, Ap.data_ptr(), mp, mp * k,
                                            Bp.data_ptr(), kp, n * kp, bx.A_PIECES_MN, st) == 0
    torch.cuda.synchronize()
    for X, P, rows, cols, ld, plane in ((A, Ap, m, k, mp, mp * k), (B, Bp, k, n, kp, n * kp)):
        want = bx.split(X, pieces=3)
        for q in range(3):
            got = P[q * plane:q * plane + ld * cols].view(cols, ld)[:, :rows].t()
            assert torch.equal(got, want[q]), q

