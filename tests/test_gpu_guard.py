"""Guard bands: out-of-bounds write and input-clobber detection for every kernel family.

compute-sanitizer is closed on this GPU pool, so this is the memcheck
substitute for writes: every operand and result lives strictly inside a larger device buffer whose
surroundings (rows between m and ld, whole columns before and after, bytes before and after the
allocation's used range) hold a sentinel bit pattern.  After each call the sentinel must be intact,
inputs bit-identical to before, and the results still correct (bit-identical to the same call on
plain buffers).  Covered: the splits (same layout, transposed, both operands in either A layout),
the GEMM in each schedule (1-CTA, 2-CTA pairs, TMA multicast, stream-K tail, promote-every-MMA
short k, scaled pieces, FP64 collection, fused A, beta != 0, the FP32 accumulator carry and a
caller workspace of exactly bf16x_gemm_workspace_size bytes) and the LU factorisation."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu

SENT = 0x7FBADBAD            # a NaN bit pattern no kernel writes


def _guarded(rows, cols, data=None, pad_r=(5, 11), pad_c=(3, 2), dtype=torch.float32):
    """(big, view): view = big[pad_r[0] : pad_r[0] + rows, pad_c[0] : pad_c[0] + cols], column-major,
    ld = rows + pad_r[0] + pad_r[1]; everything else in `big` holds the sentinel."""
    R, Cc = rows + sum(pad_r), cols + sum(pad_c)
    big = torch.empty_strided((R, Cc), (1, R), dtype=dtype, device="cuda")
    big.view(torch.int32 if dtype == torch.float32 else torch.int16).fill_(SENT if dtype == torch.float32 else 0x7BAD)
    view = big[pad_r[0]:pad_r[0] + rows, pad_c[0]:pad_c[0] + cols]
    if data is not None:
        view.copy_(torch.as_tensor(data, device="cuda"))
    return big, view


def _outside_intact(big, view_slices):
    mask = torch.ones(big.shape, dtype=torch.bool, device="cuda")
    mask[view_slices] = False
    bits = big.view(torch.int32)[mask]
    return bool((bits == SENT).all().item())


def _ld(t):
    return t.stride(1)


CASES = [  # (m, n, k, variant, hooks)
    (129, 257, 33, 6, {}),
    (333, 517, 77, 3, {"cg": 1}),
    (333, 517, 77, 9, {}),                       # fused A (x9 default)
    (333, 517, 77, 9, {"fused_a": 0}),
    (200, 300, 16, 6, {}),                       # promote-every-MMA short k
    (777, 129, 300, 5, {}),
    (2304, 2560, 1024, 6, {"mc": 1}),            # stream-K tail (90 tiles, 16 intervals)
    (2304, 2560, 520, 3, {"mc": 2}),             # TMA multicast, ragged k
    (1000, 1300, 520, 6, {"mc": 4}),             # 2 x 2 pairs sharing A and B, ragged super-tiles
]


@pytest.fixture
def hooks():
    L = bx.lib()

    def set_(h):
        L.bf16x_tune(h.get("cg", 0), 0, 0)
        L.bf16x_multicast(h.get("mc", 0))
        L.bf16x_fused_a(h.get("fused_a", -1))
    yield set_
    L.bf16x_tune(0, 0, 0)
    L.bf16x_multicast(0)
    L.bf16x_fused_a(-1)


@pytest.mark.parametrize("flags", [0, bx.SCALED_PIECES, bx.FP64_COMBINE], ids=["plain", "scaled", "fp64"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}x{c[1]}x{c[2]}_x{c[3]}_{'_'.join(f'{a}{b}' for a, b in c[4].items())}")
def test_gemm_guard_bands(hooks, case, flags):
    m, n, k, v, h = case
    if flags == bx.FP64_COMBINE and v == 1:
        pytest.skip("no FP64 collection for x1")
    hooks(h)
    A = synthetic.wide(m, k, seed=m + k)
    B = synthetic.wide(k, n, seed=n + k)
    C0 = synthetic.uniform(m, n, seed=m + n)
    Ab, Av = _guarded(m, k, A)
    Bb, Bv = _guarded(k, n, B, pad_r=(2, 6), pad_c=(1, 4))
    Cb, Cv = _guarded(m, n, C0, pad_r=(7, 1), pad_c=(2, 3))
    A_before, B_before = Ab.clone(), Bb.clone()
    bx.gemm_raw(m, n, k, 1.25, Av.data_ptr(), _ld(Av), Bv.data_ptr(), _ld(Bv), 0.5, Cv.data_ptr(), _ld(Cv), variant=v,
                flags=flags)
    torch.cuda.synchronize()
    assert torch.equal(Ab.view(torch.int32), A_before.view(torch.int32)), "A modified"
    assert torch.equal(Bb.view(torch.int32), B_before.view(torch.int32)), "B modified"
    assert _outside_intact(Cb, (slice(7, 7 + m), slice(2, 2 + n))), "write outside C"
    # same call on plain buffers: same bits
    Ad, Bd = torch.from_numpy(np.asfortranarray(A)).cuda(), torch.from_numpy(np.asfortranarray(B)).cuda()
    Cd = torch.from_numpy(np.asfortranarray(C0)).cuda()
    bx.gemm_raw(m, n, k, 1.25, Ad.data_ptr(), m, Bd.data_ptr(), k, 0.5, Cd.data_ptr(), m, variant=v, flags=flags)
    torch.cuda.synchronize()
    assert torch.equal(Cv.contiguous().view(torch.int32), Cd.contiguous().view(torch.int32))


@pytest.mark.parametrize("variant", [3, 6, 9])
def test_gemm_workspace_and_carry_guard_bands(hooks, variant):
    """Caller workspace of exactly bf16x_gemm_workspace_size bytes inside a sentinel-filled
    allocation, and a k-chunked call through the FP32 accumulator carry (chunk 1 ACC_OUT into a
    guarded carry buffer, chunk 2 ACC_IN into C; the carry shares C's leading dimension): nothing
    outside the workspace, the carry's m x n block or C's is written, and the result equals the
    unchunked call bit for bit (chunk edge on a 128 multiple, BF16X_NO_STREAM_K)."""
    hooks({"fused_a": 0})
    m, n, k, k1 = 333, 270, 600, 256
    A = synthetic.uniform(m, k, seed=1)
    B = synthetic.uniform(k, n, seed=2)
    Ad, Bd = torch.from_numpy(np.asfortranarray(A)).cuda(), torch.from_numpy(np.asfortranarray(B)).cuda()
    ws = bx.workspace_size(m, n, k, variant)
    pad = 4096
    W = torch.empty(ws + 2 * pad, dtype=torch.uint8, device="cuda").fill_(0xA5)
    Cb, Cv = _guarded(m, n)
    Gb, Gv = _guarded(m, n)                                     # same padding -> same ld as C
    L = bx.lib()
    st = torch.cuda.current_stream().cuda_stream
    f = bx.NO_STREAM_K
    assert L.bf16x_gemm_ex(m, n, k1, 1.0, Ad.data_ptr(), m, Bd.data_ptr(), k, 0.0, Cv.data_ptr(), _ld(Cv), variant,
                           f | bx.ACC_OUT, None, 0, 0, None, 0, 0, Gv.data_ptr(), W.data_ptr() + pad, ws, st) == 0
    torch.cuda.synchronize()
    assert _outside_intact(Cb, (slice(5, 5 + m), slice(3, 3 + n))) and \
        (Cv.contiguous().view(torch.int32) == SENT).all(), "C written by an ACC_OUT call"
    assert L.bf16x_gemm_ex(m, n, k - k1, 1.0, Ad.data_ptr() + k1 * m * 4, m, Bd.data_ptr() + k1 * 4, k, 0.0,
                           Cv.data_ptr(), _ld(Cv), variant, f | bx.ACC_IN, None, 0, 0, None, 0, 0, Gv.data_ptr(),
                           W.data_ptr() + pad, ws, st) == 0
    torch.cuda.synchronize()
    assert (W[:pad] == 0xA5).all() and (W[pad + ws:] == 0xA5).all(), "write outside the workspace"
    assert _outside_intact(Cb, (slice(5, 5 + m), slice(3, 3 + n))), "write outside C"
    assert _outside_intact(Gb, (slice(5, 5 + m), slice(3, 3 + n))), "write outside the carry"
    want = bx.gemm(Ad, Bd, variant=variant, no_stream_k=True)
    torch.cuda.synchronize()
    assert torch.equal(Cv.contiguous().view(torch.int32), want.contiguous().view(torch.int32))


def test_split_guard_bands():
    """K1 into piece planes with ldp > rows, and both operands in one launch (A transposed or in its
    own layout): no write outside each plane's rows x cols block, the source unchanged."""
    L = bx.lib()
    st = torch.cuda.current_stream().cuda_stream
    m, n, k = 333, 250, 129
    A = synthetic.wide(m, k, seed=3)
    B = synthetic.wide(k, n, seed=4)
    Ab, Av = _guarded(m, k, A)
    Bb, Bv = _guarded(k, n, B)
    A_before, B_before = Ab.clone(), Bb.clone()
    # same layout (ldp = m + 13) and transposed (ldp = k + 7) into guarded uint16 planes
    for transpose, rows, cols, ldp in ((False, m, k, m + 13), (True, k, m, k + 7)):
        P = torch.empty(3 * ldp * cols + 64, dtype=torch.int16, device="cuda").fill_(0x7BAD)
        base = P.data_ptr() + 64
        bx.split_raw(m, k, Av.data_ptr(), _ld(Av), base, base + 2 * ldp * cols, base + 4 * ldp * cols, ldp,
                     transpose=transpose)
        torch.cuda.synchronize()
        assert (P[:32] == 0x7BAD).all() and (P[32 + 3 * ldp * cols:] == 0x7BAD).all(), transpose
        for q in range(3):
            plane = P[32 + q * ldp * cols:32 + (q + 1) * ldp * cols].view(cols, ldp)
            assert (plane[:, rows:] == 0x7BAD).all(), (transpose, q)
    # both operands in one launch, K-major A and A in its own layout
    for flags, ldap, aplane in ((0, k + 7, (k + 7) * m), (bx.A_PIECES_MN, m + 11, (m + 11) * k)):
        ldbp = k + 9
        Ap = torch.empty(3 * aplane + 64, dtype=torch.int16, device="cuda").fill_(0x7BAD)
        Bp = torch.empty(3 * ldbp * n + 64, dtype=torch.int16, device="cuda").fill_(0x7BAD)
        assert L.bf16x_split_operands_ex(m, n, k, Av.data_ptr(), _ld(Av), Bv.data_ptr(), _ld(Bv), 3,
                                         Ap.data_ptr() + 64, ldap, aplane, Bp.data_ptr() + 64, ldbp, ldbp * n, flags,
                                         st) == 0
        torch.cuda.synchronize()
        acols, arows = (k, m) if flags else (m, k)
        for q in range(3):
            pa = Ap[32 + q * aplane:32 + q * aplane + ldap * acols].view(acols, ldap)
            assert (pa[:, arows:] == 0x7BAD).all(), (flags, q)
            pb = Bp[32 + q * ldbp * n:32 + (q + 1) * ldbp * n].view(n, ldbp)
            assert (pb[:, k:] == 0x7BAD).all(), (flags, q)
        assert (Ap[:32] == 0x7BAD).all() and (Ap[32 + 3 * aplane:] == 0x7BAD).all()
        assert (Bp[:32] == 0x7BAD).all() and (Bp[32 + 3 * ldbp * n:] == 0x7BAD).all()
    assert torch.equal(Ab.view(torch.int32), A_before.view(torch.int32))
    assert torch.equal(Bb.view(torch.int32), B_before.view(torch.int32))


@pytest.mark.parametrize("n", [300, 777])
def test_getrf_guard_bands(n):
    """LU of a matrix view with ld > n inside a sentinel-filled buffer, through the C ABI: nothing
    outside the n x n block and the n pivots is written; the factors equal those of a plain call."""
    L = bx.lib()
    A = synthetic.uniform(n, n, seed=n)
    Ab, Av = _guarded(n, n, A, pad_r=(9, 5), pad_c=(4, 6))
    piv = torch.empty(n + 64, dtype=torch.int32, device="cuda").fill_(SENT)
    import ctypes
    info = ctypes.c_int(0)
    rc = L.bf16x_getrf(n, Av.data_ptr(), _ld(Av), piv.data_ptr() + 128, 3, 64, ctypes.byref(info))
    torch.cuda.synchronize()
    assert rc == 0 and info.value == 0
    assert _outside_intact(Ab, (slice(9, 9 + n), slice(4, 4 + n))), "write outside the matrix"
    assert (piv[:32] == SENT).all() and (piv[32 + n:] == SENT).all(), "write outside ipiv"
    LU, ipiv, _ = bx.getrf(torch.from_numpy(np.asfortranarray(A)).cuda(), variant=3, nb=64)
    torch.cuda.synchronize()
    assert torch.equal(Av.contiguous().view(torch.int32), LU.contiguous().view(torch.int32))
    assert torch.equal(piv[32:32 + n], ipiv)


def test_guard_detector_sees_a_stray_write():
    """The detector itself: one element written just past the view (row m, inside ld) is found."""
    Cb, Cv = _guarded(40, 30, pad_r=(7, 1), pad_c=(2, 3))
    assert _outside_intact(Cb, (slice(7, 47), slice(2, 32)))
    Cb[47, 10] = 1.0
    assert not _outside_intact(Cb, (slice(7, 47), slice(2, 32)))
