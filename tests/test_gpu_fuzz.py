"""Seeded random sweep of the GEMM boundary (bf16x_gemm_ex): shapes 1..700 x 1..700 x 1..1200,
every variant, both CTA modes, random leading-dimension padding, alpha / beta (beta = 0 or not),
the N2 flags (scaled pieces, FP64 collection) and BF16X_NO_STREAM_K, through three entry paths:
the library's own split (A in its own layout), pre-split K-major A pieces (bf16x_split_t) and
pre-split pieces in A's own layout (bf16x_split + BF16X_A_PIECES_MN).  All three must agree bit
for bit, and the result must meet the parity bar against the oracle (normwise error <= 2x the
oracle's on uniform inputs, P:257-277 with R19's alpha / beta)."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu

RATIO = 2.0
PA = {1: 1, 3: 2, 5: 2, 6: 3, 7: 3, 8: 3, 9: 3}
PB = {1: 1, 3: 2, 5: 3, 6: 3, 7: 3, 8: 3, 9: 3}


def _case(seed):
    g = np.random.default_rng(seed)
    m, n = (int(x) for x in g.integers(1, 701, size=2))
    k = int(g.integers(1, 1201))
    v = int(g.choice([1, 3, 5, 6, 7, 8, 9]))
    cg = int(g.choice([1, 2]))
    flags = 0
    if g.random() < 0.25:
        flags |= bx.SCALED_PIECES
    elif g.random() < 0.25 and v != 1:
        flags |= bx.FP64_COMBINE
    if g.random() < 0.5:
        flags |= bx.NO_STREAM_K
    pads = [int(x) for x in g.integers(0, 9, size=3)]
    alpha = float(g.choice([1.0, -1.0, 0.75, 3.0]))
    beta = float(g.choice([0.0, 0.0, 1.0, -0.5]))
    return m, n, k, v, cg, flags, pads, alpha, beta


def _dev(X, ld):
    rows, cols = X.shape
    big = torch.empty_strided((ld, cols), (1, ld), dtype=torch.float32, device="cuda")
    big[:rows].copy_(torch.from_numpy(np.asfortranarray(X)))
    return big


def _pieces(X, npieces, transpose, scaled):
    """Planes of X (device, column-major with its ld) into one buffer: same layout (ldp = round8(rows))
    or transposed (ldp = round8(cols)).  Returns (buffer, ldp, plane)."""
    rows, cols = X.shape[0], X.shape[1]
    L = bx.lib()
    st = torch.cuda.current_stream().cuda_stream
    ldp = ((cols if transpose else rows) + 7) // 8 * 8
    plane = ldp * (rows if transpose else cols)
    P = torch.zeros(max(1, 3 * plane), dtype=torch.int16, device="cuda")
    p = [P.data_ptr() + 2 * q * plane if q < npieces else None for q in range(3)]
    f = (bx.SPLIT_TRANSPOSED if transpose else 0) | (bx.SCALED_PIECES if scaled else 0)
    L.bf16x_split_ex.argtypes = [bx._i64, bx._i64, bx._vp, bx._i64, bx._vp, bx._vp, bx._vp, bx._i64, bx._u, bx._vp]
    assert L.bf16x_split_ex(rows, cols, X.data_ptr(), X.stride(1), p[0], p[1], p[2], ldp, f, st) == 0
    return P, ldp, plane


@pytest.fixture
def tune():
    yield bx.lib().bf16x_tune
    bx.lib().bf16x_tune(0, 0, 0)


@pytest.mark.parametrize("seed", range(160))
def test_gemm_ex_random(orc, tune, seed):
    m, n, k, v, cg, flags, pads, alpha, beta = _case(seed)
    tune(cg, 0, 0)
    A = synthetic.uniform(m, k, seed=seed)
    B = synthetic.uniform(k, n, seed=seed + 1000)
    C0 = synthetic.uniform(m, n, seed=seed + 2000)
    lda, ldb, ldc = m + pads[0], k + pads[1], m + pads[2]
    Ad, Bd = _dev(A, lda), _dev(B, ldb)
    Ad_v, Bd_v = Ad[:m], Bd[:k]
    outs = []
    scaled = bool(flags & bx.SCALED_PIECES)
    for path in ("internal", "kmajor", "mn"):
        Cd = _dev(C0, ldc)
        if path == "internal":
            bx.gemm_raw(m, n, k, alpha, Ad.data_ptr(), lda, Bd.data_ptr(), ldb, beta, Cd.data_ptr(), ldc, variant=v,
                        flags=flags)
        else:
            Pa, ldap, aplane = _pieces(Ad_v, PA[v], path == "kmajor", scaled)
            Pb, ldbp, bplane = _pieces(Bd_v, PB[v], False, scaled)
            bx.gemm_raw(m, n, k, alpha, 0, lda, 0, ldb, beta, Cd.data_ptr(), ldc, variant=v,
                        flags=flags | (bx.A_PIECES_MN if path == "mn" else 0), A_pieces=Pa.data_ptr(), ldap=ldap,
                        a_plane=aplane, B_pieces=Pb.data_ptr(), ldbp=ldbp, b_plane=bplane)
        torch.cuda.synchronize()
        outs.append(Cd[:m].cpu().numpy())
    case = (m, n, k, v, cg, flags, pads, alpha, beta)
    assert np.array_equal(outs[0].view(np.int32), outs[1].view(np.int32)), ("kmajor", case)
    assert np.array_equal(outs[0].view(np.int32), outs[2].view(np.int32)), ("mn", case)
    O = orc.gemm(A, B, C=C0, alpha=alpha, beta=beta, variant=v, scaled=scaled,
                 fp64_combine=bool(flags & bx.FP64_COMBINE))
    C64 = orc.dgemm(A, B) * alpha + beta * C0.astype(np.float64)
    eg = orc.normwise_error(outs[0], C64, A, B)
    eo = orc.normwise_error(O, C64, A, B)
    assert eg <= RATIO * eo or eg <= 1e-30, (case, eg, eo)
