"""K1 parity: the CUDA split against the oracle, bit-exact (north star: "Split outputs:
bit-exact against the oracle").  Exhaustive over all 2^32 FP32 bit patterns, plus the
layouts the GEMM uses (column-major with ld > rows, transposed, ragged shapes)."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu

CHUNK = 1 << 27


def test_all_2_32_patterns_bit_exact(orc):
    """Every FP32 pattern (incl. +-0, subnormals, the overflow band, +-Inf, every NaN)."""
    dev = torch.device("cuda")
    first_bad = None
    for c in range((1 << 32) // CHUNK):
        first = c * CHUNK
        pats = torch.arange(first, first + CHUNK, dtype=torch.int64, device=dev).to(torch.int32)
        x = pats.view(torch.float32)
        g = bx.split(x)
        want = orc.split_patterns(first, CHUNK)
        for q in range(3):
            got = g[q].cpu().numpy().view(np.uint16)
            if not np.array_equal(got, want[q]):
                i = int(np.flatnonzero(got != want[q])[0])
                first_bad = (hex(first + i), q, hex(int(got[i])), hex(int(want[q][i])))
                break
        if first_bad:
            break
    assert first_bad is None, f"pattern/piece/gpu/oracle: {first_bad}"


@pytest.mark.parametrize("rows,cols,ld", [(1, 1, 1), (7, 3, 9), (129, 65, 130), (256, 33, 256), (1000, 17, 1003),
                                          (64, 128, 64), (200, 300, 204), (130, 257, 131), (513, 1030, 520)])
def test_layouts_same_and_transposed(orc, rows, cols, ld):
    """Column-major with ld > rows, and the transposed (K-major) output used for A."""
    X = synthetic.wide(ld, cols, seed=rows * 31 + cols)
    Xd = torch.from_numpy(np.asfortranarray(X)).cuda()          # ld x cols column-major buffer
    want = orc.split(np.asfortranarray(X[:rows, :]))
    ldp = rows + 5
    outs = [torch.full((cols * ldp,), 0xABCD, dtype=torch.int32, device="cuda").to(torch.uint16) for _ in range(3)]
    bx.split_raw(rows, cols, Xd.data_ptr(), ld, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), ldp)
    torch.cuda.synchronize()
    for q in range(3):
        got = outs[q].cpu().numpy().view(np.uint16).reshape(cols, ldp).T[:rows]
        assert np.array_equal(got, want[q])
    ldt = cols + 3
    outs = [torch.zeros((rows * ldt,), dtype=torch.uint16, device="cuda") for _ in range(3)]
    bx.split_raw(rows, cols, Xd.data_ptr(), ld, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), ldt,
                 transpose=True)
    torch.cuda.synchronize()
    for q in range(3):
        got = outs[q].cpu().numpy().view(np.uint16).reshape(rows, ldt)[:, :cols]
        assert np.array_equal(got, want[q])


def test_fewer_pieces_and_empty(orc):
    X = synthetic.uniform(300, 4, seed=2)
    Xd = torch.from_numpy(X).cuda()
    b0, b1 = bx.split(Xd, pieces=2)
    w = orc.split(X)
    assert np.array_equal(b0.cpu().numpy().view(np.uint16), w[0])
    assert np.array_equal(b1.cpu().numpy().view(np.uint16), w[1])
    e = torch.zeros((0, 5), dtype=torch.float32, device="cuda")
    assert all(t.numel() == 0 for t in bx.split(e))
