"""N4 parity: bf16x_gesv16_batched (fully 16-bit LU + FP64 refinement) against the
oracle's gesv16_ir on the same seeded systems.  Every operation is the oracle's in the oracle's
order with explicit round-to-nearest, so the solutions, verdicts and iteration counts are
compared bit for bit; the batch covers BF16 / binary16 / FP32, with and without pivoting, the
paper's n = 50 and a ragged n, and a singular system."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu


def _systems(n, kappas, trials, seed0=0):
    As, bs, tols = [], [], []
    for kappa in kappas:
        for s in range(trials):
            A, _ = synthetic.conditioned(n, kappa, seed=seed0 + s)
            As.append(A)
            bs.append(A.astype(np.float64) @ synthetic.rhs(n, seed=seed0 + s + 1000))
            tols.append(kappa * 2.0 ** -53)
    return np.stack(As), np.stack(bs), np.array(tols)


@pytest.mark.parametrize("pivot", [True, False])
@pytest.mark.parametrize("fmt", ["bf16", "fp16", "fp32"])
@pytest.mark.parametrize("n", [50, 37])
def test_gesv16_bit_exact_vs_oracle(orc, n, fmt, pivot):
    A, b, tol = _systems(n, (10.0, 1e3), 6)
    x, conv, its, info = bx.gesv16_batched(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(),
                                           torch.from_numpy(tol).cuda(), fmt=fmt, pivot=pivot, max_iter=60)
    x, conv, its, info = (t.cpu().numpy() for t in (x, conv, its, info))
    for s in range(A.shape[0]):
        r = orc.gesv16_ir(A[s], b[s], fmt=fmt, pivot=pivot, tol=tol[s], max_iter=60)
        assert info[s] == r["info"]
        assert bool(conv[s]) == r["converged"] and its[s] == r["iterations"], (s, conv[s], its[s], r)
        assert np.array_equal(x[s], r["x"]), s


def test_gesv16_singular_and_identity(orc):
    n = 16
    A = np.stack([np.eye(n, dtype=np.float32), synthetic.uniform(n, n, seed=2)])
    A[1][:, 5] = 0.0
    b = np.ones((2, n))
    x, conv, its, info = bx.gesv16_batched(torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda(),
                                           torch.full((2,), 2.0 ** -53, dtype=torch.float64).cuda(), fmt="bf16")
    assert conv.tolist() == [1, 0] and its.tolist()[0] == 0 and info.tolist() == [0, 6]
    assert np.array_equal(x.cpu().numpy()[0], np.ones(n))
