"""Race detection by repetition (compute-sanitizer is closed on this GPU pool, DESIGN.md section
9): every cross-CTA protocol of the library must give the same bits on every run --
  * stream-K tail tiles (contributor publishes its FP32 partial with an epoch flag, the owner
    spins on it) -- 81 and 288 tiles on 74 clusters, k >= 768 (12+ promotion intervals);
  * TMA multicast of B across the two CTA pairs of a cluster (shared-stage release by both);
  * bf16x9's fused-A converter warps (cluster-scope arrivals on the leader's barrier);
  * the LU's 16-CTA cluster sub-panel (DSMEM st.async exchange per column), its panel update
    (last-block U store) and the cooperative triangular solves (per-block ready flags).
Any lost or reordered handshake shows up as a run that differs from the first."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx
import synthetic

pytestmark = pytest.mark.gpu


def _same(runs):
    first = runs[0].view(torch.int32)
    return all(torch.equal(r.view(torch.int32), first) for r in runs[1:])


@pytest.mark.parametrize("m,n,k,variant", [(2304, 2304, 768, 6), (4096, 4608, 1000, 3), (2304, 2304, 1024, 9)])
def test_stream_k_repeatable(m, n, k, variant):
    A = torch.from_numpy(synthetic.uniform(m, k, seed=1)).cuda()
    B = torch.from_numpy(synthetic.uniform(k, n, seed=2)).cuda()
    runs = [bx.gemm(A, B, variant=variant).clone() for _ in range(25)]
    torch.cuda.synchronize()
    assert _same(runs)


@pytest.mark.parametrize("mc", [2, 4])
def test_multicast_repeatable(mc):
    L = bx.lib()
    A = torch.from_numpy(synthetic.uniform(2048, 768, seed=3)).cuda()
    B = torch.from_numpy(synthetic.uniform(768, 2560, seed=4)).cuda()
    L.bf16x_multicast(mc)
    try:
        runs = [bx.gemm(A, B, variant=6).clone() for _ in range(20)]
        torch.cuda.synchronize()
    finally:
        L.bf16x_multicast(0)
    assert _same(runs)


def test_lu_repeatable():
    n = 1536
    A, _ = synthetic.conditioned(n, 1e3, seed=5)
    Ad = torch.from_numpy(A).cuda()
    fac = [bx.getrf(Ad, variant=3, nb=256) for _ in range(4)]
    torch.cuda.synchronize()
    assert all(torch.equal(f[0].view(torch.int32), fac[0][0].view(torch.int32)) for f in fac[1:])
    assert all(torch.equal(f[1], fac[0][1]) for f in fac[1:])
    b = torch.from_numpy(A.astype(np.float64) @ synthetic.rhs(n, seed=6)).cuda()
    xs = [bx.gesv_ir(Ad, b, variant=3, nb=256)[0].clone() for _ in range(3)]
    torch.cuda.synchronize()
    assert all(torch.equal(x, xs[0]) for x in xs[1:])
