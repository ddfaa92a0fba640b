"""N3 parity: the Fig. 5 element-error measure on the GPU's bf16x_getrf against the
oracle's LU with the same split-GEMM updates on the same seeded matrices: the GPU factors' mean
elementwise error (vs FP64 elimination with the same pivots, R26) is within 2x of the oracle's,
and the averaged bf16x6-over-FP32 improvement holds for the GPU factors too."""
import numpy as np
import pytest
import torch

import paper_1904_06376_b200 as bx

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale", [1.0, 1e10])
@pytest.mark.parametrize("n", [300, 700])
def test_fig5_gpu_vs_oracle(orc, n, scale):
    eg, eo, e32 = [], [], []
    for s in range(6):
        g = np.random.Generator(np.random.PCG64([n, s, 55]))
        A = (g.uniform(-1.0, 1.0, (n, n)) * scale).astype(np.float32)
        LU, ipiv, info = bx.getrf(torch.from_numpy(np.asfortranarray(A)).cuda(), variant=6, nb=64)
        assert info == 0
        eg.append(orc.lu_element_error(A, LU.cpu().numpy(), ipiv.cpu().numpy()))
        LUo, ipo, _ = orc.getrf(A, variant=6, nb=64)
        eo.append(orc.lu_element_error(A, LUo, ipo))
        LU32, ip32, _ = orc.getrf(A, variant=0, nb=64)
        e32.append(orc.lu_element_error(A, LU32, ip32))
    eg, eo, e32 = map(np.array, (eg, eo, e32))
    assert 0.5 <= eg.mean() / eo.mean() <= 2.0, (eg, eo)
    assert (e32 / eg).mean() > 1.0, (e32, eg)
