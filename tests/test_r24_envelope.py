"""Reading R24 (DESIGN.md sections 2 and 7) on the CPU: why configs[0]'s Gaussian-exponent arm is
held to the mean over seeds while the uniform and wide arms are held to 2x the oracle per seed.

* The paper's algorithm itself (each Z^(i,j) an FP32 FMA chain over k, bins added
  smallest first) run with k summed in reverse order -- an equally valid sequential order
  -- stays within 1.2x of the forward-order oracle on every uniform and wide seed, but reaches
  3x-4x on Gaussian seeds: there a single product dominates C and the per-seed bar measures
  summation-order luck.
* The library's schedule for this size (promote every K = 16 MMA, bins smallest first; the GPU
  equals it bit for bit, tests/test_gpu_schedule.py), evaluated on the fitted tcgen05 model
  (tests/tc_model.py), stays within 2x per seed on uniform / wide inputs and within the recorded
  Gaussian envelope (mean <= 2, every seed <= 3).
Test infrastructure only (oracle + model); no GPU."""
import numpy as np
import pytest

import synthetic
import tc_model

SEEDS = {"uniform": range(0, 20), "wide": range(100, 120), "gauss": range(200, 220)}   # test_gpu_configs.py


def _pair(dist, s):
    return synthetic.by_name(dist, 64, 64, seed=s), synthetic.by_name(dist, 64, 64, seed=s + 50_000)


@pytest.mark.parametrize("variant", [6, 9])
def test_summation_order_sensitivity(orc, variant):
    worst = {}
    for dist, seeds in SEEDS.items():
        r = []
        for s in seeds:
            A, B = _pair(dist, s)
            C64 = orc.dgemm(A, B)
            ef = orc.normwise_error(orc.gemm(A, B, variant=variant), C64, A, B)
            Ar, Br = np.ascontiguousarray(A[:, ::-1]), np.ascontiguousarray(B[::-1, :])   # same product, k reversed
            er = orc.normwise_error(orc.gemm(Ar, Br, variant=variant), C64, A, B)
            r.append(er / ef)
        worst[dist] = max(r)
    assert worst["uniform"] <= 1.2 and worst["wide"] <= 1.2, worst
    assert worst["gauss"] >= 3.0, worst


@pytest.mark.parametrize("variant", [6, 9])
def test_kernel_schedule_envelope(orc, variant):
    for dist, seeds in SEEDS.items():
        r = []
        for s in seeds:
            A, B = _pair(dist, s)
            C64 = orc.dgemm(A, B)
            G = tc_model.simulate(A, B, variant, interval=128, promote_every_mma=True)
            eg = orc.normwise_error(G, C64, A, B)
            eo = orc.normwise_error(orc.gemm(A, B, variant=variant), C64, A, B)
            r.append(eg / eo)
        if dist == "gauss":
            assert np.mean(r) <= 2.0 and max(r) <= 3.0, (dist, np.mean(r), max(r))
        else:
            assert max(r) <= 2.0, (dist, max(r))
