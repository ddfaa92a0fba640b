"""K3: tcgen05 (kind::f16, FP32 accumulate) rounding probe through the product GEMM.

variant 1 (one BF16 product per term, inputs exactly BF16 so no residual pieces) with
m = 128, n = 256, k = 32 runs exactly one promotion interval: two K=16 MMAs into one TMEM
accumulator (the first overwrites it), then G = 0 + TMEM (exact) and C = 1*G (exact).  So
C[0, 0] is the tensor core's own FP32 result for the crafted sums below."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1904_06376_b200 as bx

u = 2.0 ** -23          # ulp of 1.0 (just above)


def run(terms):
    """terms: list of (k index, value) placed in A[0, k]; B[:, 0] = 1.  Returns C[0,0]."""
    m, n, k = 128, 256, 32
    A = np.zeros((m, k), dtype=np.float32, order="F")
    B = np.zeros((k, n), dtype=np.float32, order="F")
    for kk, v in terms:
        A[0, kk] = v
        assert np.float32(v) == v
    B[:, 0] = 1.0
    C = bx.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), variant=1)
    torch.cuda.synchronize()
    return float(C[0, 0].item())


def classify(got, exact, rn, rz):
    if got == exact:
        return "exact"
    if got == rn and got != rz:
        return "round-to-nearest"
    if got == rz and got != rn:
        return "toward-zero"
    if got == rn == rz:
        return "rn=rz"
    return "other"


out = {}
cases = {
    "within_mma_+0.75ulp": ([(0, 1.0), (1, 0.75 * u)], 1 + u, 1.0),
    "within_mma_+0.25ulp": ([(0, 1.0), (1, 0.25 * u)], 1.0, 1.0),
    "within_mma_-0.25ulp_below1": ([(0, 1.0), (1, -0.125 * u)], 1.0, 1 - u / 2),
    "across_mma_+0.75ulp": ([(0, 1.0), (16, 0.75 * u)], 1 + u, 1.0),
    "across_mma_-0.125ulp_below1": ([(0, 1.0), (16, -0.125 * u)], 1.0, 1 - u / 2),
    "within_mma_15_terms_2^-27": ([(0, 1.0)] + [(i, 2.0 ** -27) for i in range(1, 16)], 1 + u, 1.0),
    "across_mma_15_terms_2^-27": ([(0, 1.0)] + [(16 + i, 2.0 ** -27) for i in range(15)], 1 + u, 1.0),
    "within_mma_cancel_1-1+2^-40": ([(0, 1.0), (1, -1.0), (2, 2.0 ** -40)], 2.0 ** -40, 2.0 ** -40),
    "within_mma_2^-30_next_to_1": ([(0, 1.0), (1, 2.0 ** -30), (2, -1.0)], 2.0 ** -30, 0.0),
}
for name, (terms, rn, rz) in cases.items():
    exact = float(sum(np.float64(v) for _, v in terms))
    got = run(terms)
    out[name] = {"got": got, "exact": exact, "rn": rn, "rz": rz, "verdict": classify(got, exact, rn, rz)}
print(json.dumps(out, indent=1))
