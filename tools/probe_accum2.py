"""K3b: a finer probe of tcgen05 kind::f16 FP32 accumulation (extends tools/probe_accum.py).

Method as probe_accum.py: variant 1 (one BF16 product per term; every input value is exactly
BF16, so there are no residual pieces), m = 128, n = 256, k = 32 = one promotion interval of
two K=16 MMAs into one TMEM accumulator (the first overwrites it); C[0, 0] is the tensor
core's FP32 result.  k indices 0..15 are the first MMA, 16..31 the second (so "across" cases
test how the running accumulator enters the next MMA step).

The cases separate the candidate models of one MMA step D = sum(16 products) + C:
  per-addend truncation toward zero at the largest addend's 24-bit window (no guard bits),
  guard bits g (the window is 24 + g bits), truncation toward -inf (two's complement floor),
  and exact-sum-then-round (RZ / RN) of the result.
Output: JSON {case: {got, exact, terms}} on stdout and in gpurun_out/probe_accum2.json."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx

u = 2.0 ** -23


def run(terms):
    m, n, k = 128, 256, 32
    A = np.zeros((m, k), dtype=np.float32, order="F")
    B = np.zeros((k, n), dtype=np.float32, order="F")
    for kk, v in terms:
        A[0, kk] += v
        assert np.float32(v) == v
        b = np.array([v], dtype=np.float32).view(np.uint32)[0]
        assert (b & 0xFFFF) == 0, ("not bf16", v)
    B[:, 0] = 1.0
    C = bx.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), variant=1)
    torch.cuda.synchronize()
    return float(C[0, 0].item())


cases = {}
# rounding direction inside one MMA
cases["w_1+0.75u"] = [(0, 1.0), (1, 0.75 * u)]
cases["w_1+0.5u"] = [(0, 1.0), (1, 0.5 * u)]
cases["w_1+0.5u+0.5u"] = [(0, 1.0), (1, 0.5 * u), (2, 0.5 * u)]
cases["w_-1-0.75u"] = [(0, -1.0), (1, -0.75 * u)]
cases["w_1-0.25u"] = [(0, 1.0), (1, -0.25 * u)]
cases["w_2-0.75u"] = [(0, 2.0), (1, -0.75 * u)]
cases["w_-2+0.75u"] = [(0, -2.0), (1, 0.75 * u)]
cases["w_1.5-1-0.25u"] = [(0, 1.5), (1, -1.0), (2, -0.25 * u)]
# guard bits: 2^g copies of 2^-(23+g) sum exactly to u
for g in range(1, 5):
    cases[f"w_guard{g}"] = [(0, 1.0)] + [(1 + i, 2.0 ** -(23 + g)) for i in range(2 ** g)]
# carry out of the top binade: 1 + 1 (exponent grows) with a low bit that only the pre-carry window holds
cases["w_1+1+u"] = [(0, 1.0), (1, 1.0), (2, u)]
cases["w_1+1+0.5u+0.5u"] = [(0, 1.0), (1, 1.0), (2, u), (3, u)]
cases["w_1.5+1.5+u"] = [(0, 1.5), (1, 1.5), (2, u)]
# which addend sets the window: the max product, or the max of the exact sum?
cases["w_cancel_2-1.75+2^-27"] = [(0, 2.0), (1, -1.75), (2, 2.0 ** -27)]
cases["w_cancel_1-1+2^-40"] = [(0, 1.0), (1, -1.0), (2, 2.0 ** -40)]
# the accumulator entering the second MMA
cases["x_acc(1+u)+tiny"] = [(0, 1.0), (1, u), (16, 2.0 ** -24), (17, 2.0 ** -24)]
cases["x_acc0.75u+1"] = [(0, 0.75 * u), (16, 1.0)]
cases["x_acc1+0.75u"] = [(0, 1.0), (16, 0.75 * u)]
cases["x_acc-1-0.75u"] = [(0, -1.0), (16, -0.75 * u)]
cases["x_acc1-0.25u"] = [(0, 1.0), (16, -0.25 * u)]
cases["x_acc(1+u)-1"] = [(0, 1.0), (1, u), (16, -1.0)]
cases["x_acc2^-30+1-1"] = [(0, 2.0 ** -30), (16, 1.0), (17, -1.0)]
for g in range(1, 4):
    cases[f"x_guard{g}"] = [(0, 1.0)] + [(16 + i, 2.0 ** -(23 + g)) for i in range(2 ** g)]
# products (not just A values): B = 1 everywhere, so products = A values; nothing else to vary

out = {}
for name, terms in cases.items():
    exact = float(sum(np.float64(v) for _, v in terms))
    got = run(terms)
    out[name] = {"got": got, "got_hex": np.float32(got).view(np.uint32).item(), "exact": exact,
                 "err_ulps_of_1": (got - exact) / u, "terms": [[kk, v] for kk, v in terms]}
s = json.dumps(out, indent=1)
print(s)
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/probe_accum2.json", "w") as f:
    f.write(s)
