"""K3c: random single-interval MMA results for fitting the tcgen05 accumulation model.

variant 1 (the product of the b0 pieces only), m = 128, n = 256 and k = 16 (one MMA step
from a zero accumulator) or k = 32 (two steps: the second adds into the first's result):
each of the 32768 outputs is one independent sample of the tensor core's FP32 result.
Writes gpurun_out/probe_accum3.npz with A, B, C per (distribution, k)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx
import synthetic

out = {}
for dist in ("uniform", "wide", "gauss"):
    for k in (16, 32):
        A = synthetic.by_name(dist, 128, k, seed=7 + k)
        B = synthetic.by_name(dist, k, 256, seed=9 + k)
        if dist == "uniform":   # mixed signs of near-equal magnitude: cancellation
            B = np.asfortranarray(np.abs(B))
        C = bx.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), variant=1)
        torch.cuda.synchronize()
        out[f"{dist}/{k}/A"] = A
        out[f"{dist}/{k}/B"] = B
        out[f"{dist}/{k}/C"] = C.cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/probe_accum3.npz", **out)
print("ok", len(out))
