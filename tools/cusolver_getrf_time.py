"""Context for the LU (a6): cuSOLVER's FP32 getrf (torch.linalg.lu_factor, a library) and its FP64
getrf at n = 4096 / 8192 / 16384 beside bf16x_getrf with bf16x3 / bf16x6 trailing updates (device
time between CUDA events, min of 3, after a warm-up)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx
import synthetic


def tm(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


for n in (4096, 8192, 16384):
    A = torch.from_numpy(np.asfortranarray(synthetic.uniform(n, n, seed=n))).cuda()
    A64 = A.double()
    r = {"cusolver_fp32": tm(lambda: torch.linalg.lu_factor(A)),
         "cusolver_fp64": tm(lambda: torch.linalg.lu_factor(A64)),
         "bf16x3": tm(lambda: bx.getrf(A, variant=3)),
         "bf16x6": tm(lambda: bx.getrf(A, variant=6))}
    print(f"n={n}: " + "  ".join(f"{k} {v:.2f} ms" for k, v in r.items()), flush=True)
