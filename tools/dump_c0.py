"""Dump GPU outputs of configs[0]-style problems (64 x 64 x k, uniform / wide / Gaussian
exponent arms, 20 seeds each) for x3 / x6 / x9 under the library's schedules, so the
accumulation model (tools/tc_model.py) can be checked bit for bit offline.
Writes gpurun_out/dump_c0.npz: key f"{sched}/{dist}/{k}/{seed}/{v}" -> C (64 x 64 FP32)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx
import synthetic

SEEDS = {"uniform": range(0, 20), "wide": range(100, 120), "gauss": range(200, 220)}
L = bx.lib()
scheds = {"default": lambda: None, "split_acc": lambda: L.bf16x_split_acc(1)}
if len(sys.argv) > 1:
    scheds = {k: v for k, v in scheds.items() if k in sys.argv[1:]}
out = {}
for name, setup in scheds.items():
    L.bf16x_split_acc(0)
    L.bf16x_tune(0, 0, 0)
    setup()
    for k in (64, 256):
        for dist, ss in SEEDS.items():
            for s in ss:
                A = synthetic.by_name(dist, 64, k, seed=s)
                B = synthetic.by_name(dist, k, 64, seed=s + 50_000)
                Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
                for v in (3, 6, 9):
                    C = bx.gemm(Ad, Bd, variant=v)
                    torch.cuda.synchronize()
                    out[f"{name}/{dist}/{k}/{s}/{v}"] = C.cpu().numpy()
L.bf16x_split_acc(0)
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed("gpurun_out/dump_c0.npz", **out)
print("dumped", len(out))
