"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck,
one tool per run): K1 splits, K2 in each schedule (2-CTA pairs, 1-CTA, TMA multicast, stream-K
tail, scaled pieces, FP64 "d" combine, bf16x9 fused A, k-chunk carry, red.add epilogue), the LU
(cluster sub-panel, panel update, laswp, TRSM, triangular solves), GMRES-IR and the batched
16-bit LU.  Usage: compute-sanitizer --tool <t> python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx
import synthetic

L = bx.lib()
dev = "cuda"


def t(a):
    return torch.from_numpy(np.asfortranarray(a)).to(dev)


A = t(synthetic.uniform(300, 200, seed=1))
B = t(synthetic.uniform(200, 520, seed=2))
# K1
for q in bx.split(A):
    pass
bx.split(A, scaled=True)
bx.split(A.t().contiguous())
# K2 schedules
bx.gemm(A, B, variant=6)                              # 2-CTA pairs, 64-k intervals
bx.gemm(A, B, variant=3, cta_group=1)                 # 1-CTA
bx.gemm(A, B, variant=9)                              # fused A (bf16x9 default)
bx.gemm(A, B, variant=6, scaled=True)                 # scaled pieces (scale-input-d)
bx.gemm(A, B, variant=6, fp64_combine=True)           # "d" variant
Cb = t(synthetic.uniform(300, 520, seed=3))
bx.gemm(A, B, Cb, alpha=-1.0, beta=1.0, variant=3)    # beta != 0
L.bf16x_red_add(1)
bx.gemm(A, B, Cb, alpha=-1.0, beta=1.0, variant=3)    # red.global.add epilogue
L.bf16x_red_add(-1)
L.bf16x_multicast(2)
bx.gemm(t(synthetic.uniform(600, 200, seed=4)), B, variant=6)   # two pairs per cluster, B multicast
L.bf16x_multicast(0)
A2 = t(synthetic.uniform(2304, 256, seed=5))
B2 = t(synthetic.uniform(256, 2304, seed=6))
bx.gemm(A2, B2, variant=6)                            # 81 tiles on 74 clusters: stream-K tail
# k-chunk carry (ACC_IN / ACC_OUT) through the column-sharded path, world 1
from paper_1904_06376_b200.distributed import gemm_colsharded
C3 = torch.empty_strided((300, 520), (1, 300), dtype=torch.float32, device=dev)
A3 = t(synthetic.uniform(300, 600, seed=7))
B3 = t(synthetic.uniform(600, 520, seed=8))
gemm_colsharded(A3, B3, C3, variant=6, sub_blocks=2, k_chunks=3)
torch.cuda.synchronize()
# LU + IR, GMRES-IR, 16-bit batched
n = 300
Al, _ = synthetic.conditioned(n, 1e3, seed=1)
b = Al.astype(np.float64) @ synthetic.rhs(n, seed=2)
bx.gesv_ir(t(Al), torch.from_numpy(b).to(dev), variant=3, nb=64)
bx.gesv_gmres_ir(t(Al), torch.from_numpy(b).to(dev), variant=3, nb=64, restart=20)
As = torch.from_numpy(np.stack([synthetic.conditioned(20, 1e2, seed=s)[0] for s in range(4)])).to(dev)
bs = torch.from_numpy(np.stack([np.ones(20) for _ in range(4)])).to(dev)
bx.gesv16_batched(As, bs, torch.full((4,), 1e-10, dtype=torch.float64, device=dev), fmt="bf16")
torch.cuda.synchronize()
print("sanitize cases done, launches:", bx.launch_count())
