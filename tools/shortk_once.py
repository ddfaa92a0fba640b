"""One LU-shaped trailing update for ncu: C[j:, j:] -= A[j:, j-256:j] @ A[j-256:j, j:] (x3, k = 256,
ld 8192, beta = 1): python tools/shortk_once.py [j] [beta] [iters]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

N, KB = 8192, 256
j = int(sys.argv[1]) if len(sys.argv) > 1 else 256
beta = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
M = (torch.rand(N, N, device="cuda") * 2 - 1).t()
base, mn = M.data_ptr(), N - j
for _ in range(iters):
    bx.gemm_raw(mn, mn, KB, -1.0, base + ((j - KB) * N + j) * 4, N, base + (j * N + (j - KB)) * 4, N, beta,
                base + (j * N + j) * 4, N, variant=3)
torch.cuda.synchronize()
print("ok")
