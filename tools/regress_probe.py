"""Bench-regime A/B of the MMA issuer's lazy stage waits (bf16x_lazy_full 1) vs eager (0), x6
at 4096^3: 100 back-to-back split + GEMM calls over 2 rotating input sets, 1 s pause before
each batch, alternating arms: tools/regress_probe.py [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
n, v = 4096, 6
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
g = torch.Generator(device="cuda").manual_seed(1)
A = [(torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1).float() for _ in range(2)]
B = [(torch.rand(n, n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1).float() for _ in range(2)]
C = torch.empty(n, n, device="cuda")
res = {0: [], 1: []}
for r in range(reps):
    for lazy in (1, 0):
        L.bf16x_lazy_full(lazy)
        for i in range(5):
            bx.gemm(A[i % 2], B[i % 2], C, variant=v)
        torch.cuda.synchronize()
        time.sleep(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(100):
            bx.gemm(A[i % 2], B[i % 2], C, variant=v)
        e1.record()
        torch.cuda.synchronize()
        res[lazy].append(e0.elapsed_time(e1) / 100)
for lazy in (1, 0):
    t = sorted(res[lazy])
    print(f"x6 4096^3 lazy={lazy}: ms/step min {t[0]:.4f} median {t[len(t)//2]:.4f} "
          f"({2 * n ** 3 / t[len(t)//2] / 1e9:.1f} TFLOPS median)", flush=True)
L.bf16x_lazy_full(1)
