"""x3 / x1: promotion interval 64 k (2 stages) vs 128 k (4 stages), time per call (split + GEMM)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "8192"])]:
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    for v in (3, 1):
        for rep in range(2):
            for spi in (2, 4):
                L.bf16x_tune(0, 0, spi)
                for _ in range(3):
                    bx.gemm(A, B, C, variant=v)
                torch.cuda.synchronize()
                time.sleep(0.5)
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                it = 40 if n <= 4096 else 10
                s.record()
                for _ in range(it):
                    bx.gemm(A, B, C, variant=v)
                e.record()
                torch.cuda.synchronize()
                ms = s.elapsed_time(e) / it
                print(f"n={n} x{v} spi={spi}: {ms:.3f} ms {2 * n ** 3 / ms / 1e9:.1f} eff TF", flush=True)
L.bf16x_tune(0, 0, 0)
