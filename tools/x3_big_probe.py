"""16384^3 x3: 64-k intervals (spi 0 = default, 2) vs 128-k intervals (spi 4, multicast schedule), burst timing."""
import sys, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1904_06376_b200 as bx
L = bx.lib()
n = 16384
A = torch.rand(n, n, device="cuda") * 2 - 1
B = torch.rand(n, n, device="cuda") * 2 - 1
C = torch.empty(n, n, device="cuda")
for rep in range(2):
    for spi in (0, 4):
        L.bf16x_tune(0, 0, spi)
        torch.cuda.synchronize(); time.sleep(1.0)
        bx.gemm(A, B, C, variant=3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            bx.gemm(A, B, C, variant=3)
        e1.record(); torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 3
        print(f"16384^3 x3 spi={spi} (0 = default 64-k; 4 = 128-k + multicast): {t:.2f} ms {2 * n ** 3 / t / 1e9:.1f} TF", flush=True)
L.bf16x_tune(0, 0, 0)
