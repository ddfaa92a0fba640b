import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, paper_1904_06376_b200 as bx
L = bx.lib()
for n in (4096, 8192):
    A = torch.rand(n, n, device="cuda") * 2 - 1; B = torch.rand(n, n, device="cuda") * 2 - 1; C = torch.empty(n, n, device="cuda")
    for v in (3, 6, 9):
        for rep in range(2):
            for spi in (0, 4):
                L.bf16x_tune(0, 0, spi)
                for _ in range(3): bx.gemm(A, B, C, variant=v, fp64_combine=True)
                torch.cuda.synchronize(); time.sleep(0.3)
                it = 20 if n == 4096 else 4
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(it): bx.gemm(A, B, C, variant=v, fp64_combine=True)
                e1.record(); torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / it
                print(f"n={n} x{v}d spi={spi}: {ms:.3f} ms {2*n**3/ms/1e9:.1f} TF", flush=True)
L.bf16x_tune(0, 0, 0)
