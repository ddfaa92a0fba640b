import os, sys, time
sys.path.insert(0, '.')
import torch, paper_1904_06376_b200 as bx
for n in (4096, 8192):
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    for v in (9, 6):
        for _ in range(3): bx.gemm(A, B, C, variant=v)
        torch.cuda.synchronize(); time.sleep(0.5)
        it = max(2, int(2e12 / (2 * n ** 3)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(it): bx.gemm(A, B, C, variant=v)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / it
        print(n, v, round(ms, 4), round(2 * n ** 3 / ms / 1e9, 1))
