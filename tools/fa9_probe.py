import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, paper_1904_06376_b200 as bx
L = bx.lib()
for n in (2048, 4096, 6144, 8192):
    A = torch.rand(n, n, device="cuda") * 2 - 1; B = torch.rand(n, n, device="cuda") * 2 - 1; C = torch.empty(n, n, device="cuda")
    for v in (8, 9):
        res = {}
        for rep in range(3):
            for fa in (0, 1):
                L.bf16x_fused_a(fa)
                for _ in range(3): bx.gemm(A, B, C, variant=v)
                torch.cuda.synchronize(); time.sleep(0.3)
                it = max(3, int(1e12 / (2 * n ** 3)))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(it): bx.gemm(A, B, C, variant=v)
                e1.record(); torch.cuda.synchronize()
                res.setdefault(fa, []).append(e0.elapsed_time(e1) / it)
        t0, t1 = sorted(res[0])[1], sorted(res[1])[1]
        print(f"n={n} x{v}: pre-pass {t0*1e3:.1f} us | fused-A {t1*1e3:.1f} us ({100*(t0/t1-1):+.1f} %)", flush=True)
L.bf16x_fused_a(0)
