import os, sys, time
sys.path.insert(0, "/root/repo")
import torch, paper_1904_06376_b200 as bx
for n in (4096, 8192):
    A = torch.rand(n, n, device="cuda") * 2 - 1; B = torch.rand(n, n, device="cuda") * 2 - 1; C = torch.empty(n, n, device="cuda")
    for v in (3, 6, 9):
        for _ in range(3): bx.gemm(A, B, C, variant=v)
        torch.cuda.synchronize(); ts = []
        for rep in range(3):
            time.sleep(0.3); it = 40 if n == 4096 else 8
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(it): bx.gemm(A, B, C, variant=v)
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1) / it)
        ms = sorted(ts)[1]
        print(f"{os.environ.get('TAG','')} n={n} x{v}: {ms*1e3:.1f} us {2*n**3/ms/1e9:.1f} TF", flush=True)
