"""First-contact GPU check: tiny split + GEMM per variant and cta_group vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synthetic
import paper_1904_06376_b200 as bx

bx.device_check()
print(torch.cuda.get_device_name(), flush=True)
for (m, n, k) in [(128, 256, 32), (256, 256, 64), (300, 520, 100), (1024, 1024, 1024)]:
    A = synthetic.uniform(m, k, seed=1); B = synthetic.uniform(k, n, seed=2)
    C64 = oracle.dgemm(A, B)
    for cg in (1, 2):
        for v in (1, 3, 6, 9):
            t = time.time()
            C = bx.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), variant=v, cta_group=cg)
            torch.cuda.synchronize()
            G = C.cpu().numpy()
            eg = oracle.normwise_error(G, C64, A, B)
            eo = oracle.normwise_error(oracle.gemm(A, B, variant=v), C64, A, B)
            print(f"m{m} n{n} k{k} cg{cg} v{v}: gpu {eg:.3e} oracle {eo:.3e} ratio {eg/eo:.3f}  ({time.time()-t:.2f}s)", flush=True)
