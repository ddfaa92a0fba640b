"""One bf16x_getrf of a seeded uniform n x n matrix (profiling driver): tools/lu_once.py [n] [variant] [nb]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nb = int(sys.argv[3]) if len(sys.argv) > 3 else 256
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).t().contiguous().t()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.time()
    LU, ipiv, info = bx.getrf(A, variant=variant, nb=nb)
    torch.cuda.synchronize()
    print(f"getrf n={n} variant={variant} nb={nb} info={info} wall_ms={(time.time() - t0) * 1e3:.2f}", flush=True)
