"""Factor a seeded matrix with the library in BF16X_LIB (default: the in-tree one) and save LU and
ipiv (tools/lu_bits.py n out.npz), or compare two such files (tools/lu_bits.py --cmp a.npz b.npz):
bit identity of the factorisation across two builds."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if sys.argv[1] == "--cmp":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    same = np.array_equal(a["LU"].view(np.uint32), b["LU"].view(np.uint32)) and np.array_equal(a["ipiv"], b["ipiv"])
    print(f"{sys.argv[2]} vs {sys.argv[3]}: bit-identical factors {same}")
    sys.exit(0 if same else 1)
import torch

import paper_1904_06376_b200 as bx

n = int(sys.argv[1])
g = torch.Generator(device="cuda").manual_seed(7)
A = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).t().contiguous().t()
LU, ipiv, info = bx.getrf(A, variant=3)
torch.cuda.synchronize()
np.savez(sys.argv[2], LU=LU.cpu().numpy(), ipiv=ipiv.cpu().numpy())
print("saved", sys.argv[2], "info", info)
