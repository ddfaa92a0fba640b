"""K2 alone on pre-split pieces, a few launches (for ncu): python tools/gemm_pieces_once.py m n k variant iters"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

m, n, k, v = (int(x) for x in sys.argv[1:5])
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 3
L = bx.lib()
kp = (k + 7) // 8 * 8
p = bx.PIECES[v]
A = (torch.rand(k, m, device="cuda") * 2 - 1).t()
B = (torch.rand(n, k, device="cuda") * 2 - 1).t()
C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device="cuda")
Ap = torch.empty(p * m * kp, dtype=torch.uint16, device="cuda")
Bp = torch.empty(p * n * kp, dtype=torch.uint16, device="cuda")
bx._check(L.bf16x_split_operands(m, n, k, A.data_ptr(), m, B.data_ptr(), k, p, Ap.data_ptr(), kp, m * kp, Bp.data_ptr(),
                                 kp, n * kp, int(torch.cuda.current_stream().cuda_stream)), "split")
for _ in range(iters):
    bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), m, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                a_plane=m * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp)
torch.cuda.synchronize()
print("ok")
