"""K2 alone on pre-split pieces for a k sweep (m = n = 4096, x3 and x6, 3 launches each): run
under `ncu --metrics gpu__time_duration.sum` for per-launch device times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
m = n = 4096
for k in (16, 64, 256, 1024):
    for v in (3, 6):
        kp = (k + 7) // 8 * 8
        p = bx.PIECES[v]
        A = (torch.rand(k, m, device="cuda") * 2 - 1).t()
        B = (torch.rand(n, k, device="cuda") * 2 - 1).t()
        C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device="cuda")
        Ap = torch.empty(p * m * kp, dtype=torch.uint16, device="cuda")
        Bp = torch.empty(p * n * kp, dtype=torch.uint16, device="cuda")
        bx._check(L.bf16x_split_operands(m, n, k, A.data_ptr(), m, B.data_ptr(), k, p, Ap.data_ptr(), kp, m * kp,
                                         Bp.data_ptr(), kp, n * kp, int(torch.cuda.current_stream().cuda_stream)), "split")
        for _ in range(3):
            bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), m, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                        a_plane=m * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp)
        torch.cuda.synchronize()
print("ok")
