"""Cost of the promote-every-MMA schedule at short k: K2 alone (pre-split pieces), m = n = 4096
(or argv[1]), k = 16 / 64 / 128, x3 / x6 / x9, library default (PM) vs bf16x_pm_max_k(0)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
mn = int(sys.argv[1]) if len(sys.argv) > 1 else 4096


def tm(fn, it=50):
    fn()
    torch.cuda.synchronize()
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


for k in (16, 64, 128):
    for v in (3, 6, 9):
        kp = (k + 7) // 8 * 8
        p = bx.PIECES[v]
        A = (torch.rand(k, mn, device="cuda") * 2 - 1).t()
        B = (torch.rand(mn, k, device="cuda") * 2 - 1).t()
        C = torch.empty_strided((mn, mn), (1, mn), dtype=torch.float32, device="cuda")
        Ap = torch.empty(p * mn * kp, dtype=torch.uint16, device="cuda")
        Bp = torch.empty(p * mn * kp, dtype=torch.uint16, device="cuda")
        bx._check(L.bf16x_split_operands(mn, mn, k, A.data_ptr(), mn, B.data_ptr(), k, p, Ap.data_ptr(), kp, mn * kp,
                                         Bp.data_ptr(), kp, mn * kp, int(torch.cuda.current_stream().cuda_stream)), "split")

        def g():
            bx.gemm_raw(mn, mn, k, 1.0, 0, mn, 0, k, 0.0, C.data_ptr(), mn, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                        a_plane=mn * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=mn * kp)
        res = {}
        for rep in range(2):
            res.setdefault("PM", []).append(tm(g))
            L.bf16x_pm_max_k(0)
            res.setdefault("interval", []).append(tm(g))
            L.bf16x_pm_max_k(128)
        print(f"{mn}x{mn}x{k} x{v}: promote every MMA {min(res['PM']):.1f} us, 32-k intervals {min(res['interval']):.1f} us",
              flush=True)
