"""Short-k K2 with staggered cluster starts (bf16x_stagger probe hook): the clusters that own one
tile fewer (mode 0) or the upper half of the clusters (mode 1) start their loads `ns` late, so the
per-tile C store bursts of the two halves no longer coincide.  K2 alone on pre-split pieces,
m = n = 4096, beta = 0; CUDA events over 50 back-to-back launches after a pause."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
m = n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
KS = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [256, 512, 1024]


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


for k in KS:
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

        def g():
            bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), m, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                        a_plane=m * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp)
        g()
        ref = C.clone()
        res = {}
        for rep in range(2):
            L.bf16x_stagger(0, 0)
            res.setdefault("base", []).append(tm(g))
            for mode in (0, 1):
                for ns in (1000, 2000, 3000, 4500):
                    L.bf16x_stagger(ns, mode)
                    res.setdefault(f"m{mode}/{ns}", []).append(tm(g))
                    assert torch.equal(C, ref)
            L.bf16x_stagger(0, 0)
        roof = v * 2.0 * m * n * k / 1691.9e12 * 1e6
        print(f"{m}x{n}x{k} x{v}: " + "  ".join(f"{kk} {min(vv):.1f} ({100 * roof / min(vv):.0f}%)"
                                               for kk, vv in res.items()), flush=True)
