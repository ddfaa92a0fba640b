"""Short-k schedule options for the K2 kernel alone (pre-split pieces, m = n = 4096, beta = 0):
default vs 128-k promotion intervals (bf16x_tune spi = 4; x1 / x3 only) vs stream-K off,
k = 256 / 512 / 1024, x3 / x6.  CUDA events over 50 back-to-back launches after a pause."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
m = n = 4096


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


for k in (256, 512, 1024):
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
        res = {}
        for rep in range(2):
            res.setdefault("default", []).append(tm(g))

            if v == 3:
                L.bf16x_tune(0, 0, 4)
                res.setdefault("128k", []).append(tm(g))
                L.bf16x_tune(0, 0, 0)
            L.bf16x_stream_k(0)
            res.setdefault("no-sk", []).append(tm(g))
            L.bf16x_stream_k(1)
        roof = v * 2.0 * m * n * k / 1691.9e12 * 1e6
        print(f"{m}x{n}x{k} x{v}: " + "  ".join(f"{kk} {min(vv):.1f} us ({100 * roof / min(vv):.0f} % of R/{v})"
                                               for kk, vv in res.items()), flush=True)
