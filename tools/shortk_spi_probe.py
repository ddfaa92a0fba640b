"""Short-k K2 alone (pre-split pieces, m = n = 4096) vs the promotion interval (bf16x_tune spi:
0 = library default, 1 / 2 / 4 stages of 32 k) and with the beta = 0 C stores skipped (dbg bit 0),
CUDA events over 20 launches: python tools/shortk_spi_probe.py [k list] [variants]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
m = n = 4096
ks = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["256", "512", "1024"])]
vs = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["3", "6"])]


def tm(fn, it=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


for k in ks:
    for v in vs:
        kp = (k + 7) // 8 * 8
        p = bx.PIECES[v]
        A = (torch.rand(k, m, device="cuda") * 2 - 1).t()
        B = (torch.rand(n, k, device="cuda") * 2 - 1).t()
        C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device="cuda")
        Ap = torch.empty(p * m * kp, dtype=torch.uint16, device="cuda")
        Bp = torch.empty(p * n * kp, dtype=torch.uint16, device="cuda")
        bx._check(L.bf16x_split_operands(m, n, k, A.data_ptr(), m, B.data_ptr(), k, p, Ap.data_ptr(), kp, m * kp,
                                         Bp.data_ptr(), kp, n * kp, int(torch.cuda.current_stream().cuda_stream)), "split")

        def run():
            bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), m, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                        a_plane=m * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp)
        flops = 2.0 * m * n * k * v
        for spi in (0, 1, 2, 4):
            if spi == 4 and v not in (1, 3):
                continue
            L.bf16x_tune(0, 0, spi)
            outs = []
            for dbg in (0, 1):
                L.bf16x_gemm_debug(dbg)
                outs.append(tm(run))
            L.bf16x_gemm_debug(0)
            print(f"k={k} x{v} spi={spi}: {outs[0]:.1f} us ({flops / outs[0] / 1e6:.0f} MMA TF/s, "
                  f"{100 * flops / outs[0] / 1e6 / 1691.9:.0f} % of burst)  without C stores {outs[1]:.1f} us", flush=True)
        L.bf16x_tune(0, 0, 0)
