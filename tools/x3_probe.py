"""x3 at 4096^3 / 8192^3: multicast of B across two CTA pairs, promotion interval, raster group."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
for n in (4096, 8192):
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    for mc, spi, g in ((0, 0, 0), (0, 3, 0), (0, 0, 0), (0, 3, 0)):
        L.bf16x_multicast(mc)
        L.bf16x_tune(0, 0, spi)
        L.bf16x_group_m(g)
        for _ in range(3):
            bx.gemm(A, B, C, variant=3)
        torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            time.sleep(0.3)
            it = 40 if n == 4096 else 8
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(it):
                bx.gemm(A, B, C, variant=3)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / it)
        ms = sorted(ts)[1]
        print(f"n={n} x3 multicast={mc} spi={spi} group={g}: {ms * 1e3:.1f} us {2 * n ** 3 / ms / 1e9:.1f} TF", flush=True)
L.bf16x_multicast(0)
L.bf16x_tune(0, 0, 0)
L.bf16x_group_m(0)
