"""MMA issuer: lazy per-stage waits (1) vs all of an interval's stages up front (0), and x3 with
128-k promotion intervals (spi 4): step time (split + GEMM) and bit-identity, uniform [-1, 1]:
tools/lazy_probe.py [n,...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()


def step_us(A, B, C, v, it=None):
    # burst regime: 0.5 s idle, 5 warm-up calls, then ~25 ms of timed calls
    n = A[0].shape[0]
    it = it or max(4, int(25e-3 / (2 * n ** 3 * v / 3 / 1.2e15)))
    torch.cuda.synchronize()
    time.sleep(0.5)
    for i in range(5):
        bx.gemm(A[i % 2], B[i % 2], C, variant=v)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(it):
        bx.gemm(A[i % 2], B[i % 2], C, variant=v)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "8192"])]:
    A = [torch.rand(n, n, device="cuda") * 2 - 1 for _ in range(2)]
    B = [torch.rand(n, n, device="cuda") * 2 - 1 for _ in range(2)]
    C = torch.empty(n, n, device="cuda")
    for v, spis in ((3, (2, 4)), (6, (0,)), (9, (0,))):
        for spi in spis:
            L.bf16x_tune(0, 0, spi)
            res, outs = {}, {}
            for rep in range(3):
                for lazy in (0, 1):
                    L.bf16x_lazy_full(lazy)
                    res.setdefault(lazy, []).append(step_us(A, B, C, v))
                    bx.gemm(A[0], B[0], C, variant=v)
                    torch.cuda.synchronize()
                    outs[lazy] = C.clone()
            same = torch.equal(outs[0].view(torch.int32), outs[1].view(torch.int32))
            t0, t1 = min(res[0]), min(res[1])
            print(f"n={n} x{v} spi={spi}: eager {t0:.1f} us ({2 * n ** 3 / t0 / 1e6:.1f} TF)  lazy {t1:.1f} us "
                  f"({2 * n ** 3 / t1 / 1e6:.1f} TF)  bit-identical={same}", flush=True)
L.bf16x_tune(0, 0, 0)
L.bf16x_lazy_full(1)
