"""Fused A (A converted inside the GEMM, B pre-split) vs the pre-pass: bit-identity and time per call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()


def run(n, v, mode, iters):
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    L.bf16x_fused_a(1 if mode > 0 else 0)
    L.bf16x_tune(0, 0, int(os.environ.get("FA_SPI", "0")) if mode > 0 else 0)
    for _ in range(3):
        bx.gemm(A, B, C, variant=v)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        bx.gemm(A, B, C, variant=v)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters, C


for n in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096"])]:
    for v in (3, 6, 9):
        torch.manual_seed(0)
        t0, C0 = run(n, v, 0, 30)
        for mode in (1,):
            torch.manual_seed(0)
            time.sleep(0.5)
            t1, C1 = run(n, v, mode, 30)
            same = torch.equal(C0.view(torch.int32), C1.view(torch.int32))
            print(f"n={n} x{v}: pre-pass {t0:.3f} ms {2*n**3/t0/1e9:.1f} TF | fused-A {t1:.3f} ms "
                  f"{2*n**3/t1/1e9:.1f} TF  bit-identical={same}", flush=True)
L.bf16x_fused_a(0)
