"""Per-SM throughput of the GEMM with the persistent grid capped at 148 / 132 / 116 / 100 / 74 CTAs
(bf16x_max_ctas hook), 4096^3 x3 / x6: a kernel bound by a shared resource (L2, HBM) speeds up per SM
when fewer SMs run; a per-SM-bound kernel does not."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1904_06376_b200 as bx
L = bx.lib()
n = 4096
A = torch.rand(n, n, device="cuda") * 2 - 1; B = torch.rand(n, n, device="cuda") * 2 - 1; C = torch.empty(n, n, device="cuda")
for v in (3, 6):
    for ctas in (148, 132, 116, 100, 74):
        L.bf16x_max_ctas(ctas)
        for _ in range(3): bx.gemm(A, B, C, variant=v)
        torch.cuda.synchronize(); time.sleep(0.3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): bx.gemm(A, B, C, variant=v)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 20
        print(f"x{v} ctas {ctas}: {ms*1e3:.1f} us, per-SM efficiency vs 148: {(148/ctas) / (ms):.4f}", flush=True)
    L.bf16x_max_ctas(0)
