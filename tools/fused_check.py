"""Fused-split GEMM quick check: parity vs the pre-pass path and the oracle, and timing."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1904_06376_b200 as bx

L = bx.lib()
L.bf16x_fused_split.argtypes = [ctypes.c_int]


def run(A, B, v, fused):
    L.bf16x_fused_split(fused)
    C = bx.gemm(A, B, variant=v)
    torch.cuda.synchronize()
    return C


for (m, n, k) in [(256, 256, 64), (512, 512, 512), (300, 700, 333), (1024, 2048, 1000)]:
    A = (torch.rand(m, k, device="cuda") * 2 - 1).t().contiguous().t()
    B = (torch.rand(k, n, device="cuda") * 2 - 1).t().contiguous().t()
    C64 = A.double() @ B.double()
    for v in (3, 6, 9):
        Cf = run(A, B, v, 1)
        Cp = run(A, B, v, 0)
        den = float(torch.linalg.norm(A.double()) * torch.linalg.norm(B.double()))
        ef = float(torch.linalg.norm(Cf.double() - C64)) / den
        ep = float(torch.linalg.norm(Cp.double() - C64)) / den
        print(f"{m}x{n}x{k} v{v}: fused err {ef:.3e} prepass err {ep:.3e} bit-equal(S=1 ref?) "
              f"{bool(torch.equal(Cf, Cp))}", flush=True)


def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


for n in (4096, 8192):
    A = (torch.rand(n, n, device="cuda") * 2 - 1)
    B = (torch.rand(n, n, device="cuda") * 2 - 1)
    C = torch.empty(n, n, device="cuda")
    for v in (3, 6, 9):
        for fused in (1, 0):
            L.bf16x_fused_split(fused)
            ms = timeit(lambda: bx.gemm(A, B, C, variant=v))
            print(f"n={n} v{v} fused={fused}: {ms:.3f} ms {2 * n**3 / ms / 1e9:.1f} TFLOPS", flush=True)
L.bf16x_fused_split(1)
