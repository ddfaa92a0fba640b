"""Host<->device bandwidth on the box (pinned memory), to bound the e2e (host-buffer) GEMM:
H2D alone, D2H alone, both directions at once on two streams."""
import time

import torch

n = 4096
A = torch.empty(n * n * 2, dtype=torch.float32).pin_memory()   # A and B: 134 MB
C = torch.empty(n * n, dtype=torch.float32).pin_memory()       # C: 67 MB
dA = torch.empty_like(A, device="cuda")
dC = torch.empty_like(C, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, it=10):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / it


h2d = t(lambda: dA.copy_(A, non_blocking=True))
d2h = t(lambda: C.copy_(dC, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        dA.copy_(A, non_blocking=True)
    with torch.cuda.stream(s2):
        C.copy_(dC, non_blocking=True)


bo = t(both)
print(f"H2D 134 MB: {h2d * 1e3:.2f} ms {A.numel() * 4 / h2d / 1e9:.1f} GB/s")
print(f"D2H  67 MB: {d2h * 1e3:.2f} ms {C.numel() * 4 / d2h / 1e9:.1f} GB/s")
print(f"both      : {bo * 1e3:.2f} ms")
print(f"e2e bound at 4096^3: {2 * n ** 3 / bo / 1e12:.1f} TFLOPS (both directions overlapped)")
