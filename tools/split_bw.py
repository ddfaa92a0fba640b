"""K1 bandwidth probe: algorithmic GB/s of the split kernels (same layout, transposed, both
operands in one launch) vs a plain device copy, inputs rotated over 4 buffers (> L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx


def timeit(fn, nbuf, iters=40, warm=8):
    for i in range(warm):
        fn(i % nbuf)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(iters):
        fn(i % nbuf)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
NB = 4
X = [torch.rand(n, n, device="cuda") * 2 - 1 for _ in range(NB)]
P = [torch.empty(3 * n * n, dtype=torch.uint16, device="cuda") for _ in range(NB)]
Y = [torch.empty(n, n, device="cuda") for _ in range(NB)]
for name, tr in (("same", False), ("trans", True)):
    def f(i, tr=tr):
        p = P[i].data_ptr()
        bx.split_raw(n, n, X[i].data_ptr(), n, p, p + 2 * n * n, p + 4 * n * n, n, transpose=tr)
    ms = timeit(f, NB)
    print(f"split {name:5s} n={n}: {ms * 1e3:.1f} us  {10 * n * n / ms / 1e6:.0f} GB/s algorithmic", flush=True)
L = bx.lib()


def fab(i):
    a = P[i].data_ptr()
    b = P[(i + 2) % NB].data_ptr()
    L.bf16x_split_operands(n, n, n, X[i].data_ptr(), n, X[(i + 1) % NB].data_ptr(), n, 3, a, n, n * n, b, n, n * n,
                           None)   # (K-major A)


ms = timeit(fab, NB)
print(f"split_ab    n={n}: {ms * 1e3:.1f} us  {20 * n * n / ms / 1e6:.0f} GB/s algorithmic (both operands)", flush=True)


def fmn(i):
    a = P[i].data_ptr()
    b = P[(i + 2) % NB].data_ptr()
    L.bf16x_split_operands_ex(n, n, n, X[i].data_ptr(), n, X[(i + 1) % NB].data_ptr(), n, 3, a, n, n * n, b, n, n * n,
                              bx.A_PIECES_MN, None)


ms = timeit(fmn, NB)
print(f"split_ab_mn n={n}: {ms * 1e3:.1f} us  {20 * n * n / ms / 1e6:.0f} GB/s algorithmic (both, A in its own layout)",
      flush=True)
ms = timeit(lambda i: Y[i].copy_(X[i]), NB)
print(f"copy fp32   n={n}: {ms * 1e3:.1f} us  {8 * n * n / ms / 1e6:.0f} GB/s", flush=True)
Z = [torch.empty(3 * n * n, dtype=torch.uint16, device="cuda") for _ in range(NB)]
ms = timeit(lambda i: Z[i].fill_(7), NB)
print(f"fill 6B/el  n={n}: {ms * 1e3:.1f} us  {6 * n * n / ms / 1e6:.0f} GB/s (write only)", flush=True)
