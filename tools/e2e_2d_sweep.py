"""bf16x_gemm_host 2D block pipeline: e2e time vs the (row blocks R, column blocks Cb) grid and
the column-chunk pipeline, for n^3 (argv[1]) and variants argv[2] (default 3,6,9)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
vs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "3,6,9").split(",")]
A = torch.empty_strided((n, n), (1, n), dtype=torch.float32).pin_memory()
B = torch.empty_strided((n, n), (1, n), dtype=torch.float32).pin_memory()
C = torch.empty_strided((n, n), (1, n), dtype=torch.float32).pin_memory()
A.uniform_(-1, 1)
B.uniform_(-1, 1)
L = bx.lib()


def med(f, reps=7):
    for _ in range(2):
        f()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2]


for v in vs:
    f = lambda: bx.gemm_host_ptr(n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, v)
    L.bf16x_host_2d(0)
    t = med(f)
    print(f"n={n} x{v} chunks(12): {t * 1e3:.3f} ms", flush=True)
    for R, Cb in [(1, 8), (2, 4), (2, 8), (4, 4), (4, 8), (8, 8), (2, 2)]:
        L.bf16x_host_2d((R << 4) | Cb)
        t = med(f)
        print(f"n={n} x{v} 2d R={R} Cb={Cb}: {t * 1e3:.3f} ms", flush=True)
    L.bf16x_host_2d(1)
    t = med(f)
    print(f"n={n} x{v} 2d auto: {t * 1e3:.3f} ms", flush=True)
