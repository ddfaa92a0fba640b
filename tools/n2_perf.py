"""CUDA-event timing of the N2 options (scaled pieces R29, FP64 collection R30) against the
default path, split + GEMM per call (iteration tool, not the bench contract)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "8192"])]
for n in sizes:
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    for v in (3, 6, 9):
        for sc, d in ((False, False), (True, False), (False, True), (True, True)):
            ms = timeit(lambda: bx.gemm(A, B, C, variant=v, scaled=sc, fp64_combine=d))
            tf = 2 * n ** 3 / ms / 1e9
            print(f"n={n} x{v}{'d' if d else ''}{' scaled' if sc else ''}: {ms:.3f} ms {tf:.1f} eff TFLOPS "
                  f"({100 * tf / (1658.0 / v):.1f}% of R/{v})", flush=True)
