"""e2e (bf16x_gemm_host, pinned host buffers) vs host-pipeline depth (column chunks, 2D block
pipeline off) and the 2D block pipeline (default), n^3 x6 (n = argv[1], default 4096)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
v = 6
A = torch.empty_strided((n, n), (1, n), dtype=torch.float32).pin_memory()
B = torch.empty_strided((n, n), (1, n), dtype=torch.float32).pin_memory()
C = torch.empty_strided((n, n), (1, n), dtype=torch.float32).pin_memory()
A.uniform_(-1, 1)
B.uniform_(-1, 1)
L = bx.lib()
def med(f):
    for _ in range(3):
        f()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2]


f = lambda: bx.gemm_host_ptr(n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, v)
t = med(f)
print(f"2d blocks (default): {t * 1e3:.3f} ms  {2 * n ** 3 / t / 1e12:.1f} TFLOPS (median of 10)", flush=True)
L.bf16x_host_2d(0)
for ch in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "4", "8", "12", "16"])]:
    L.bf16x_host_chunks(ch)
    f = lambda: bx.gemm_host_ptr(n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, v)
    for _ in range(3):
        f()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    t = ts[len(ts) // 2]
    print(f"chunks={ch}: {t * 1e3:.3f} ms  {2 * n ** 3 / t / 1e12:.1f} TFLOPS (median of 10)", flush=True)

# timeline of one pipelined call at the default depth
import ctypes
L.bf16x_host_chunks(0)
L.bf16x_host_2d(0)
L.bf16x_host_timeline(1, None, 0)
f = lambda: bx.gemm_host_ptr(n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n, v)
f()
f()
buf = (ctypes.c_float * 64)()
cnt = L.bf16x_host_timeline(0, buf, 64)
print("timeline (ms): start 0, A landed %.3f, A split %.3f" % (buf[1], buf[2]))
for j in range((cnt - 4 + 2) // 3):
    print("  chunk %2d: B landed %.3f  GEMM done %.3f  C back %.3f" % ((j,) + tuple(buf[4 + 3 * j + q] for q in range(3))))
