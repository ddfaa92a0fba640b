"""Host cost of one bx.gemm call (ctypes + C ABI + launches) against its GPU time, small k."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
for (m, n, k) in [(64, 64, 64), (4096, 4096, 256), (4096, 4096, 1024), (4096, 4096, 4096)]:
    A = torch.rand(m, k, device="cuda")
    B = torch.rand(k, n, device="cuda")
    C = torch.empty(m, n, device="cuda")
    for _ in range(5):
        bx.gemm(A, B, C, variant=3)
    torch.cuda.synchronize()
    it = 200 if k <= 1024 else 50
    t0 = time.perf_counter()
    for _ in range(it):
        bx.gemm(A, B, C, variant=3)
    t_host = (time.perf_counter() - t0) / it
    torch.cuda.synchronize()
    t_all = (time.perf_counter() - t0) / it
    # raw C ABI (no Python-side layout logic): bf16x_gemm_ex on column-major views
    st = torch.cuda.current_stream().cuda_stream
    t0 = time.perf_counter()
    for _ in range(it):
        L.bf16x_gemm_ex(n, m, k, 1.0, B.data_ptr(), n, A.data_ptr(), k, 0.0, C.data_ptr(), n, 3, 0, None, 0, 0,
                        None, 0, 0, None, None, 0, st)
    t_raw = (time.perf_counter() - t0) / it
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        bx.gemm(A, B, C, variant=3)
    e1.record()
    torch.cuda.synchronize()
    print(f"{m}x{n}x{k} x3: host {t_host * 1e6:.1f} us/call (raw ABI {t_raw * 1e6:.1f}), loop incl. drain {t_all * 1e6:.1f} us, "
          f"device {e0.elapsed_time(e1) / it * 1e3:.1f} us/call", flush=True)
