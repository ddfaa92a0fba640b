"""GEMM time vs tile-raster group height (bf16x_group_m), 4096^3 x6 by default; run under
`ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum` for the DRAM side."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
groups = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2", "4", "8", "16"])]
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
L = bx.lib()
A = torch.rand(n, n, device="cuda") * 2 - 1
B = torch.rand(n, n, device="cuda") * 2 - 1
C = torch.empty(n, n, device="cuda")
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
for g in [g for _ in range(reps) for g in groups]:
    L.bf16x_group_m(g)
    time.sleep(float(os.environ.get("PAUSE", "0")))
    for _ in range(3):
        bx.gemm(A, B, C, variant=6)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        bx.gemm(A, B, C, variant=6)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    print(f"group_m={g}: {ms:.3f} ms/call (split + GEMM)  {2 * n ** 3 / ms / 1e9:.1f} eff TFLOPS", flush=True)
