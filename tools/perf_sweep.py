"""Throughput sweep (split + GEMM per call, CUDA events, median of 3 timed batches with pauses
between configurations): every variant at 4096^3, 8192^3, 16384^3, plus the N2 options for x6.
Writes JSON lines to stdout."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

_peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
PEAK = json.load(open(_peaks))["bf16_tflops"] if os.path.exists(_peaks) else 1658.0
sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "8192", "16384"])]
for n in sizes:
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    cases = [(v, {}) for v in (3, 5, 6, 7, 8, 9)] + [(6, {"fp64_combine": True}), (6, {"scaled": True})]
    for v, kw in cases:
        it = max(2, int(2e12 / (2 * n ** 3)))
        for _ in range(2):
            bx.gemm(A, B, C, variant=v, **kw)
        torch.cuda.synchronize()
        ts = []
        for rep in range(3):
            time.sleep(0.5)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(it):
                bx.gemm(A, B, C, variant=v, **kw)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / it)
        ts.sort()
        ms = ts[1]
        tf = 2 * n ** 3 / ms / 1e9
        name = f"x{v}" + ("d" if kw.get("fp64_combine") else "") + (" scaled" if kw.get("scaled") else "")
        print(json.dumps({"n": n, "variant": name, "ms": round(ms, 4), "eff_tflops": round(tf, 1),
                          "pct_of_R_over_Pp": round(100 * tf / (PEAK / v), 1)}), flush=True)
