"""GEMM time and bits vs the multicast mode (bf16x_multicast: 1 off, 2 B across 2 pairs, 4 = 2 x 2
pairs sharing A and B).  Usage: python tools/mc_probe.py [n] [variant] [modes] [iters] [reps]
Bit identity is checked with BF16X_NO_STREAM_K (stream-K's split tiles depend on the cluster count);
times are for the default schedule.  PAUSE=s sleeps between modes (power state); GROUP=g sets
the raster group height (bf16x_group_m)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
v = int(sys.argv[2]) if len(sys.argv) > 2 else 6
modes = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["2", "4"])]
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 5
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
m = int(os.environ.get("M", n))
k = int(os.environ.get("K", n))
L = bx.lib()
if os.environ.get("GROUP"):
    L.bf16x_group_m(int(os.environ["GROUP"]))      # tile raster group height (0 = default)
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(k, m, device="cuda", generator=g) * 2 - 1).t()    # column-major m x k
B = (torch.rand(n, k, device="cuda", generator=g) * 2 - 1).t()    # column-major k x n
ref = None
for mode in modes:
    L.bf16x_multicast(mode)
    C = bx.gemm(A, B, variant=v, no_stream_k=True)
    torch.cuda.synchronize()
    if ref is None:
        ref = C.clone()
        print(f"mode {mode}: reference bits", flush=True)
    else:
        same = torch.equal(C, ref)
        print(f"mode {mode}: bit-identical to mode {modes[0]} (no stream-K): {same}", flush=True)
    del C
flops = 2.0 * m * n * k
for _ in range(reps):
    for mode in modes:
        L.bf16x_multicast(mode)
        time.sleep(float(os.environ.get("PAUSE", "0")))
        C = bx.gemm(A, B, variant=v)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            bx.gemm(A, B, C, variant=v)
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        print(f"{m}x{n}x{k} x{v} mode {mode}: {ms:.3f} ms/call (split + GEMM)  {flops / ms / 1e9:.1f} eff TFLOPS",
              flush=True)
L.bf16x_multicast(0)
