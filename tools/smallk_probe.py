"""Short-k schedule (tile N 128, 4 TMEM buffers) vs the default (tile N 256, 2 buffers):
split + GEMM per call, m = n = 4096 (or argv[1]), k in argv[2]."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
mn = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ks = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["256", "512", "1024", "2048"])]
for k in ks:
    A = torch.rand(mn, k, device="cuda") * 2 - 1
    B = torch.rand(k, mn, device="cuda") * 2 - 1
    C = torch.empty(mn, mn, device="cuda")
    for v in (3, 6, 9):
        res = {}
        for rep in range(2):
            for mode, lim in (("N256", 0), ("N128x4", 1 << 30)):
                L.bf16x_smallk(lim)
                for _ in range(3):
                    bx.gemm(A, B, C, variant=v)
                torch.cuda.synchronize()
                time.sleep(0.2)
                it = 100
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(it):
                    bx.gemm(A, B, C, variant=v)
                e1.record()
                torch.cuda.synchronize()
                res.setdefault(mode, []).append(e0.elapsed_time(e1) / it)
                if rep == 0 and mode == "N256":
                    ref = C.clone()
                if rep == 0 and mode == "N128x4":
                    same = torch.equal(ref.view(torch.int32), C.view(torch.int32))
        print(f"{mn}x{mn}x{k} x{v}: N256 {min(res['N256']) * 1e3:.1f} us  N128x4 {min(res['N128x4']) * 1e3:.1f} us "
              f"({2 * mn * mn * k / min(res['N256']) / 1e9:.0f} -> {2 * mn * mn * k / min(res['N128x4']) / 1e9:.0f} TF)"
              f"  bit-identical={same}", flush=True)
L.bf16x_smallk(512)
