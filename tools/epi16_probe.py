"""16 vs 8 promotion/epilogue warps (bf16x_epi16 hook), split + GEMM per call, and bit-identity."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
for n in (4096, 8192):
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    for v in (3, 5, 6, 9):
        res = {}
        for rep in range(2):
            for mask in (0, 1 << v):
                L.bf16x_epi16(mask)
                for _ in range(3):
                    bx.gemm(A, B, C, variant=v)
                torch.cuda.synchronize()
                time.sleep(0.3)
                it = 40 if n == 4096 else 8
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(it):
                    bx.gemm(A, B, C, variant=v)
                e1.record()
                torch.cuda.synchronize()
                res.setdefault(mask, []).append(e0.elapsed_time(e1) / it)
                if rep == 0:
                    if mask == 0:
                        ref = C.clone()
                    else:
                        same = torch.equal(ref.view(torch.int32), C.view(torch.int32))
        t8, t16 = min(res[0]), min(res[1 << v])
        print(f"n={n} x{v}: 8 warps {t8 * 1e3:.1f} us ({2 * n ** 3 / t8 / 1e9:.1f} TF) | 16 warps {t16 * 1e3:.1f} us "
              f"({2 * n ** 3 / t16 / 1e9:.1f} TF)  bit-identical={same}", flush=True)
L.bf16x_epi16(0)
