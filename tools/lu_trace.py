"""Per-phase cycles of the sub-panel kernel's column step (clock64 of thread 0 of every CTA, summed
over one getrf): tools/lu_trace.py [n] [mode 0|1|2]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
L = bx.lib()
g = torch.Generator(device="cuda")
g.manual_seed(1)
A = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).t().contiguous().t()
L.bf16x_lu_subpanel_bulk(mode)
bx.getrf(A, variant=3)
torch.cuda.synchronize()
L.bf16x_lu_subpanel_bulk(mode | 4)
L.bf16x_lu_subpanel_trace(None, 1)
bx.getrf(A, variant=3)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (16 * 32))()
L.bf16x_lu_subpanel_trace(buf, 0)
L.bf16x_lu_subpanel_bulk(mode)
cols = n
names = ["apply", "cand+sync1", "exchange(w0)", "winner+sync2", "retire->next", "book(w1,cta0)", "kernel total"]
print(f"n={n} mode={mode}: cycles per column (thread 0 of each CTA; kernel total per launch / 32)")
for r in range(16):
    v = [buf[r * 32 + q] for q in range(8)]
    ww = [buf[r * 32 + 8 + q] / cols for q in range(16)]
    if v[7] == 0:
        continue
    per = [x / cols for x in v[:6]] + [v[6] / v[7] / 32]
    print(f"  cta {r:2d}: " + "  ".join(f"{nm} {x:7.0f}" for nm, x in zip(names, per)) + f"  launches {v[7]}")
    print("          warp work (sync2 -> arrival at sync1): " + " ".join(f"{x:.0f}" for x in ww))
