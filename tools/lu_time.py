"""Factorisation device time (report.factor_ms of bf16x_gesv_ir), min / median of R runs in one
process: tools/lu_time.py [n] [variant] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx
import synthetic

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
v = int(sys.argv[2]) if len(sys.argv) > 2 else 3
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
A = torch.from_numpy(np.asfortranarray(synthetic.diagdom(n, seed=1))).cuda()
b = torch.from_numpy(synthetic.rhs(n, seed=2)).cuda()
f = []
hms = []
import ctypes
bx.lib().bf16x_lu_host_ms.restype = ctypes.c_double
if os.environ.get("BF16X_RED_ADD"):   # trailing-update epilogue: 0 fmaf (load C), -1 red.add (default)
    bx.lib().bf16x_red_add(int(os.environ["BF16X_RED_ADD"]))
for _ in range(reps):
    x, rep, hist = bx.gesv_ir(A, b, variant=v)
    f.append(rep.factor_ms)
    hms.append(bx.lib().bf16x_lu_host_ms())
print(f"host enqueue ms: {[round(t, 2) for t in hms]}", flush=True)
f.sort()
print(f"n={n} x{v} red_add={os.environ.get('BF16X_RED_ADD', '-1')}: factor_ms min {f[0]:.2f} median {f[len(f) // 2]:.2f} (all {[round(t, 2) for t in f]})", flush=True)
