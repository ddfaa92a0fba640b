"""Sub-panel record exchange: 9 st.async per peer (0) vs one bulk DSMEM copy per peer (1) vs
keys only by st.async + the winning row read from its CTA (2) vs keys by plain remote stores
polled locally + the row read from its CTA (3).
Factorisation device time (bf16x_getrf between CUDA events) and bit-identity of LU / ipiv:
tools/lu_bulk_probe.py [n,...] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

ns = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "8192"])]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
L = bx.lib()
for n in ns:
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    A = (torch.rand(n, n, device="cuda", generator=g) * 2 - 1).t().contiguous().t()
    out = {}
    for mode in (0, 2, 3, 0, 2, 3):
        L.bf16x_lu_subpanel_bulk(mode)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            LU, ipiv, info = bx.getrf(A, variant=3)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out.setdefault(mode, []).append((min(ts), LU.clone(), ipiv.clone()))
    same = all(torch.equal(out[m][i][1].view(torch.int32), out[0][0][1].view(torch.int32)) and
               torch.equal(out[m][i][2], out[0][0][2]) for m in (0, 2, 3) for i in range(2))
    print(f"n={n}: st.async {min(t for t, _, _ in out[0]):.2f} ms  keys st.async {min(t for t, _, _ in out[2]):.2f} ms  "
          f"keys st+poll {min(t for t, _, _ in out[3]):.2f} ms  (getrf incl. host enqueue, min of {reps})  bit-identical={same}", flush=True)
