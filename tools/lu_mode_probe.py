"""LU sub-panel exchange mode 2 (keys by st.async + mbarrier, default) vs 3 (keys by plain remote stores
polled locally): factorisation device time (bf16x_gesv_ir report.factor_ms), r09.  (A mode 4 with
64-bit release stores and acquire polling was measured from a build that had it: slower, not kept;
profiles/r09/lu_exchange_modes.txt.)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1904_06376_b200 as bx, synthetic
L = bx.lib()
for n in (4096, 8192, 16384):
    A = torch.from_numpy(np.asfortranarray(synthetic.diagdom(n, seed=1))).cuda()
    b = torch.from_numpy(synthetic.rhs(n, seed=2)).cuda()
    res = {}
    for mode in (2, 3, 2, 3):
        L.bf16x_lu_subpanel_bulk(mode)
        t = []
        for _ in range(3):
            x, rep, hist = bx.gesv_ir(A, b, variant=3)
            t.append(rep.factor_ms)
        res.setdefault(mode, []).append(min(t))
    L.bf16x_lu_subpanel_bulk(2)
    print(f"n={n}: mode 2 {res[2]} ms, mode 3 {res[3]} ms (factor_ms, min of 3, two rounds)", flush=True)
