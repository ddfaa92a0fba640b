"""LU sub-panel exchange / update modes by factorisation device time (bf16x_gesv_ir report.factor_ms,
min of 3, two rounds) and bit-identity of the factors (bf16x_getrf): mode 2 (keys by st.async +
mbarrier, default), 3 (keys by plain remote stores polled locally), r09.  (Mode 18 = 2 + 16, step t-1's
update of each row deferred past its column t and done while warp 0 exchanges the keys, was measured
from a build that had it -- bit-identical, 3 % slower, and that build's extra registers slowed every
mode by ~5 %; not kept: profiles/r09/lu_deferred_update.txt.)
tools/lu_mode_probe.py [modes, e.g. 2,3] [n, e.g. 4096,8192]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx
import synthetic

L = bx.lib()
modes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2", "3"])]
ns = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["4096", "8192", "16384"])]
for n in ns:
    A = torch.from_numpy(np.asfortranarray(synthetic.diagdom(n, seed=1))).cuda()
    U = torch.from_numpy(np.asfortranarray(synthetic.uniform(n, n, seed=n))).cuda()
    b = torch.from_numpy(synthetic.rhs(n, seed=2)).cuda()
    res, fac = {}, {}
    for mode in modes + modes:
        L.bf16x_lu_subpanel_bulk(mode)
        t = []
        for _ in range(3):
            x, rep, hist = bx.gesv_ir(A, b, variant=3)
            t.append(rep.factor_ms)
        res.setdefault(mode, []).append(round(min(t), 3))
        LU, ipiv, _ = bx.getrf(U, variant=3)
        fac[mode] = (LU, ipiv)
    L.bf16x_lu_subpanel_bulk(2)
    ref = fac[modes[0]]
    same = {m: bool(torch.equal(fac[m][0].view(torch.int32), ref[0].view(torch.int32)) and torch.equal(fac[m][1], ref[1]))
            for m in modes}
    print(f"n={n}: " + "  ".join(f"mode {m} {res[m]} ms" for m in modes) + f"  bit-identical to mode {modes[0]}: {same}",
          flush=True)
