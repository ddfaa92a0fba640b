"""(r09 probe; needs a build with the bf16x_lu_subpanel_dyn hook, not kept) LU sub-panel cluster size per sub-panel (hook 1) vs w.cl CTAs for every
sub-panel (0): factors and pivots bit-identical, factorisation device time (bf16x_gesv_ir
report.factor_ms, min of 4) at n = 2048 / 4096 / 8192 / 16384, bf16x3."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1904_06376_b200 as bx
import synthetic

L = bx.lib()
for n in (2048, 4096, 8192, 16384):
    A = torch.from_numpy(np.asfortranarray(synthetic.diagdom(n, seed=1) if n > 4096 else synthetic.uniform(n, n, seed=n))).cuda()
    b = torch.from_numpy(synthetic.rhs(n, seed=2)).cuda()
    out = {}
    for dyn in (0, 1):
        L.bf16x_lu_subpanel_dyn(dyn)
        LU, ipiv, info = bx.getrf(A, variant=3)
        torch.cuda.synchronize()
        t = []
        for _ in range(4):
            x, rep, hist = bx.gesv_ir(A, b, variant=3)
            t.append(rep.factor_ms)
        out[dyn] = (LU.clone(), ipiv.clone(), min(t))
    L.bf16x_lu_subpanel_dyn(1)
    same = torch.equal(out[0][0].view(torch.int32), out[1][0].view(torch.int32)) and torch.equal(out[0][1], out[1][1])
    print(f"n={n}: fixed clusters {out[0][2]:.2f} ms, per-sub-panel clusters {out[1][2]:.2f} ms, factors bit-identical {same}",
          flush=True)
