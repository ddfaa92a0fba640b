"""GMRES-IR Arnoldi counts at n = 384 (tests/test_gpu_gmres.py::test_conditioned_vs_oracle) with the
short-k promote-every-MMA schedule on (library default) and off (bf16x_pm_max_k(0)), beside the
oracle's; also the factor backward error of each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_1904_06376_b200 as bx
import synthetic

L = bx.lib()
n = 384
for kappa in (1e2, 1e4, 1e6, 1e8):
    for v in (3, 6):
        A, _ = synthetic.conditioned(n, kappa, seed=int(np.log10(kappa)) + 60)
        b = A.astype(np.float64) @ synthetic.rhs(n, seed=8)
        ro = oracle.gmres_ir(A, b, variant=v, nb=64)
        out = []
        for pm in (128, 0):
            L.bf16x_pm_max_k(pm)
            Ad = torch.from_numpy(np.asfortranarray(A)).cuda()
            bd = torch.from_numpy(np.ascontiguousarray(b)).cuda()
            x, rep, hist = bx.gesv_gmres_ir(Ad, bd, variant=v, nb=64, restart=200, inner_tol=1e-10, max_iter=30)
            out.append(f"pm{pm}: conv {rep.converged} outer {rep.iterations} inner {rep.inner_iterations}")
        L.bf16x_pm_max_k(128)
        print(f"kappa {kappa:.0e} x{v}: oracle outer {ro['iterations']} inner {ro['inner_iterations']} | " + " | ".join(out), flush=True)
