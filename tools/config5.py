"""configs[4]: LU + iterative refinement, n = 8192, bf16x3 trailing-update GEMMs, condition
numbers 1e1..1e12, vs the FP64 truth.  A = U diag(s) V^T (Haar U, V from FP64 QR of Gaussian
matrices, generated on the GPU with a seeded torch generator -- input generation only),
s geometric from 1 to 1/kappa, rounded to FP32 (reading R15); x_true ~ N(0,1) FP64; b = A x_true
in FP64.  Prints one JSON line per kappa."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
variant = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kappas = [float(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1e1", "1e2", "1e4", "1e6", "1e8", "1e10", "1e12"])]
solvers = (sys.argv[4].split(",") if len(sys.argv) > 4 else ["ir", "gmres"])
dev = torch.device("cuda")
g = torch.Generator(device=dev)
for kappa in kappas:
    g.manual_seed(int(np.log10(kappa)) + 500)
    U, R = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g))
    U = U * torch.sign(torch.diagonal(R))[None, :]
    V, R = torch.linalg.qr(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g))
    V = V * torch.sign(torch.diagonal(R))[None, :]
    s = torch.logspace(0, -np.log10(kappa), n, dtype=torch.float64, device=dev)
    A64 = (U * s[None, :]) @ V.T
    A = A64.float().t().contiguous().t()           # FP32, column-major
    del U, V, R, A64
    if os.environ.get("CONFIG5_NO_SVD"):
        kappa_meas = None
    else:
        sv = torch.linalg.svdvals(A.double())
        kappa_meas = float(sv[0] / sv[-1])
    x_true = torch.randn(n, dtype=torch.float64, device=dev, generator=g)
    b = A.double() @ x_true
    for solver in solvers:
        torch.cuda.synchronize()
        t0 = time.time()
        if solver == "gmres":
            x, rep, hist = bx.gesv_gmres_ir(A, b, variant=variant, nb=256, restart=200, max_iter=30)
        else:
            x, rep, hist = bx.gesv_ir(A, b, variant=variant, nb=256, max_iter=30)
        torch.cuda.synchronize()
        wall = time.time() - t0
        fe = float(torch.linalg.norm(x - x_true) / torch.linalg.norm(x_true))
        print(json.dumps({"n": n, "solver": solver, "variant": variant, "kappa_target": kappa,
                          "kappa_measured": kappa_meas, "converged": bool(rep.converged),
                          "iterations": rep.iterations, "inner_iterations": rep.inner_iterations, "info": rep.info,
                          "forward_error": fe, "backward_error": rep.backward_error,
                          "final_residual_inf": rep.final_residual, "tol": rep.tol,
                          "factor_ms": rep.factor_ms, "refine_ms": rep.refine_ms, "wall_s": wall,
                          "history": [float(h) for h in hist]}), flush=True)
