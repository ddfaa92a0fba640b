"""N3, the Fig. 5 SGETRF experiment at GPU sizes: element errors of bf16x_getrf
(x3 / x6 / x9 trailing updates) and of cuSOLVER's FP32 LU (torch.linalg.lu_factor, the SGETRF
comparator -- a library, as MKL SGETRF was for the paper) against the FP64 elimination of P A
with each factorisation's own pivots (torch.linalg.lu_factor(pivot=False) in FP64; R26).  Data
uniform in [-1, 1] and [-1e10, 1e10] (the paper's two ranges).  One JSON line per (n, range).
    python tools/fig5_getrf.py [n,...] [seeds]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_06376_b200 as bx

ns = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["1024", "2048", "4096"])]
seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 4
torch.backends.cuda.matmul.allow_tf32 = False
dev = torch.device("cuda")


def perm_from_ipiv(ipiv):            # 0-based LAPACK interchange sequence -> row permutation
    n = ipiv.numel()
    p = torch.arange(n, device=ipiv.device)
    ip = ipiv.tolist()
    pl = p.tolist()
    for j, q in enumerate(ip):
        pl[j], pl[q] = pl[q], pl[j]
    return torch.tensor(pl, device=ipiv.device)


def element_error(A, LU, p):
    D, piv = torch.linalg.lu_factor(A.double()[p], pivot=False)
    den = D.abs()
    mask = den > 0
    return float(((LU.double() - D).abs()[mask] / den[mask]).mean())


for n in ns:
    for scale in (1.0, 1e10):
        errs = {"fp32_cusolver": [], "x3": [], "x6": [], "x9": []}
        g = torch.Generator(device=dev)
        for s in range(seeds):
            g.manual_seed(1000 * n + s)
            A = ((torch.rand(n, n, device=dev, generator=g) * 2 - 1) * scale).float()
            A = A.t().contiguous().t()
            LU32, piv32 = torch.linalg.lu_factor(A)             # 1-based pivots (LAPACK)
            errs["fp32_cusolver"].append(element_error(A, LU32, perm_from_ipiv(piv32.to(torch.int64) - 1)))
            for v in (3, 6, 9):
                LU, ipiv, info = bx.getrf(A, variant=v, nb=256)
                errs[f"x{v}"].append(element_error(A, LU, perm_from_ipiv(ipiv.to(torch.int64))))
        mean = {k: sum(v) / len(v) for k, v in errs.items()}
        print(json.dumps({"n": n, "range": f"[-{scale:g}, {scale:g}]", "seeds": seeds, "mean_element_error": mean,
                          "improvement_fp32_over_x6": mean["fp32_cusolver"] / mean["x6"],
                          "improvement_fp32_over_x9": mean["fp32_cusolver"] / mean["x9"],
                          "improvement_fp32_over_x3": mean["fp32_cusolver"] / mean["x3"]}), flush=True)
