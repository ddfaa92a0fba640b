"""N4: the paper's refinement table (% converged and mean iterations of LU-IR with
FP32 / BF16 / FP16 factors, n = 50, cond 1e1..1e4, 100 trials) computed with
bf16x_gesv16_batched on the GPU -- all 1200 systems of a pivoting mode in three launches.
Matrices: synthetic.conditioned (Haar U, V; geometric singular values 1..1/kappa) and, with
--mode large, one singular value 1 and the rest 1/kappa (R28); b = A x_true; tol = kappa*2^-53.
    python tools/n4_table.py [--no-pivot] [--mode geometric|large] [--trials 100] [--max-iter 100]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1904_06376_b200 as bx
import synthetic

ap = argparse.ArgumentParser()
ap.add_argument("--no-pivot", action="store_true")
ap.add_argument("--mode", default="geometric")
ap.add_argument("--trials", type=int, default=100)
ap.add_argument("--max-iter", type=int, default=100)
ap.add_argument("--n", type=int, default=50)
args = ap.parse_args()
PAPER = {("fp32", 10): (100, 3.47), ("bf16", 10): (45, 39.3556), ("fp16", 10): (90, 16.2667),
         ("fp32", 100): (100, 2.67), ("bf16", 100): (32, 41.125), ("fp16", 100): (91, 16.989),
         ("fp32", 1000): (100, 2.49), ("bf16", 1000): (29, 47.0345), ("fp16", 1000): (89, 19.4831),
         ("fp32", 10000): (100, 2.39), ("bf16", 10000): (21, 48.4286), ("fp16", 10000): (91, 13.5604)}


def conditioned_large(n, kappa, seed):
    A, _ = synthetic.conditioned(n, 1.0, seed=seed)          # Haar-random orthogonal (kappa = 1)
    g = np.random.Generator(np.random.PCG64([seed, 9]))
    U, _ = np.linalg.qr(g.standard_normal((n, n)))
    s = np.full(n, 1.0 / kappa)
    s[0] = 1.0
    return np.asfortranarray(((U * s) @ A.astype(np.float64)).astype(np.float32))


rows = []
for kappa in (10, 100, 1000, 10000):
    As, bs = [], []
    for t in range(args.trials):
        if args.mode == "large":
            A = conditioned_large(args.n, float(kappa), t)
        else:
            A, _ = synthetic.conditioned(args.n, float(kappa), seed=t)
        As.append(A)
        bs.append(A.astype(np.float64) @ synthetic.rhs(args.n, seed=t + 1000))
    Ad = torch.from_numpy(np.stack(As)).cuda()
    bd = torch.from_numpy(np.stack(bs)).cuda()
    tol = torch.full((args.trials,), kappa * 2.0 ** -53, dtype=torch.float64, device="cuda")
    for fmt in ("fp32", "bf16", "fp16"):
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        start.record()
        x, conv, its, info = bx.gesv16_batched(Ad, bd, tol, fmt=fmt, pivot=not args.no_pivot, max_iter=args.max_iter)
        end.record()
        torch.cuda.synchronize()
        c = conv.cpu().numpy().astype(bool)
        it = its.cpu().numpy()
        pc, pi = PAPER[(fmt, kappa)]
        rows.append({"precision": fmt, "cond": kappa, "pct_converged": 100.0 * c.mean(),
                     "mean_iterations": float(it[c].mean()) if c.any() else None,
                     "paper_pct": pc, "paper_iterations": pi, "gpu_ms": start.elapsed_time(end),
                     "pivot": not args.no_pivot, "mode": args.mode, "n": args.n, "trials": args.trials})
        print(json.dumps(rows[-1]), flush=True)
