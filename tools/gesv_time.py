"""gesv_ir end to end at n = 8192 (kappa 1e1): events around the call, min of 3 after a warm-up (tools/gesv_time.py)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1904_06376_b200 as bx, synthetic
n = 8192
A, _ = synthetic.conditioned(n, 1e1, seed=5)
b = np.ones(n)
Ad = torch.from_numpy(A).cuda(); bd = torch.from_numpy(b).cuda()
bx.gesv_ir(Ad, bd, variant=3)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); x, rep, hist = bx.gesv_ir(Ad, bd, variant=3); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"gesv_ir n={n} k=1e1: min {min(ts):.2f} ms, iterations {rep.iterations}, factor_ms {rep.factor_ms:.2f}, refine_ms {rep.refine_ms:.2f}")
