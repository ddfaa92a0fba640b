"""A/B of two library builds on the LU: factors bit-identical? factorisation time (min of 4).
python tools/lu_ab.py <libA> <libB> [n]  (each build runs in its own subprocess)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_1904_06376_b200 as bx, synthetic
n = %d
A = torch.from_numpy(np.asfortranarray(synthetic.conditioned(n, 1e3, seed=5)[0])).cuda()
LU, ipiv, info = bx.getrf(A, variant=3, nb=256)
np.save(os.environ["OUT"], LU.cpu().numpy())
b = torch.from_numpy(synthetic.rhs(n, seed=2)).cuda()
ts = []
for _ in range(4):
    x, rep, hist = bx.gesv_ir(A, b, variant=3)
    ts.append(rep.factor_ms)
print(json.dumps({"factor_ms_min": min(ts), "all": ts}))
'''
n = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
res = {}
for tag, lib in (("A", sys.argv[1]), ("B", sys.argv[2])):
    env = dict(os.environ, BF16X_LIB=lib, OUT=f"/tmp/lu_{tag}.npy")
    out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, n)], env=env, capture_output=True, text=True)
    res[tag] = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    print(tag, lib, res[tag], flush=True)
import numpy as np
a, b = np.load("/tmp/lu_A.npy"), np.load("/tmp/lu_B.npy")
print("factors bit-identical:", np.array_equal(a.view(np.uint32), b.view(np.uint32)),
      "differing elements:", int(np.sum(a.view(np.uint32) != b.view(np.uint32))))
