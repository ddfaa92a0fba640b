"""Run the split GEMM a few times at one size (for ncu captures): python tools/gemm_once.py n variant iters
(env MC: bf16x_multicast mode)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_06376_b200 as bx
if os.environ.get("MC"):
    bx.lib().bf16x_multicast(int(os.environ["MC"]))   # multicast mode (tools/mc_probe.py)
n = int(sys.argv[1]); v = int(sys.argv[2]); iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A = torch.rand(n, n, device="cuda") * 2 - 1
B = torch.rand(n, n, device="cuda") * 2 - 1
C = torch.empty(n, n, device="cuda")
for _ in range(iters):
    bx.gemm(A, B, C, variant=v)
torch.cuda.synchronize()
print("ok")
