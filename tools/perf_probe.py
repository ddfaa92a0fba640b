"""Quick CUDA-event timing of split and GEMM (not the bench contract; for iteration)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1904_06376_b200 as bx

def timeit(fn, iters=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(iters):
        s.record(); fn(); e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts)//2]

sizes = [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["4096", "8192"])]
variants = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "3", "6", "9"])]
cgs = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "2"])]
spis = [int(x) for x in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["0"])]
tns = [int(x) for x in (sys.argv[5].split(",") if len(sys.argv) > 5 else ["0"])]
L = bx.lib()
for n in sizes:
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    # split only
    outs = [torch.empty(n * n, dtype=torch.uint16, device="cuda") for _ in range(3)]
    ms = timeit(lambda: bx.split_raw(n, n, A.data_ptr(), n, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), n))
    print(f"split same  n={n}: {ms*1e3:.1f} us  {10*n*n/ms/1e6:.0f} GB/s", flush=True)
    ms = timeit(lambda: bx.split_raw(n, n, A.data_ptr(), n, outs[0].data_ptr(), outs[1].data_ptr(), outs[2].data_ptr(), n, transpose=True))
    print(f"split trans n={n}: {ms*1e3:.1f} us  {10*n*n/ms/1e6:.0f} GB/s", flush=True)
    for cg in cgs:
      for bn in spis:
       for tn in tns:
        L.bf16x_tune(cg, tn, bn)
        for v in variants:
            ms = timeit(lambda: bx.gemm(A, B, C, variant=v))
            tf = 2 * n**3 / ms / 1e9
            roof = 1658.0 / v
            print(f"gemm n={n} v{v} cg{cg} spi{bn} tn{tn}: {ms:.3f} ms  {tf:.1f} eff TFLOPS  ({100*tf/roof:.1f}% of R/{v}; mma {tf*v:.0f} TF)", flush=True)
    L.bf16x_tune(0, 0, 0)
    ms = timeit(lambda: torch.matmul(A.bfloat16(), B.bfloat16()))
    print(f"torch bf16 matmul (incl casts) n={n}: {ms:.3f} ms", flush=True)
    Ab, Bb = A.bfloat16(), B.bfloat16()
    ms = timeit(lambda: torch.matmul(Ab, Bb))
    print(f"torch bf16 matmul n={n}: {ms:.3f} ms {2*n**3/ms/1e9:.0f} TFLOPS", flush=True)
    torch.backends.cuda.matmul.allow_tf32 = False
    ms = timeit(lambda: torch.matmul(A, B))
    print(f"torch fp32 sgemm n={n}: {ms:.3f} ms {2*n**3/ms/1e9:.1f} TFLOPS", flush=True)
