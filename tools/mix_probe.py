"""Two concurrent GEMM launches over disjoint column blocks of C: the 2 x 2 multicast schedule
(clusters of 8, 120 SMs) on the first n1 columns and 1-pair launches capped at the remaining SMs
on the rest, vs the single default launch.  K2 alone on pre-split pieces (MN-major A), 16384^3
x6 by default.  Usage: python tools/mix_probe.py [n] [variant] [fractions] [iters] [reps]
env SECOND_MC (multicast mode of the second launch, default 1), CAP (its CTA cap, default 28)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
v = int(sys.argv[2]) if len(sys.argv) > 2 else 6
fracs = [float(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["0.8", "0.84"])]
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 5
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
mc2 = int(os.environ.get("SECOND_MC", "1"))
cap = int(os.environ.get("CAP", "28"))
m = k = n
L = bx.lib()
p = bx.PIECES[v]
kp = (k + 7) // 8 * 8
mp = (m + 7) // 8 * 8
g = torch.Generator(device="cuda").manual_seed(1)
A = (torch.rand(k, m, device="cuda", generator=g) * 2 - 1).t()
B = (torch.rand(n, k, device="cuda", generator=g) * 2 - 1).t()
C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device="cuda")
Ap = torch.empty(p * mp * k, dtype=torch.uint16, device="cuda")
Bp = torch.empty(p * n * kp, dtype=torch.uint16, device="cuda")
s0 = torch.cuda.current_stream()
bx._check(L.bf16x_split_operands_ex(m, n, k, A.data_ptr(), m, B.data_ptr(), k, p, Ap.data_ptr(), mp, mp * k,
                                    Bp.data_ptr(), kp, n * kp, bx.A_PIECES_MN, s0.cuda_stream), "split")
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def gemm_cols(c0, nc, stream):
    bx._check(L.bf16x_gemm_ex(m, nc, k, 1.0, None, m, None, k, 0.0, C.data_ptr() + c0 * m * 4, m, v,
                              bx.A_PIECES_MN, Ap.data_ptr(), mp, mp * k, Bp.data_ptr() + c0 * kp * 2, kp, n * kp,
                              None, None, 0, stream.cuda_stream), "gemm_ex")


def single():
    L.bf16x_multicast(0)
    L.bf16x_max_ctas(0)
    gemm_cols(0, n, s0)


def mixed(f):
    n1 = int(round(n * f / 512)) * 512
    s1.wait_stream(s0)
    s2.wait_stream(s0)
    L.bf16x_multicast(4)
    L.bf16x_max_ctas(0)
    gemm_cols(0, n1, s1)
    L.bf16x_multicast(mc2)
    L.bf16x_max_ctas(cap)
    gemm_cols(n1, n - n1, s2)
    L.bf16x_multicast(0)
    L.bf16x_max_ctas(0)
    s0.wait_stream(s1)
    s0.wait_stream(s2)


def tm(fn):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    for _ in range(iters):
        fn()
    e1.record(s0)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


flops = 2.0 * m * n * k
single()
torch.cuda.synchronize()
ref = C.clone()
for f in fracs:
    C.zero_()
    mixed(f)
    torch.cuda.synchronize()
    print(f"f={f}: C equal to the single launch: {torch.equal(C, ref)} (stream-K tails may differ in rounding)")
for _ in range(reps):
    time.sleep(float(os.environ.get("PAUSE", "0")))
    ms = tm(single)
    print(f"single (default schedule): {ms:.3f} ms  {flops / ms / 1e9:.1f} eff TFLOPS", flush=True)
    for f in fracs:
        time.sleep(float(os.environ.get("PAUSE", "0")))
        ms = tm(lambda: mixed(f))
        print(f"mixed f={f} (mc4 | mc{mc2} cap {cap}): {ms:.3f} ms  {flops / ms / 1e9:.1f} eff TFLOPS", flush=True)
