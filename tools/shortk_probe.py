"""LU trailing-update shape: C[j:, j:] -= A[j:, j-256:j] @ A[j-256:j, j:] (x3, k = 256, all
operands inside one column-major 8192^2 matrix, ld 8192), beta = 1 vs beta = 0, against the
HBM time of reading + writing the C block (torch in-place add on the same strided view):
tools/shortk_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

N, KB = 8192, 256
M = (torch.rand(N, N, device="cuda") * 2 - 1).t()      # column-major view: M[i, j] at i + j*N
ld = N
base = M.data_ptr()


def tm(fn, it=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


for j in (256, 2048, 4096, 6144, 7680):
    mn = N - j
    a = base + ((j - KB) * ld + j) * 4          # A21: rows j.., cols j-256..j
    b = base + (j * ld + (j - KB)) * 4          # U12: rows j-256..j, cols j..
    c = base + (j * ld + j) * 4
    res = {}
    for beta in (1.0, 0.0):
        res[beta] = tm(lambda: bx.gemm_raw(mn, mn, KB, -1.0 if beta else 1.0, a, ld, b, ld, beta, c, ld, variant=3))
    L = bx.lib()
    L.bf16x_red_add(1)
    t_red = tm(lambda: bx.gemm_raw(mn, mn, KB, -1.0, a, ld, b, ld, 1.0, c, ld, variant=3))
    L.bf16x_red_add(-1)
    view = M[j:, j:]
    t_copy = tm(lambda: view.mul_(1.0))
    mnk = 2 * mn * mn * KB
    print(f"j={j} mn={mn}: beta=1 {res[1.0]:.1f} us  beta=1 red.add {t_red:.1f} us  beta=0 {res[0.0]:.1f} us  C rd+wr (torch) {t_copy:.1f} us  "
          f"C bytes/beta1 time {8 * mn * mn / res[1.0] / 1e3:.0f} GB/s  MMA {3 * mnk / res[1.0] / 1e6:.0f} TF/s", flush=True)
