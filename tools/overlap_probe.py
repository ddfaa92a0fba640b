"""Feasibility of overlapping the next problem's split with the current GEMM: split_ab on a few
SMs' worth of blocks, GEMM on a capped grid, and both concurrently on two streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
n = 4096
v = 6
kp = n
A = [torch.rand(n, n, device="cuda") * 2 - 1 for _ in range(2)]
B = [torch.rand(n, n, device="cuda") * 2 - 1 for _ in range(2)]
C = torch.empty(n, n, device="cuda")
P = [(torch.empty(3 * n * kp, dtype=torch.uint16, device="cuda"), torch.empty(3 * n * kp, dtype=torch.uint16, device="cuda"))
     for _ in range(2)]
s_main = torch.cuda.current_stream()
s_side = torch.cuda.Stream()


def split(i, stream):
    Ap, Bp = P[i]
    L.bf16x_split_operands(n, n, n, A[i].data_ptr(), n, B[i].data_ptr(), n, 3, Ap.data_ptr(), kp, n * kp, Bp.data_ptr(),
                           kp, n * kp, stream.cuda_stream)


def gemm(i, stream):
    Ap, Bp = P[i]
    bx.gemm_raw(n, n, n, 1.0, 0, n, 0, n, 0.0, C.data_ptr(), n, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                a_plane=n * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp, stream=stream)


def t(fn, it=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


for g in (0, 128, 64, 32):
    L.bf16x_split_grid(g)
    ms = t(lambda: split(0, s_main))
    print(f"split_ab grid={g or 1184}: {ms * 1e3:.1f} us  {20 * n * n / ms / 1e6:.0f} GB/s", flush=True)
L.bf16x_split_grid(0)
for c in (0, 140, 136, 132):
    L.bf16x_max_ctas(c)
    ms = t(lambda: gemm(0, s_main))
    print(f"gemm max_ctas={c or 148}: {ms * 1e3:.1f} us", flush=True)
# pipelined: GEMM(i) on main while split(i+1) on side, capped grids
for c, g in ((140, 64), (136, 96), (132, 128), (140, 32)):
    L.bf16x_max_ctas(c)
    L.bf16x_split_grid(g)
    ev = [torch.cuda.Event() for _ in range(4)]

    def pipe(steps=20):
        split(0, s_main)
        for i in range(steps):
            cur, nxt = i % 2, (i + 1) % 2
            e_g = torch.cuda.Event()
            gemm(cur, s_main)
            s_side.wait_stream(s_main) if False else None
            # next split: its buffers were last read by GEMM(i-1), which precedes GEMM(i) on main
            e_prev = torch.cuda.Event()
            e_prev.record(s_main)
            if i + 1 < steps:
                split(nxt, s_side)
                e_s = torch.cuda.Event()
                e_s.record(s_side)
                s_main.wait_event(e_s)
    for _ in range(2):
        pipe(4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_main)
    pipe(20)
    e1.record(s_main)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"pipelined max_ctas={c} split_grid={g}: {ms * 1e3:.1f} us/step  {2 * n ** 3 / ms / 1e9:.1f} eff TFLOPS", flush=True)
L.bf16x_max_ctas(0)
L.bf16x_split_grid(0)
