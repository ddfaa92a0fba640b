"""Per-CTA timeline of one K2 launch (bf16x_gemm_debug bit 1, %globaltimer): kernel start,
prologue done, and per tile the first / last promotion and the C issue, then the final store
completion.  Prints per-CTA phase durations (median / max over CTAs) for a short-k GEMM on
pre-split pieces: python tools/gemm_trace.py m n k variant"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes

import numpy as np
import torch

import paper_1904_06376_b200 as bx

m, n, k, v = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (4096, 4096, 256, 3)
extra_dbg = int(sys.argv[5]) if len(sys.argv) > 5 else 0     # dbg bits 4 (STG path), 8 (plain stores)
L = bx.lib()
L.bf16x_gemm_trace.argtypes = [ctypes.c_void_p]
kp = (k + 7) // 8 * 8
p = bx.PIECES[v]
A = (torch.rand(k, m, device="cuda") * 2 - 1).t()
B = (torch.rand(n, k, device="cuda") * 2 - 1).t()
ldc = m + int(os.environ.get("LDC_PAD", "0"))
C = torch.empty_strided((m, n), (1, ldc), dtype=torch.float32, device="cuda")
Ap = torch.empty(p * m * kp, dtype=torch.uint16, device="cuda")
Bp = torch.empty(p * n * kp, dtype=torch.uint16, device="cuda")
bx._check(L.bf16x_split_operands(m, n, k, A.data_ptr(), m, B.data_ptr(), k, p, Ap.data_ptr(), kp, m * kp, Bp.data_ptr(),
                                 kp, n * kp, int(torch.cuda.current_stream().cuda_stream)), "split")
tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")


def g():
    bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), ldc, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                a_plane=m * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp)


for _ in range(3):
    g()
torch.cuda.synchronize()
L.bf16x_gemm_trace(tr.data_ptr())
L.bf16x_gemm_debug(2 | extra_dbg)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g()
e1.record()
torch.cuda.synchronize()
L.bf16x_gemm_debug(0)
T = tr.view(148, 32).cpu().numpy().astype(np.int64)
used = T[:, 0] > 0
T = T[used]
t0 = T[:, 0].min()
R = (T - t0) / 1e3          # us since the first CTA started
print(f"{m}x{n}x{k} x{v} dbg {extra_dbg}: event time {e0.elapsed_time(e1) * 1e3:.1f} us, CTAs traced {used.sum()}")
print(f"  CTA start spread: {np.ptp(R[:, 0]):.2f} us; prologue (start -> griddepcontrol done): median {np.median(R[:, 1] - R[:, 0]):.2f} us")
for sel in (np.ones(len(T), dtype=bool),):
  for t in range(9):
    a, b, c = R[:, 2 + 3 * t], R[:, 3 + 3 * t], R[:, 4 + 3 * t]
    ok = (T[:, 2 + 3 * t] > 0) & (T[:, 4 + 3 * t] > 0) & sel
    if ok.sum() == 0:
        break
    print(f"  tile {t}: first promotion at {np.median(a[ok]):7.2f} us (max {a[ok].max():7.2f}), last at {np.median(b[ok]):7.2f}, "
          f"C issued at {np.median(c[ok]):7.2f} (max {c[ok].max():7.2f}), CTAs {ok.sum()}")
  for t in range(5):
    pl, ms = R[:, 17 + t], R[:, 22 + t]
    okp = (T[:, 17 + t] > 0) & sel
    okm = (T[:, 22 + t] > 0) & sel
    if okp.sum() == 0:
        break
    print(f"  tile {t}: producer first load at {np.median(pl[okp]):7.2f} us (max {pl[okp].max():7.2f}), "
          f"MMA first interval at {np.median(ms[okm]) if okm.any() else float('nan'):7.2f} us (leader CTAs {okm.sum()})")
lead = T[:, 29] > 0
if lead.any():
    wa, wf, tot = (T[lead, q].astype(np.float64) for q in (27, 28, 29))
    print(f"  MMA issuer (leader CTAs {lead.sum()}): waits acc_empty {np.median(wa / tot) * 100:.1f} % / full stages "
          f"{np.median(wf / tot) * 100:.1f} % of its cycles (median), total {np.median(tot):.0f} cycles")
done = R[:, 31]
print(f"  all stores complete: median {np.median(done[T[:, 31] > 0]):.2f} us, max {done[T[:, 31] > 0].max():.2f} us")
