"""Short-k GEMM breakdown (configs[2] family, LU trailing-update shape): the K2 kernel alone on
pre-split pieces, m = n = 4096, beta = 0, time vs k for x3 / x6 -- the intercept is the fixed
per-launch cost (prologue, epilogue stores, pipeline fill), the slope the MMA rate.  Also: the
same with stream-K off, and the HBM time of writing C alone (torch fill).  CUDA events, 50
back-to-back launches after a pause.  Writes gpurun_out/shortk_breakdown.json."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
mn = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ks = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "16,64,128,256,512,1024,2048".split(","))]
variants = [int(x) for x in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["3", "6"])]
dev = "cuda"


def tm(fn, it=50):
    fn()
    torch.cuda.synchronize()
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e3


rows = []
C = torch.empty_strided((mn, mn), (1, mn), dtype=torch.float32, device=dev)
t_fill = tm(lambda: C.fill_(1.0))
for k in ks:
    kp = (k + 7) // 8 * 8
    A = (torch.rand(k, mn, device=dev) * 2 - 1).t()
    B = (torch.rand(mn, k, device=dev) * 2 - 1).t()
    for v in variants:
        p = bx.PIECES[v]
        Ap = torch.empty(p * mn * kp, dtype=torch.uint16, device=dev)
        Bp = torch.empty(p * mn * kp, dtype=torch.uint16, device=dev)
        bx._check(L.bf16x_split_operands(mn, mn, k, A.data_ptr(), mn, B.data_ptr(), k, p, Ap.data_ptr(), kp, mn * kp,
                                         Bp.data_ptr(), kp, mn * kp, int(torch.cuda.current_stream().cuda_stream)),
                  "split")

        def g():
            bx.gemm_raw(mn, mn, k, 1.0, 0, mn, 0, k, 0.0, C.data_ptr(), mn, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                        a_plane=mn * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=mn * kp)
        t = tm(g)
        L.bf16x_stream_k(0)
        t_nosk = tm(g)
        L.bf16x_stream_k(1)
        t_full = tm(lambda: bx.gemm(A, B, C, variant=v))
        r = {"k": k, "variant": v, "gemm_us": t, "gemm_nosk_us": t_nosk, "split_plus_gemm_us": t_full,
             "tensor_roofline_us": v * 2.0 * mn * mn * k / 1691.9e12 * 1e6, "c_fill_us": t_fill,
             "eff_tflops": 2.0 * mn * mn * k / t / 1e6, "pct_of_R_over_Pp": 100 * (v * 2.0 * mn * mn * k / 1691.9e12 * 1e6) / t}
        rows.append(r)
        print(json.dumps(r), flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"mn": mn, "rows": rows}, open("gpurun_out/shortk_breakdown.json", "w"), indent=1)
