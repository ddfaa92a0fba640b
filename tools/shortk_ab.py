"""K2 alone on pre-split pieces (m = n = 4096, beta = 0) at k = 256 / 512 / 1024 / 4096 for x3 / x6, and
one whole 16384 x 4096 x 4096 bf16x6 call; for A/B runs of library builds (BF16X_LIB=...).
CUDA events over back-to-back launches after a pause; min of 3 repetitions."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1904_06376_b200 as bx

L = bx.lib()
m = n = 4096
tag = (os.environ.get("BF16X_LIB", "default") + " mc" + os.environ.get("MC", "0") + " spi" + os.environ.get("SPI", "0")
       + " bn" + os.environ.get("BN", "0") + " ae" + os.environ.get("AE", "0"))
MC, SPI, BN, AE = (int(os.environ.get(x, "0")) for x in ("MC", "SPI", "BN", "AE"))


def hooks(on):
    L.bf16x_multicast(MC if on else 0)
    L.bf16x_tune(0, BN if on else 0, SPI if on else 0)
    if AE:   # (r09 probe build with the alternating-epilogue kernel; not kept)
        L.bf16x_ae_max_k(AE if on else 0)


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


out = []
for k in (256, 512, 1024, 4096):
    for v in (3, 6):
        kp = (k + 7) // 8 * 8
        p = bx.PIECES[v]
        A = (torch.rand(k, m, device="cuda") * 2 - 1).t()
        B = (torch.rand(n, k, device="cuda") * 2 - 1).t()
        ldc = m + int(os.environ.get("LDC_PAD", "0"))
        C = torch.empty_strided((m, n), (1, ldc), dtype=torch.float32, device="cuda")
        Ap = torch.empty(p * m * kp, dtype=torch.uint16, device="cuda")
        Bp = torch.empty(p * n * kp, dtype=torch.uint16, device="cuda")
        bx._check(L.bf16x_split_operands(m, n, k, A.data_ptr(), m, B.data_ptr(), k, p, Ap.data_ptr(), kp, m * kp,
                                         Bp.data_ptr(), kp, n * kp, int(torch.cuda.current_stream().cuda_stream)), "split")

        def g():
            bx.gemm_raw(m, n, k, 1.0, 0, m, 0, k, 0.0, C.data_ptr(), ldc, variant=v, A_pieces=Ap.data_ptr(), ldap=kp,
                        a_plane=m * kp, B_pieces=Bp.data_ptr(), ldbp=kp, b_plane=n * kp)
        hooks(False)
        g()
        ref = C.clone()
        hooks(True)
        t = min(tm(g, 50 if k < 4096 else 20) for _ in range(3))
        same = torch.equal(C.view(torch.int32), ref.view(torch.int32))
        hooks(False)
        roof = v * 2.0 * m * n * k / 1691.9e12 * 1e6
        out.append(f"k{k} x{v} {t:.1f}us ({100 * roof / t:.0f}%){'' if same else ' DIFFERS'}")
print(tag, " ".join(out), flush=True)
