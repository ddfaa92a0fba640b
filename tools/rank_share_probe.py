"""Per-rank device time of the column-sharded 16384^3 bf16x6 GEMM (configs[3]) emulated on one
GPU: for P = 2, 4, 8 each rank splits the whole A once (its copy of the broadcast A) and runs
its block-cyclic column blocks (bench.py's sub-block rule, BF16X_NO_STREAM_K, as
distributed.gemm_colsharded does) -- no collectives, which the one-GPU box cannot run.  The
per-rank time T_P is compared with T_1 / P, T_1 = the one-GPU split + GEMM of the whole
problem (bench.py N = 1).  Writes profiles/r08/rank_share_probe.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
import paper_1904_06376_b200 as bx
import synthetic
from paper_1904_06376_b200.distributed import _PieceGemm, block_owner_layout, local_columns

m = n = k = 16384
v = 6
dev = torch.device("cuda", 0)
A = torch.from_numpy(synthetic.uniform(m, k, seed=1)).to(dev)
Bfull = torch.from_numpy(synthetic.uniform(k, n, seed=2)).to(dev)
C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device=dev)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        time.sleep(0.5)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


t1 = timed(lambda: bx.gemm(A, Bfull, C, variant=v))
rows = [{"P": 1, "ms": t1}]
for P in (2, 4, 8):
    S = bench._sub_blocks(n // P, m)
    cols = local_columns(n, P, 0, S)
    Bq = torch.empty_strided((k, len(cols)), (1, k), dtype=torch.float32, device=dev).copy_(Bfull[:, cols])
    Cq = torch.empty_strided((m, len(cols)), (1, m), dtype=torch.float32, device=dev)
    pg = _PieceGemm(A, v)
    widths = [owners[0][1] for owners in block_owner_layout(n, P, S)]

    def rank_step():
        pg.split_chunk(A, 0, k)
        off = 0
        for w in widths:
            pg.gemm(0, k, Bq[:, off:off + w], Cq[:, off:off + w], 0)
            off += w
    tp = timed(rank_step)
    rows.append({"P": P, "sub_blocks": S, "ms": tp, "ideal_ms": t1 / P, "ratio_to_ideal": tp / (t1 / P),
                 "compute_efficiency": (t1 / P) / tp})
    print(rows[-1], flush=True)
out = {"workload": "configs[3] 16384^3 bf16x6, per-rank compute of P-way column sharding emulated on 1 GPU",
       "rows": rows}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "rank_share_probe.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
