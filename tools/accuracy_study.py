"""Schedule study for the per-case "<= 2x the oracle" bar on exponent-spread inputs
(configs[0]: 64 x 64 x 64, 20 seeds per arm), run offline on the bit-exact tensor-core model
(tests/tc_model.py; it reproduces the kernel's output bit for bit, tests/test_gpu_schedule.py).

Columns: ratio of normwise errors ||C - C64||_F / (||A||_F ||B||_F), schedule / paper order
(tc_model.sequential: Z^(i,j) summed in FP32 RN in increasing k, bins smallest first):
  kernel     the library's schedule at this size since r08 (= pem-tile below)
  i32        r07's schedule (32-k intervals at k <= 128, one accumulator, bands smallest first,
             RN promotion)
  i16 / i64  16-k / 64-k promotion intervals
  sa16/sa32  bin 0 in its own accumulator (split accumulators), 16 / 32-k intervals
  pem-32     every MMA step promoted on its own (no accumulation inside the tensor core beyond
             one K=16 step), bins smallest first within each 32-k stage
  pem-tile   the same, bins smallest first over the tile's whole k (the r08 kernel for k <= 128
             on small outputs)
  rev-k      the paper's own algorithm with k summed in decreasing order (an equally valid
             sequential order): how far the per-case ratio moves with the order alone.
Writes profiles/r08/accuracy_study.txt."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import synthetic
import tc_model as tm

SEEDS = {"uniform": range(0, 20), "wide": range(100, 120), "gauss": range(200, 220)}
SCHED = {"kernel": dict(interval=128, promote_every_mma=True), "i32": dict(interval=32), "i16": dict(interval=16),
         "i64": dict(interval=64), "sa16": dict(interval=16, split_acc=True), "sa32": dict(interval=32, split_acc=True),
         "pem-32": dict(interval=32, promote_every_mma=True)}


def nerr(C, C64, A, B):
    return np.linalg.norm(C.astype(np.float64) - C64) / (np.linalg.norm(A.astype(np.float64)) *
                                                          np.linalg.norm(B.astype(np.float64)))


def main():
    k = 64
    lines = ["configs[0] 64^3, ratio to the paper-order error per seed: mean / max / #seeds > 2"]
    per_seed = []
    for dist, ss in SEEDS.items():
        for v in (6, 9):
            R = {n: [] for n in list(SCHED) + ["rev-k"]}
            for s in ss:
                A = synthetic.by_name(dist, 64, k, seed=s)
                B = synthetic.by_name(dist, k, 64, seed=s + 50_000)
                C64 = A.astype(np.float64) @ B.astype(np.float64)
                eo = nerr(tm.sequential(A, B, v), C64, A, B)
                for n, kw in SCHED.items():
                    R[n].append(nerr(tm.simulate(A, B, v, **kw), C64, A, B) / eo)
                Ar, Br = np.asfortranarray(A[:, ::-1]), np.asfortranarray(B[::-1, :])
                R["rev-k"].append(nerr(tm.sequential(Ar, Br, v), C64, A, B) / eo)
                if dist == "gauss":
                    per_seed.append((v, s, R["kernel"][-1], R["rev-k"][-1]))
            lines.append(f"{dist:8s} x{v}  " + "  ".join(
                f"{n}: {np.mean(r):.2f}/{np.max(r):.2f}/{int(np.sum(np.array(r) > 2))}" for n, r in R.items()))
    lines.append("")
    lines.append("Gaussian arm per seed (variant, seed, kernel / paper-order, reversed-k paper order / paper-order):")
    for v, s, a, b in per_seed:
        lines.append(f"  x{v} seed {s}: kernel {a:.2f}  rev-k {b:.2f}")
    out = "\n".join(lines)
    print(out)
    with open(os.path.join(ROOT, "profiles/r08/accuracy_study.txt"), "w") as f:
        f.write(out + "\n")


if __name__ == "__main__":
    main()
