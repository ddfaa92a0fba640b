#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the BF16-split FP32 GEMM (arXiv 1904.06376).

One *step* = one pass of the whole hot path over one batch of synthetic input:
split A (K1, transposed K-major pieces) -> split B (K1) -> multi-product tcgen05 GEMM with
promotion and alpha/beta epilogue (K2), i.e. exactly what one bf16x_gemm call launches.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--variant 6] [--config c2|c4]
  python bench.py --impl reference ...      # the CPU oracle on the same workload (bounded sample)

Workload (BASELINE.json configs[1]): m = n = k = 4096, bf16x6, A, B ~ U[-1,1] (FP64 draws
rounded to FP32, seeded).  Inputs rotate over two independent sets so no step reuses L2
(2 x 134 MB of FP32 inputs + 201 MB of pieces per step > 126 MB L2).  With N > 1 ranks
(torchrun, NCCL) every rank owns a 4096-column block of C (weak scaling): A is broadcast
from rank 0 and C's column blocks are all-gathered into every rank's C.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective SGEMM TFLOPS (bf16x3/x6/x9) and % of scaled BF16 tensor roofline"
CONFIGS = {
    "c2": dict(m=4096, n=4096, k=4096, label="configs[1]: 4096^3 bf16x{v} GEMM on 1 B200, uniform [-1,1] inputs"),
    "c4": dict(m=16384, n=16384, k=16384, label="configs[3]: 16384^3 bf16x{v} GEMM, uniform [-1,1] inputs"),
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), float(p["hbm_gbs"]), "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """NVML sampler of SM clock and clock-event reasons while the timed region runs."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons = [], 0
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def report(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.REASONS.items() if self.reasons & k], "samples": len(self.samples)}


def _ncu_traffic(kernel_tag: str, workload: str, kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full
    summary (profiles/ncu_summary.json), if it was captured on this workload and kernel."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            s = json.load(f)
        ent = s.get(kernel_tag)
        if ent and ent.get("workload") == workload and ent.get("kernel") == kernel:
            return float(ent["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


def cpu_baseline(m, n, k, variant, ncols, seed_a=1, seed_b=2, target_s=15.0):
    """The oracle as it stands on the host cores, on a bounded sample of output columns of the
    same workload (all m rows, full k): effective TFLOPS = 2*m*k*ncols / t.  ncols <= 0 sizes the
    sample to about `target_s` seconds from a 64-column probe."""
    import oracle
    import synthetic
    A = synthetic.uniform(m, k, seed=seed_a)
    B = synthetic.uniform(k, n, seed=seed_b)
    if ncols <= 0:
        probe = np.linspace(0, n - 1, 64).astype(np.int32)
        t0 = time.perf_counter()
        oracle.gemm(A, B, variant=variant, cols=probe)
        ncols = int(min(n, max(64, 64 * target_s / (time.perf_counter() - t0))))
    cols = np.linspace(0, n - 1, ncols).astype(np.int32)
    t0 = time.perf_counter()
    oracle.gemm(A, B, variant=variant, cols=cols)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * m * k * ncols / dt / 1e12, "unit": "TFLOPS", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"{ncols} of {n} output columns (all {m} rows, full k={k}), incl. the oracle's split of A and B; {dt:.1f} s"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = CONFIGS[args.config]
    m, n, k, v = cfg["m"], cfg["n"], cfg["k"], args.variant
    import oracle
    import synthetic
    A = synthetic.uniform(m, k, seed=1)
    B = synthetic.uniform(k, n, seed=2)
    ncols = args.ref_cols
    rng = np.random.default_rng(0)
    def step(i):
        cols = np.sort(rng.choice(n, size=ncols, replace=False)).astype(np.int32)
        oracle.gemm(A, B, variant=v, cols=cols)
    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = time.perf_counter() - t0
    value = 2.0 * m * k * ncols * args.steps / dt / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["label"].format(v=v), "m": m, "n": n, "k": k, "variant": v,
                   "sample_per_step": f"{ncols} random output columns (all rows, full k)"},
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": f"{ncols} of {n} output columns per step, {args.steps} steps"},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1904_06376_b200 as bx
    import synthetic

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bx.device_check()
    cfg = CONFIGS[args.config]
    v = args.variant
    p = bx.PIECES[v]
    m, k = cfg["m"], cfg["k"]
    n_loc = cfg["n"]                    # columns of C per rank (weak scaling)
    n_tot = n_loc * world
    kp = (k + 7) // 8 * 8
    dev = torch.device("cuda", local)

    # two independent input sets (rotated), column-major; A broadcast from rank 0 when N > 1
    sets = []
    for s in range(2):
        A = torch.from_numpy(synthetic.uniform(m, k, seed=1 + 2 * s)).to(dev) if rank == 0 else \
            torch.empty_strided((m, k), (1, m), dtype=torch.float32, device=dev)
        B = torch.from_numpy(synthetic.uniform(k, n_loc, seed=100 + 2 * s + 1000 * rank)).to(dev)
        sets.append((A, B))
    C_loc = torch.empty_strided((m, n_loc), (1, m), dtype=torch.float32, device=dev)
    C_full = torch.empty((n_tot, m), dtype=torch.float32, device=dev) if world > 1 else None  # C^T row-major = C col-major
    Ap = torch.empty(p * m * kp, dtype=torch.uint16, device=dev)
    Bp = torch.empty(p * n_loc * kp, dtype=torch.uint16, device=dev)
    a_pl = [Ap.data_ptr() + 2 * q * m * kp for q in range(3)]
    b_pl = [Bp.data_ptr() + 2 * q * n_loc * kp for q in range(3)]
    st = torch.cuda.current_stream()
    sh = int(st.cuda_stream)
    L = bx.lib()

    def step(i, ev=None):
        A, B = sets[i % 2]
        if world > 1:
            dist.broadcast(A, src=0)
        if ev is not None:
            ev[0].record(st)
        bx._check(L.bf16x_split_operands(m, n_loc, k, A.data_ptr(), m, B.data_ptr(), k, p, Ap.data_ptr(), kp,
                                         m * kp, Bp.data_ptr(), kp, n_loc * kp, sh), "split_operands")
        if ev is not None:
            ev[1].record(st)
        bx._check(L.bf16x_gemm_ex(m, n_loc, k, 1.0, None, m, None, k, 0.0, C_loc.data_ptr(), m, v, 0,
                                  Ap.data_ptr(), kp, m * kp, Bp.data_ptr(), kp, n_loc * kp, None, None, 0, sh),
                  "gemm_ex")
        if ev is not None:
            ev[2].record(st)
        if world > 1:
            dist.all_gather_into_tensor(C_full, C_loc.t())  # column blocks land contiguously in C

    overlap = world > 1 and not args.no_overlap
    if overlap:
        from paper_1904_06376_b200.distributed import gemm_colsharded
        C_cm = C_full.t()                                   # m x n_tot column-major

    def step_dist(i):
        # the library's column-sharded GEMM: A broadcast in 4 k-chunks with the
        # first sub-block computing as they land (accumulator carry), 4 sub-blocks per rank, each
        # sub-round's all-gather on a side stream overlapping the next sub-round's GEMM
        A, B = sets[i % 2]
        gemm_colsharded(A, B, C_cm, variant=v, sub_blocks=4, k_chunks=4)

    run_step = step_dist if overlap else step
    for i in range(args.warmup):
        run_step(i)
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = bx.launch_count()
    with ClockSampler(local) as clk:
        # timed region: K steps back to back, no event between the launches (an event record
        # between the split and the PDL-launched GEMM would cost the programmatic overlap)
        t_start.record(st)
        for i in range(args.steps):
            run_step(i)
        t_end.record(st)
        torch.cuda.synchronize()
    launches = bx.launch_count() - launches0
    # per-kernel durations for the roofline: the same K steps with CUDA events around every
    # launch on the launching stream, after a pause that lets the board's power budget recover
    # (back-to-back, the second ~60 ms of tensor load runs ~10 % slower on these boards)
    time.sleep(1.0)
    if world > 1:
        dist.barrier()
    for i in range(args.steps):
        step(i, evs[i])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    total_ms = t_start.elapsed_time(t_end)
    split_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    gemm_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    if world > 1:
        t = torch.tensor([total_ms, split_ms, gemm_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, split_ms, gemm_ms = (float(x) for x in t.tolist())
    ms_step = total_ms / args.steps
    flops_step = 2.0 * m * n_tot * k
    value = flops_step / (ms_step * 1e-3) / 1e12

    peak_burst, peak_sust, hbm, peak_src = _peaks()
    mma_flops = v * 2.0 * m * n_loc * k           # algorithmic BF16 MMA flops per GEMM launch
    achieved = mma_flops / (gemm_ms * 1e-3) / 1e12
    workload = cfg["label"].format(v=v)
    cg = bx.default_cta_group()
    kname = f"gemm_split_kernel<{cg},{v},256,{2 if cg == 2 else 1}>"
    traffic = _ncu_traffic(f"gemm_split_kernel_v{v}", workload, kname)
    split_bytes = (4 + 2 * p) * (m * k + k * n_loc)

    # e2e: the public host-buffer entry point (H2D of A and B from pinned memory, GEMM, D2H of C)
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    A_h = torch.empty_strided((m, k), (1, m), dtype=torch.float32).pin_memory()
    B_h = torch.empty_strided((k, n_loc), (1, k), dtype=torch.float32).pin_memory()
    C_h = torch.empty_strided((m, n_loc), (1, m), dtype=torch.float32).pin_memory()
    A_h.copy_(sets[0][0].cpu())
    B_h.copy_(sets[0][1].cpu())
    L.bf16x_set_stream(sh)
    bx.gemm_host_ptr(m, n_loc, k, 1.0, A_h.data_ptr(), m, B_h.data_ptr(), k, 0.0, C_h.data_ptr(), m, v)  # warm
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(e2e_steps):
        bx.gemm_host_ptr(m, n_loc, k, 1.0, A_h.data_ptr(), m, B_h.data_ptr(), k, 0.0, C_h.data_ptr(), m, v)
    e1.record(st)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = flops_step / (e2e_ms * 1e-3) / 1e12

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "mma_dtype": "bf16 x bf16 -> f32 (tcgen05 kind::f16)",
        "data": "synthetic",
        "config": {"workload": workload, "m": m, "n": n_tot, "k": k, "n_per_gpu": n_loc, "variant": v,
                   "inputs": "A, B ~ U[-1,1] (FP64 draws rounded to FP32), seeded, column-major",
                   "l2": "inputs rotate over 2 sets (2 x 134 MB FP32 + 201 MB pieces per step > 126 MB L2); no flush",
                   "parallelism": (f"column blocks of C, dp{world}"
                                   + (" (gemm_colsharded: 4 sub-blocks, A in 4 k-chunks, overlapped all-gathers)"
                                      if overlap else " (broadcast, split, GEMM, all-gather in sequence)"))
                   if world > 1 else "single GPU"},
        "pct_of_scaled_roofline": 100.0 * value / world / (peak_burst / v),
        "split_ms": split_ms, "gemm_ms": gemm_ms,
        "split_gbs": split_bytes / (split_ms * 1e-3) / 1e9,
        "roofline": {"bound": "tensor", "kernel": kname, "achieved": achieved,
                     "peak": peak_burst, "unit": "TFLOP/s", "frac": achieved / peak_burst, "traffic": traffic,
                     "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                     "achieved_def": f"{v} products x 2mnk BF16 MMA flops per launch / mean CUDA-event launch time (events around each launch, in a second pass of the same K steps after a 1 s pause)",
                     "frac_of_sustained": achieved / peak_sust},
        "e2e": {"value": e2e_value, "unit": "TFLOPS", "h2d_bytes_per_step": 4 * (m * k + k * n_loc),
                "d2h_bytes_per_step": 4 * m * n_loc, "steps": e2e_steps,
                "api": "bf16x_gemm_host (pinned host buffers; H2D A,B + split + GEMM + D2H C)"},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clk.report(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(m, cfg["n"], k, v, args.cpu_cols)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", type=int, default=6, choices=[1, 3, 6, 9])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-cols", type=int, default=0, help="oracle sample (columns) for cpu_baseline; 0 = about 15 s")
    ap.add_argument("--ref-cols", type=int, default=32, help="oracle sample (columns) per --impl reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-overlap", action="store_true",
                    help="N > 1: broadcast / split / GEMM / all-gather in sequence instead of gemm_colsharded")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
