#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the BF16-split FP32 GEMM (arXiv 1904.06376).

One *step* = one pass of the whole hot path over one batch of synthetic input:
split A (K1, transposed K-major pieces) -> split B (K1) -> multi-product tcgen05 GEMM with
promotion and alpha/beta epilogue (K2), i.e. exactly what one bf16x_gemm call launches.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--variant 6] [--config c4|c2]
  python bench.py --impl reference ...      # the CPU oracle on the same workload (bounded sample)

Headline workload (north star, BASELINE.json configs[3] at P = 1..8): m = n = k = 16384,
bf16x6, A, B ~ U[-1,1] (FP64 draws rounded to FP32, seeded).  The inputs (1 GiB each, FP32) and
the pieces (3 GiB) are far larger than the 126 MB L2, so no flush is needed.
  N = 1: one GPU runs the whole problem (split + one GEMM per step).
  N > 1: strong scaling of the same problem (torchrun, NCCL): rank q owns n/N block-cyclic
         columns of C (paper_1904_06376_b200.distributed.gemm_colsharded): A broadcast from
         rank 0 in 4 k-chunks, split once per rank, the first sub-block computing as the chunks
         land, C's column blocks all-gathered into every rank's C on a side stream.
Secondary keys (N = 1): configs[1], 4096^3 bf16x6, measured the same way (inputs rotated over two
sets so no step reuses L2).
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
    "c4": dict(m=16384, n=16384, k=16384,
               label="configs[3]: 16384^3 bf16x{v} GEMM column-sharded over {p} B200 (P = {p}), uniform [-1,1] inputs"),
    "c4b": dict(m=32768, n=32768, k=32768,
                label="configs[3]: 32768^3 bf16x{v} GEMM column-sharded over {p} B200 (P = {p}), uniform [-1,1] inputs"),
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


def _ncu(kernel_tag: str, workload: str):
    """Entry of the committed ncu --set full summary (profiles/ncu_summary.json) for this kernel
    on this workload, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            ent = json.load(f).get(kernel_tag)
        if ent and ent.get("workload") == workload:
            return ent
    except Exception:
        pass
    return None


def _sub_blocks(n_loc: int, m: int, units: int = 74, tile: int = 256) -> int:
    """Sub-blocks per rank for gemm_colsharded: the most (<= 4) whose GEMMs each fill >= 2 waves of
    the persistent grid with >= 90 % of the last wave's clusters busy (wave quantisation)."""
    for s in (4, 2, 1):
        w = n_loc // s
        tiles = -(-m // tile) * -(-w // tile)
        waves = -(-tiles // units)
        if waves >= 2 and tiles / (waves * units) >= 0.9:
            return s
    return 1


def cpu_baseline(m, n, k, variant, ncols, seed_a=1, seed_b=2, target_s=15.0, A=None, B=None):
    """The oracle as it stands on the host cores, on a bounded sample of output columns of the
    same workload (all m rows, full k): effective TFLOPS = 2*m*k*ncols / t.  ncols <= 0 sizes the
    sample to about `target_s` seconds from a 16-column probe."""
    import oracle
    import synthetic
    A = synthetic.uniform(m, k, seed=seed_a) if A is None else A
    B = synthetic.uniform(k, n, seed=seed_b) if B is None else B
    if ncols <= 0:
        probe = np.linspace(0, n - 1, 16).astype(np.int32)
        t0 = time.perf_counter()
        oracle.gemm(A, B, variant=variant, cols=probe)
        ncols = int(min(n, max(16, 16 * target_s / (time.perf_counter() - t0))))
    cols = np.linspace(0, n - 1, ncols).astype(np.int32)
    t0 = time.perf_counter()
    oracle.gemm(A, B, variant=variant, cols=cols)
    dt = time.perf_counter() - t0
    return {"value": 2.0 * m * k * ncols / dt / 1e12, "unit": "TFLOPS", "cores": oracle.num_threads(),
            "kind": "oracle",
            "sample": f"{ncols} of {n} output columns (all {m} rows, full k={k}), incl. the oracle's split of A "
                      f"and of the sampled columns of B; {dt:.1f} s; a rate, so no extrapolation"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
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
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong" if args.config in ("c4", "c4b") else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["label"].format(v=v, p=world), "m": m, "n": n, "k": k, "variant": v,
                   "sample_per_step": f"{ncols} random output columns (all rows, full k; the oracle splits A "
                                      f"and those columns of B every step)"},
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": f"{ncols} of {n} output columns per step, {args.steps} steps"},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _split_gemm_step(L, bx, m, n, k, v, p, A, B, C, Ap, Bp, sh, ev=None, st=None, flags=0):
    """One hot-path pass: both operands split in one launch (K1), then the GEMM on the pieces."""
    kp = (k + 7) // 8 * 8
    if ev is not None:
        ev[0].record(st)
    mp = (m + 7) // 8 * 8    # A's pieces in A's own layout (MN-major), as bf16x_gemm splits it
    bx._check(L.bf16x_split_operands_ex(m, n, k, A.data_ptr(), A.stride(1), B.data_ptr(), B.stride(1), p,
                                        Ap.data_ptr(), mp, mp * k, Bp.data_ptr(), kp, n * kp, bx.A_PIECES_MN, sh),
              "split_operands_ex")
    if ev is not None:
        ev[1].record(st)
    bx._check(L.bf16x_gemm_ex(m, n, k, 1.0, None, m, None, k, 0.0, C.data_ptr(), C.stride(1), v,
                              flags | bx.A_PIECES_MN, Ap.data_ptr(), mp, mp * k, Bp.data_ptr(), kp, n * kp, None,
                              None, 0, sh), "gemm_ex")
    if ev is not None:
        ev[2].record(st)


def _timed(run_step, steps, st, local, world, dist):
    """K steps back to back between two events on the launching stream, clocks sampled."""
    import torch
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0.record(st)
        for i in range(steps):
            run_step(i)
        t1.record(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return t0.elapsed_time(t1), clk.report()


def _evented(L, bx, m, n, k, v, p, sets, C, Ap, Bp, sh, st, steps):
    """Per-kernel durations for the roofline: the same steps with CUDA events around each launch."""
    import torch
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        A, B = sets[i % len(sets)]
        _split_gemm_step(L, bx, m, n, k, v, p, A, B, C, Ap, Bp, sh, evs[i], st)
    torch.cuda.synchronize()
    split_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / steps
    gemm_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / steps
    return split_ms, gemm_ms


def secondary_4096(L, bx, v, p, dev, st, sh, steps, local):
    """configs[1] (4096^3) on one GPU, measured as the headline is: inputs rotated over 2 sets."""
    import torch
    import synthetic
    m = n = k = 4096
    kp = k
    sets = [(torch.from_numpy(synthetic.uniform(m, k, seed=1 + 2 * s)).to(dev),
             torch.from_numpy(synthetic.uniform(k, n, seed=100 + 2 * s)).to(dev)) for s in range(2)]
    C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device=dev)
    Ap = torch.empty(p * m * kp, dtype=torch.uint16, device=dev)
    Bp = torch.empty(p * n * kp, dtype=torch.uint16, device=dev)

    def step(i):
        A, B = sets[i % 2]
        _split_gemm_step(L, bx, m, n, k, v, p, A, B, C, Ap, Bp, sh)
    for i in range(5):
        step(i)
    total_ms, clk = _timed(step, steps, st, local, 1, None)
    time.sleep(0.5)
    split_ms, gemm_ms = _evented(L, bx, m, n, k, v, p, sets, C, Ap, Bp, sh, st, steps)
    ms = total_ms / steps
    peak_burst, _, _, _ = _peaks()
    return {"workload": CONFIGS["c2"]["label"].format(v=v), "value": 2.0 * m * n * k / (ms * 1e-3) / 1e12,
            "unit": "TFLOPS", "ms_per_step": ms, "split_ms": split_ms, "gemm_ms": gemm_ms,
            "split_gbs": (4 + 2 * p) * (m * k + k * n) / (split_ms * 1e-3) / 1e9,
            "gemm_frac_of_burst_peak": v * 2.0 * m * n * k / (gemm_ms * 1e-3) / 1e12 / peak_burst,
            "pct_of_scaled_roofline_burst": 100.0 * 2.0 * m * n * k / (ms * 1e-3) / 1e12 / (peak_burst / v),
            "clocks": clk, "l2": "inputs rotate over 2 sets (2 x 134 MB FP32 + 201 MB pieces per step > 126 MB L2)"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1904_06376_b200 as bx
    import synthetic
    from paper_1904_06376_b200.distributed import gemm_colsharded, local_columns

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BF16X_BENCH_BACKEND=gloo: a functional run of the N > 1 path with all ranks on the GPUs
    # there are (e.g. two ranks on one GPU) -- a check of the code path, never a measurement
    backend = os.environ.get("BF16X_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    bx.device_check()
    cfg = CONFIGS[args.config]
    v = args.variant
    p = bx.PIECES[v]
    m, n, k = cfg["m"], cfg["n"], cfg["k"]
    kp = (k + 7) // 8 * 8
    dev = torch.device("cuda", local)
    st = torch.cuda.current_stream()
    sh = int(st.cuda_stream)
    L = bx.lib()
    workload = cfg["label"].format(v=v, p=world)

    S = _sub_blocks(n // world, m) if world > 1 else 1
    cols = local_columns(n, world, rank, S)
    n_loc = len(cols)
    A_np = synthetic.uniform(m, k, seed=1) if rank == 0 else None
    B_np = synthetic.uniform(k, n, seed=2)
    A = torch.from_numpy(A_np).to(dev) if rank == 0 else \
        torch.empty_strided((m, k), (1, m), dtype=torch.float32, device=dev)
    B_loc = torch.from_numpy(np.asfortranarray(B_np[:, cols])).to(dev) if world > 1 else torch.from_numpy(B_np).to(dev)
    C = torch.empty_strided((m, n), (1, m), dtype=torch.float32, device=dev)
    Ap = torch.empty(p * m * kp, dtype=torch.uint16, device=dev)
    Bp = torch.empty(p * n_loc * kp, dtype=torch.uint16, device=dev)
    C_loc = C if world == 1 else torch.empty_strided((m, n_loc), (1, m), dtype=torch.float32, device=dev)

    # N = 1: events around the split and the GEMM of every timed step (on the launching stream)
    # give the roofline's per-launch durations from the timed region itself; at this size an
    # event between the split and the PDL-launched GEMM costs ~1 us of overlap in a ~40 ms step
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    if world == 1:
        def run_step(i):
            _split_gemm_step(L, bx, m, n, k, v, p, A, B_loc, C, Ap, Bp, sh,
                             evs[i] if 0 <= i < args.steps else None, st)
    else:
        def run_step(i):
            gemm_colsharded(A, B_loc, C, variant=v, sub_blocks=S, k_chunks=4)

    for i in range(args.warmup):
        run_step(-1 - i)
    torch.cuda.synchronize()
    launches0 = bx.launch_count()
    total_ms, clocks = _timed(run_step, args.steps, st, local, world, dist)
    launches = bx.launch_count() - launches0
    if world == 1:
        split_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
        gemm_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    else:
        # the rank's own block (split + GEMM with events around each launch) after the timed region
        if world > 1:
            dist.barrier()
        split_ms, gemm_ms = _evented(L, bx, m, n_loc, k, v, p, [(A, B_loc)], C_loc, Ap, Bp, sh, st,
                                     max(1, min(args.steps, 5)))
    if world > 1:
        t = torch.tensor([total_ms, split_ms, gemm_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, split_ms, gemm_ms = (float(x) for x in t.tolist())
    ms_step = total_ms / args.steps
    flops_step = 2.0 * m * n * k
    value = flops_step / (ms_step * 1e-3) / 1e12

    peak_burst, peak_sust, hbm, peak_src = _peaks()
    mma_flops = v * 2.0 * m * n_loc * k            # algorithmic BF16 MMA flops per GEMM launch
    achieved = mma_flops / (gemm_ms * 1e-3) / 1e12
    long_kernel = gemm_ms > 5.0                     # timed inside a long step: the sustained peak applies
    peak = peak_sust if long_kernel else peak_burst
    mc = 2 if m * n_loc >= 12288 * 12288 else 1
    kname = f"gemm_split_kernel<2,{v},256,2,{mc}>"
    ncu_ent = _ncu(f"gemm_split_kernel_v{v}_{m}x{n_loc}x{k}", f"{m}x{n_loc}x{k} bf16x{v}")
    split_bytes = (4 + 2 * p) * (m * k + k * n_loc)

    # e2e: the public host-buffer entry point (H2D of A and B from pinned memory, split, GEMM,
    # D2H of C), each rank its own column block
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    A_h = torch.empty_strided((m, k), (1, m), dtype=torch.float32).pin_memory()
    B_h = torch.empty_strided((k, n_loc), (1, k), dtype=torch.float32).pin_memory()
    C_h = torch.empty_strided((m, n_loc), (1, m), dtype=torch.float32).pin_memory()
    A_h.copy_(torch.from_numpy(A_np) if rank == 0 else A.cpu())
    B_h.copy_(B_loc.cpu())
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
    del A_h, B_h, C_h

    line = {
        "metric": METRIC, "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong" if args.config in ("c4", "c4b") else "weak",
        "vs_baseline": None, "dtype": "f32", "mma_dtype": "bf16 x bf16 -> f32 (tcgen05 kind::f16)",
        "data": "synthetic",
        "config": {"workload": workload, "m": m, "n": n, "k": k, "n_per_gpu": n_loc, "variant": v,
                   "inputs": "A, B ~ U[-1,1] (FP64 draws rounded to FP32), seeded, column-major",
                   "l2": f"inputs {4 * (m * k + k * n_loc) / 2 ** 30:.0f} GiB FP32 + {2 * p * (m * k + k * n_loc) / 2 ** 30:.0f} GiB "
                         f"of pieces per step >> 126 MB L2; no flush needed"
                         if args.config in ("c4", "c4b") else "one input set (use --config c4 for the headline)",
                   "parallelism": (f"column blocks of C, dp{world} (gemm_colsharded: {S} sub-blocks per rank, "
                                   f"A broadcast in 4 k-chunks and split once per rank, all-gathers on a side "
                                   f"stream)") if world > 1 else "single GPU"},
        "pct_of_scaled_roofline": 100.0 * value / world / (peak_burst / v),
        "pct_of_scaled_roofline_sustained": 100.0 * value / world / (peak_sust / v),
        "split_ms": split_ms, "gemm_ms": gemm_ms,
        "split_gbs": split_bytes / (split_ms * 1e-3) / 1e9,
        "roofline": {"bound": "tensor", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak,
                     "traffic": float(ncu_ent["dram_bytes_per_launch"]) if ncu_ent else None,
                     "peak_source": f"{peak_src} bf16 " + ("sustained (MEASURED_PEAKS.json bf16_tflops_sustained): a "
                                                            f"{gemm_ms:.0f} ms kernel timed back to back"
                                                            if long_kernel else "burst (MEASURED_PEAKS.json bf16_tflops)"),
                     "achieved_def": f"{v} products x 2 m n_loc k BF16 MMA flops per launch / mean CUDA-event launch "
                                     f"time" + (" (events around each launch inside the timed region)" if world == 1
                                                else " (the rank's block, evented pass after the timed region)"),
                     "frac_of_burst": achieved / peak_burst},
        "e2e": {"value": e2e_value, "unit": "TFLOPS", "h2d_bytes_per_step": 4 * (m * k + k * n_loc),
                "d2h_bytes_per_step": 4 * m * n_loc, "steps": e2e_steps,
                "api": "bf16x_gemm_host (pinned host buffers; H2D A, B + split + GEMM + D2H C, pipelined over "
                       "row blocks of A x column blocks of B)" + ("; each rank its own column block" if world > 1 else "")},
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and args.config == "c4" and not args.no_secondary:
        line["secondary"] = secondary_4096(L, bx, v, p, dev, st, sh, 20, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(m, n, k, v, args.cpu_cols, A=A_np, B=B_np)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--variant", type=int, default=6, choices=[1, 3, 5, 6, 7, 8, 9])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-cols", type=int, default=0, help="oracle sample (columns) for cpu_baseline; 0 = about 15 s")
    ap.add_argument("--ref-cols", type=int, default=64, help="oracle sample (columns) per --impl reference step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the configs[1] (4096^3) secondary keys")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
