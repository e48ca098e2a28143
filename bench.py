#!/usr/bin/env python
"""ICNNM hot-path benchmark (BASELINE.json metric: voxel-iterations/s).

Default workload: BASELINE config 2 (128x128x32 video completion, kernel
9x9x5 -> k = 405, 20% observed, 300 iterations), one complete ICNNM solve per
step on inputs already resident in HBM.  N > 1 (torchrun): every rank solves
its own independently seeded config-2 tensor (batch split, no data-path
collective) -> weak scaling; value = total voxel-iterations / max-over-ranks
device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C]
  python bench.py --impl reference ...   # reference CPU path (oracle port)

Synthetic data (BASELINE.json's generator; no datasets exist here).  Every
step's W state (0.85 GB) exceeds L2 (126 MB), so no explicit L2 flush.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "ICNNM voxel-iterations/sec"
UNIT = "voxel-iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--engine", default="tf32x3", choices=["tf32x3", "ffma"])
    ap.add_argument("--iters", type=int, default=0, help="override iterations per solve")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def measure_tf32_peak(dev: int) -> float:
    """Dense TF32 tensor throughput (cuBLAS 8192^3, best of 5) on this GPU --
    the denominator of the TF32x3 engine's roofline (MEASURED_PEAKS.json has
    only bf16)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        n = 8192
        a = torch.randn(n, n, device=f"cuda:{dev}")
        b = torch.randn(n, n, device=f"cuda:{dev}")
        for _ in range(2):
            a @ b
        best = 0.0
        for _ in range(5):
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record()
            a @ b
            s1.record()
            s1.synchronize()
            best = max(best, 2 * n ** 3 / (s0.elapsed_time(s1) * 1e-3) / 1e12)
        del a, b
        return best
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev


def load_ncu_traffic(engine: str):
    """dram bytes per launch of the dominant kernels from the committed ncu
    --set full capture (profiles/ncu_summary_*.json), if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary_latest.json")) as f:
            d = json.load(f)
        return d.get(engine)
    except Exception:
        return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# --------------------------------------------------------------------------
# reference arm: the reference's CPU path (oracle port; the C++ reference
# needs Eigen3 + FFTW3, absent in this image) on all host cores
# --------------------------------------------------------------------------
def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    ncores = os.cpu_count() or 1
    os.environ["ICNNM_ORACLE_THREADS"] = str(ncores)
    from threadpoolctl import threadpool_limits
    from paper_2604_17001_b200 import synth
    from oracle import icnnm_oracle as O
    O.WORKERS = ncores
    w = synth.WORKLOADS[args.config]
    X = w.target()
    mask = w.mask()
    with threadpool_limits(limits=ncores):
        B = O.learn_ensemble_basis(w.training(), w.kernel)
        s = O.AdmmSolver(X * mask, mask, B,
                         O.SolverConfig(max_iters=w.iters, tol_primal=1e-300, tol_change=1e-300))
        for _ in range(args.warmup):
            s.step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s.step()
        dt = time.perf_counter() - t0
    value = w.m * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"BASELINE config {args.config}", "dims": list(w.dims),
                   "kernel": list(w.kernel), "k": w.k,
                   "step": "one ADMM iteration of the literal fp64 reference loop "
                           "(solver.cpp:107-139) -- bounded sample of the "
                           f"{w.iters}-iteration solve"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "port",
                         "sample": f"{args.steps} ADMM iterations of config {args.config} "
                                   f"after {args.warmup} warm-up iterations"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_sample(w, X, mask, B, budget_s=20.0):
    """Oracle (port) on 1 core, bounded sample of the same workload."""
    os.environ["ICNNM_ORACLE_THREADS"] = "1"
    from threadpoolctl import threadpool_limits
    from oracle import icnnm_oracle as O
    O.WORKERS = 1
    with threadpool_limits(limits=1):
        ob = O.EigenBasis(B.kernel_shape, B.K, B.eigenvalues)
        s = O.AdmmSolver(X * mask, mask, ob,
                         O.SolverConfig(max_iters=w.iters, tol_primal=1e-300, tol_change=1e-300),
                         validate_basis=False)
        t0 = time.perf_counter()
        n = 0
        while True:
            s.step()
            n += 1
            if time.perf_counter() - t0 > budget_s or n >= w.iters:
                break
        dt = time.perf_counter() - t0
    return {"value": w.m * n / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{n} ADMM iterations of the literal fp64 oracle on config {w.cfg} "
                      f"(1 thread, {dt:.1f} s)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    rank, world, local = dist_env()
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2604_17001_b200 as P
    from paper_2604_17001_b200 import synth

    w = synth.WORKLOADS[args.config]
    iters = args.iters or w.iters
    dev = local
    # per-rank independent tensor (batch split, weak scaling)
    X = w.target(b=rank)
    mask = w.mask()
    M = X * mask
    B = P.learn_ensemble_basis(w.training(), w.kernel, device=dev)
    cfg = P.SolverConfig(max_iters=iters, tol_primal=1e-300, tol_change=1e-300,
                         engine=args.engine)
    S = P.Solver(X.shape, B, device=dev)
    S.upload(M, mask)

    for _ in range(args.warmup):
        S.run(cfg)
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()

    dev_s = []
    launches = 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            rep = S.run(cfg)
            dev_s.append(rep.device_seconds)
            launches += S.last_launches
    torch.cuda.synchronize(dev)
    t_local = float(sum(dev_s))
    t_max = t_local
    if dist:
        t = torch.tensor([t_local], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
        dist.barrier()
    value = w.m * iters * args.steps * world / t_max
    L = S.download()
    psnr = synth.psnr(X, L)

    # per-kernel times (live, CUDA events on the solver stream) for roofline
    S.set_profile(True)
    S.run(cfg)
    kt = S.kernel_times_ms()
    S.set_profile(False)

    line = None
    if rank == 0:
        peaks = load_peaks()
        k = w.k
        flops_fwd = 2.0 * w.m * k * k            # algorithmic, per launch
        flops_adj = 2.0 * w.m * k * k
        dom = "forward" if kt["forward"] >= kt["adjoint"] else "adjoint"
        t_dom = kt[dom] * 1e-3
        achieved = (flops_fwd if dom == "forward" else flops_adj) / t_dom / 1e12
        if args.engine == "tf32x3":
            tf32 = measure_tf32_peak(dev)
            roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": tf32 / 3.0,
                    "unit": "TFLOP/s", "frac": achieved / (tf32 / 3.0),
                    "peak_source": "measured dense TF32 (cuBLAS 8192^3 burst, %.0f TFLOP/s) / 3 "
                                   "tensor MMAs per fp32 product" % tf32,
                    "tensor_pipe_frac": 3.0 * achieved / tf32}
        else:
            ffma_peak = P.probe_ffma_tflops(dev)
            roof = {"bound": "fp32", "kernel": dom, "achieved": achieved, "peak": ffma_peak,
                    "unit": "TFLOP/s", "frac": achieved / ffma_peak,
                    "peak_source": "measured FFMA probe (icnnm_probe_ffma_tflops)"}
        traffic = load_ncu_traffic(args.engine)
        roof["traffic"] = traffic.get(dom) if isinstance(traffic, dict) else None
        roof["algorithmic_bytes"] = (8.0 if dom == "forward" else 4.0) * w.m * k
        roof["per_launch_ms"] = kt
        roof["flops_per_launch"] = flops_fwd
        e2e = None
        if not args.no_e2e:
            e2e_t = []
            for _ in range(max(1, min(args.steps, 3))):
                Mh = np.ascontiguousarray(M)
                t0 = time.perf_counter()
                Lh, r = P.icnnm_solve(Mh, mask, B, cfg, device=dev)
                e2e_t.append(time.perf_counter() - t0)
            te = float(np.mean(e2e_t))
            e2e = {"value": w.m * iters / te, "unit": UNIT,
                   "h2d_bytes_per_step": int(M.nbytes + mask.nbytes + B.K.nbytes),
                   "d2h_bytes_per_step": int(Lh.nbytes + 3 * 8 * iters),
                   "path": "icnnm_cuda_solve C ABI, host f64 buffers, incl. validation, "
                           "allocation, H2D, solve, D2H"}
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline_sample(w, X, mask, B)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (BASELINE.json generator, seeded)",
            "config": {"workload": f"BASELINE config {args.config}: {w.dims[0]}x{w.dims[1]}x"
                                   f"{w.dims[2]} kernel {w.kernel[0]}x{w.kernel[1]}x"
                                   f"{w.kernel[2]} (k={k}), {iters} iterations per step",
                       "engine": args.engine, "step": "one full ICNNM solve from HBM",
                       "l2": "inputs larger than L2 (W state %.2f GB)" % (
                           w.m * ((k + 63) // 64 * 64) * 4 / 1e9),
                       "parallelism": f"batch split x{world} (independent tensors)"},
            "psnr_db": psnr,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "hbm_peak_gbs": peaks.get("hbm_gbs"),
        }
        print(json.dumps(line), flush=True)
    S.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
