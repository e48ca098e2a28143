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
    ap.add_argument("--engine", default="f16x3", choices=["f16x3", "tf32x3", "ffma"])
    ap.add_argument("--iters", type=int, default=0, help="override iterations per solve")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dims", type=int, nargs=3, default=None,
                    help="scaled run of the config's recipe (parity / smoke only)")
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
        pw = []
        for r in self.rows:
            try:
                pw.append(float(r[2]))
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows),
                "sm_mhz_min": min(sm) if sm else None,
                "power_w_max": max(pw) if pw else None}


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


def measure_f16_peak(dev: int) -> float:
    """Dense fp16 tensor throughput (cuBLAS 8192^3, best of 5): fallback
    denominator of the F16x3 engine when MEASURED_PEAKS.json is absent."""
    import torch
    n = 8192
    a = torch.randn(n, n, device=f"cuda:{dev}", dtype=torch.float16)
    b = torch.randn(n, n, device=f"cuda:{dev}", dtype=torch.float16)
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


def cpu_baseline_sample(w, M, mask, B, budget_s=20.0):
    """Oracle (port) on 1 core, bounded sample of the same workload."""
    os.environ["ICNNM_ORACLE_THREADS"] = "1"
    from threadpoolctl import threadpool_limits
    from oracle import icnnm_oracle as O
    O.WORKERS = 1
    with threadpool_limits(limits=1):
        ob = O.EigenBasis(B.kernel_shape, B.K, B.eigenvalues)
        s = O.AdmmSolver(M, mask, ob,
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


def setup_dist(world, local):
    import torch
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return dist
    return None


def max_over_ranks(dist, dev, x):
    if not dist:
        return x
    import torch
    t = torch.tensor([x], device=f"cuda:{dev}", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    rank, world, local = dist_env()
    import torch
    dist = setup_dist(world, local)
    import paper_2604_17001_b200 as P
    from paper_2604_17001_b200 import synth

    w = synth.WORKLOADS[args.config]
    if args.dims:
        w = synth.scaled(w, tuple(args.dims))
    iters = args.iters or w.iters
    dev = local
    cfg = P.SolverConfig(max_iters=iters, tol_primal=1e-300, tol_change=1e-300,
                         engine=args.engine)
    B = P.learn_ensemble_basis(w.training(), w.kernel, device=dev)

    if args.config == 5:
        return bench_sharded(args, w, B, cfg, iters, rank, world, dev, dist)

    # batch of tensors for this rank: cfg 4 splits the 64-tensor batch over
    # the ranks (strong scaling); cfgs 1-3 give every rank its own tensor
    # (independent replicas, weak scaling)
    if args.config == 4:
        nb = w.batch
        mine = list(range(rank, nb, world))
        scaling, units_total = "strong", nb
    else:
        mine = [rank]
        scaling, units_total = "weak", world
    mask = w.mask()
    targets = {b: w.target(b=b) for b in mine}
    S = P.Solver(w.dims, B, device=dev)

    loops = []

    def step():
        t = 0.0
        n = 0
        for b in mine:
            S.upload(targets[b] * mask, mask)
            rep = S.run(cfg)
            t += rep.device_seconds
            loops.append(rep.loop_seconds)
            n += S.last_launches
        return t, n

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    dev_s = []
    launches = 0
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            t, n = step()
            dev_s.append(t)
            launches += n
    torch.cuda.synchronize(dev)
    t_max = max_over_ranks(dist, dev, float(sum(dev_s)))
    if dist:
        dist.barrier()
    value = w.m * iters * args.steps * units_total / t_max
    L = S.download()
    psnr = synth.psnr(targets[mine[-1]], L)

    # per-kernel times (live, CUDA events on the solver stream) for roofline
    S.set_profile(True)
    S.run(cfg)
    kt = S.kernel_times_ms()
    S.set_profile(False)

    if rank == 0:
        report_line(args, P, w, B, cfg, iters, dev, world, value, t_max, kt, psnr, launches,
                    clk, scaling, mask, targets[mine[0]] * mask,
                    extra={"step_device_s": [round(x, 5) for x in dev_s],
                           "loop_s": [round(x, 5) for x in loops[-args.steps:]]})
    S.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def bench_sharded(args, w, B, cfg, iters, rank, world, dev, dist):
    """BASELINE config 5: one tensor H-sharded over the ranks (halo exchange +
    one NCCL all-reduce per iteration), strong scaling."""
    import torch
    import paper_2604_17001_b200 as P
    from paper_2604_17001_b200 import synth
    local_slabs = 1
    if world == 1:
        need = w.m * ((w.k + 127) // 128 * 128) * 4
        if need > 150e9:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": 1,
                                  "unavailable": "config 5 W state (%.0f GB) exceeds one B200; "
                                                 "run with --gpus >= 2 or --dims" % (need / 1e9)}))
            return 0
    # the NCCL transport is in the loop at every N: at N = 1 a one-rank
    # communicator carries the halo shifts (self send/recv) and the all-reduce.
    # Every solve builds its own communicator, so every solve needs a fresh
    # unique id (an id bootstraps exactly one ncclCommInitRank).
    def fresh_id():
        nid = P.dist_unique_id() if rank == 0 else None
        if world > 1:
            obj = [nid]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        return nid
    X = w.target()
    mask = w.mask()
    M = X * mask
    times = []
    with ClockSampler(dev) as clk:
        for it in range(args.warmup + args.steps):
            if dist:
                dist.barrier()
            nid = fresh_id()
            row0, rows, rep = P.sharded_solve(M, mask, B, cfg, local_slabs=local_slabs,
                                              world=world, rank=rank, nccl_id=nid, device=dev)
            if it >= args.warmup:
                times.append(rep.device_seconds)
    t_max = max_over_ranks(dist, dev, float(sum(times)))
    value = w.m * iters * args.steps / t_max
    # solve-level roofline: both contractions' algorithmic flops (4 m k^2 per
    # iteration, all ranks) over the whole device time of the solve -- the
    # elementwise kernels, halo exchange and all-reduce count against it
    peaks = load_peaks()
    f16 = peaks.get("bf16_tflops") or 1650.0
    achieved = 4.0 * w.m * w.k * w.k * iters * args.steps / t_max / 1e12
    roof = {"bound": "tensor", "kernel": "whole iteration (solve-level)",
            "achieved": achieved / world, "peak": f16 / 3.0, "unit": "TFLOP/s",
            "frac": achieved / world / (f16 / 3.0),
            "peak_source": "MEASURED_PEAKS.json dense bf16 / 3 kind::f16 MMAs per fp32 product; "
                           "per GPU", "traffic": None}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (BASELINE.json generator, seeded)",
                "config": {"workload": "BASELINE config 5 %s kernel %s, %d iterations, H-sharded "
                                       "over %d ranks" % ("x".join(map(str, w.dims)),
                                                          "x".join(map(str, w.kernel)), iters, world),
                           "engine": args.engine, "parallelism": f"H-shard x{world}"},
                "psnr_db_own_rows": synth.psnr(X[row0:row0 + rows.shape[0]], rows),
                "roofline": roof,
                "transport": "NCCL (ncclSend/ncclRecv halo shifts + ncclAllReduce of the "
                             "k+8 reduction vector, captured in the solve graph)",
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def report_line(args, P, w, B, cfg, iters, dev, world, value, t_max, kt, psnr, launches, clk,
                scaling, mask, M, extra=None):
    import numpy as np
    from paper_2604_17001_b200 import synth
    peaks = load_peaks()
    k = w.k
    flops = 2.0 * w.m * k * k            # algorithmic, per launch (either contraction)
    dom = "forward" if kt["forward"] >= kt["adjoint"] else "adjoint"
    achieved = flops / (kt[dom] * 1e-3) / 1e12
    if args.engine == "tf32x3":
        tf32 = measure_tf32_peak(dev)
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": tf32 / 3.0,
                "unit": "TFLOP/s", "frac": achieved / (tf32 / 3.0),
                "peak_source": "measured dense TF32 (cuBLAS 8192^3 burst, %.0f TFLOP/s) / 3 "
                               "tensor MMAs per fp32 product" % tf32,
                "tensor_pipe_frac": 3.0 * achieved / tf32}
    elif args.engine == "f16x3":
        f16 = peaks.get("bf16_tflops")
        src = "MEASURED_PEAKS.json dense bf16 (burst)"
        if not f16:
            f16, src = measure_f16_peak(dev), "measured dense fp16 (cuBLAS 8192^3 burst)"
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": f16 / 3.0,
                "unit": "TFLOP/s", "frac": achieved / (f16 / 3.0),
                "peak_source": "%s %.0f TFLOP/s / 3 kind::f16 MMAs per fp32 product "
                               "(kind::f16 runs at the bf16 rate)" % (src, f16),
                "tensor_pipe_frac": 3.0 * achieved / f16}
    else:
        ffma_peak = P.probe_ffma_tflops(dev)
        roof = {"bound": "fp32", "kernel": dom, "achieved": achieved, "peak": ffma_peak,
                "unit": "TFLOP/s", "frac": achieved / ffma_peak,
                "peak_source": "measured FFMA probe (icnnm_probe_ffma_tflops)"}
    traffic = load_ncu_traffic(args.engine) if args.config == 2 else None
    roof["traffic"] = traffic.get(dom) if isinstance(traffic, dict) else None
    roof["algorithmic_bytes"] = (8.0 if dom == "forward" else 4.0) * w.m * k
    roof["per_launch_ms"] = kt
    roof["flops_per_launch"] = flops
    e2e = None
    if not args.no_e2e:
        e2e_t = []
        # one untimed call first: like the device-timed steps, e2e is measured
        # warm (its first call allocates the 1 GB solver state next to the
        # still-open handle solver; later calls reuse the device block cache)
        P.icnnm_solve(np.ascontiguousarray(M), mask, B, cfg, device=dev)
        for _ in range(max(1, min(args.steps, 3))):
            Mh = np.ascontiguousarray(M)
            t0 = time.perf_counter()
            Lh, r = P.icnnm_solve(Mh, mask, B, cfg, device=dev)
            e2e_t.append(time.perf_counter() - t0)
        te = float(np.mean(e2e_t))
        e2e = {"value": w.m * iters / te * (world if args.config != 4 else 1), "unit": UNIT,
               "h2d_bytes_per_step": int(M.nbytes + mask.nbytes + B.K.nbytes),
               "d2h_bytes_per_step": int(Lh.nbytes + 3 * 8 * iters),
               "path": "icnnm_cuda_solve C ABI on host f64 buffers (validation, allocation, "
                       "H2D, solve, D2H inside the timed region); one tensor per rank"}
    cpu = None
    if not args.no_cpu_baseline and w.m * k <= 3e8:
        cpu = cpu_baseline_sample(w, M, mask, B)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (BASELINE.json generator, seeded)",
        "config": {"workload": f"BASELINE config {args.config}: {w.dims[0]}x{w.dims[1]}x"
                               f"{w.dims[2]} kernel {w.kernel[0]}x{w.kernel[1]}x"
                               f"{w.kernel[2]} (k={k}), {iters} iterations per solve",
                   "engine": args.engine,
                   "step": "one full ICNNM solve from HBM" + (
                       " per tensor of the rank's share of the 64-tensor batch"
                       if args.config == 4 else ""),
                   "l2": "inputs larger than L2 (W state %.2f GB)" % (
                       w.m * ((k + 127) // 128 * 128) * 4 / 1e9),
                   "parallelism": ("batch split x%d (no communication)" % world)},
        "psnr_db": psnr,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "hbm_peak_gbs": peaks.get("hbm_gbs"),
    }
    if extra:
        line["timing_detail"] = extra
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    sys.exit(main())
