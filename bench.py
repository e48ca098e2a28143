#!/usr/bin/env python
"""ICNNM hot-path benchmark (BASELINE.json metric: voxel-iterations/s).

Default workload: BASELINE config 4 -- frame interpolation, a batch of 64
independent 128x128x32 tensors (even frames observed), kernel 7x7x5 (k = 245),
200 iterations each, one shared eigenvector set.  One *step* is the rank's
share of the 64-tensor batch (contiguous block; N = 1: all 64), each tensor a
complete ICNNM solve; the batch is split over the ranks with no inter-GPU
communication (BASELINE: "split across 1/2/4/8 GPUs"), so total work is
fixed as N grows: scaling "strong".  value = 64 * m * iterations * steps /
(max over ranks of the summed per-solve device time, CUDA events on the
solver stream; the inputs of each solve are resident in HBM before its
timed region starts).  e2e = the same metric through the public batch call
(icnnm_cuda_solve_batch: host f64 inputs, validation, H2D, solves, D2H).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C]
  python bench.py --impl reference ...   # the reference's CPU path (oracle port)

Configs 1-3 run one tensor per rank (replicas, weak scaling); config 5 is the
H-sharded single tensor (halo exchange + all-reduce; strong scaling).
Synthetic data (BASELINE.json's generator, seeded; no datasets exist here).
Every solve's W state (config 4: 0.54 GB) exceeds L2 (126 MB): no explicit
L2 flush is needed between timed iterations.
"""
from __future__ import annotations

import argparse
import hashlib
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
DEFAULT_CONFIG = 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--engine", default="f16x3", choices=["f16x3", "tf32x3", "ffma"])
    ap.add_argument("--iters", type=int, default=0, help="override iterations per solve")
    ap.add_argument("--batch", type=int, default=0, help="override the config-4 batch size")
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


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def lib_sha16() -> str:
    """Identity of the product library's kernel sources (pairs an ncu traffic
    capture with a build: the hash of the tcgen05 / elementwise kernel sources,
    which a rebuild on another box reproduces, unlike a hash of the .so)."""
    h = hashlib.sha256()
    base = os.path.join(ROOT, "paper_2604_17001_b200", "csrc")
    try:
        for name in ("icnnm_tc.cu", "icnnm_tc.cuh", "icnnm_kernels.cu", "icnnm_kernels.cuh"):
            with open(os.path.join(base, name), "rb") as f:
                h.update(f.read())
    except OSError:
        return "missing"
    return h.hexdigest()[:16]


def load_ncu_traffic(config: int, engine: str):
    """DRAM bytes (read + write) per launch of the forward / adjoint kernels
    from the committed `ncu --set full` capture of this build and config
    (profiles/ncu_traffic_r2.json, written by tools/ncu_traffic.py); None when
    the capture is of another build (then the traffic is unmeasured)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r2.json")) as f:
            d = json.load(f)
    except Exception:
        return None, "no capture"
    e = d.get(f"config{config}", {}).get(engine)
    if not e:
        return None, "no capture of this config/engine"
    if e.get("lib_sha16") != lib_sha16():
        return None, "capture is of build %s, this is %s" % (e.get("lib_sha16"), lib_sha16())
    return e, "ncu --set full, this build (%s)" % e.get("lib_sha16")


def workload(args, synth):
    w = synth.WORKLOADS[args.config]
    if args.dims:
        w = synth.scaled(w, tuple(args.dims))
    if args.iters:
        w = synth.scaled(w, w.dims, iters=args.iters)
    if args.batch and args.config == 4:
        import dataclasses
        w = dataclasses.replace(w, batch=args.batch)
    return w


def rank_share(nb: int, rank: int, world: int):
    """Contiguous block of the batch for this rank (as icnnm_cuda_solve_batch
    splits over devices)."""
    return list(range(nb * rank // world, nb * (rank + 1) // world))


# --------------------------------------------------------------------------
# reference arm: the reference's CPU path.  The C++ reference needs Eigen3 +
# FFTW3 (absent in this image), so this is the fp64 oracle port of its
# solver (oracle/icnnm_oracle.py) on all host cores.  Inputs come from
# synthgen; neither module loads the product library.
# --------------------------------------------------------------------------
def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    ncores = os.cpu_count() or 1
    os.environ["ICNNM_ORACLE_THREADS"] = str(ncores)
    from threadpoolctl import threadpool_limits
    import synthgen as synth
    from oracle import icnnm_oracle as O
    O.WORKERS = ncores
    w = workload(args, synth)
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
        "scaling": "strong" if args.config == 4 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (BASELINE.json generator, seeded)",
        "config": {"workload": f"BASELINE config {args.config}", "dims": list(w.dims),
                   "kernel": list(w.kernel), "k": w.k, "iterations": w.iters,
                   "batch": w.batch,
                   "step": "one ADMM iteration of the literal fp64 reference loop "
                           "(solver.cpp:107-139) on tensor 0 of the batch -- a bounded "
                           f"sample of the {w.batch} x {w.iters}-iteration workload"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "port",
                         "sample": f"{args.steps} ADMM iterations of config {args.config} "
                                   f"tensor 0 after {args.warmup} warm-up iterations"},
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
                      f"tensor 0 (1 thread, {dt:.1f} s)"}


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
    import synthgen as synth

    w = workload(args, synth)
    iters = w.iters
    dev = local
    cfg = P.SolverConfig(max_iters=iters, tol_primal=1e-300, tol_change=1e-300,
                         engine=args.engine)
    B = P.learn_ensemble_basis(w.training(), w.kernel, device=dev)

    if args.config == 5:
        return bench_sharded(args, w, B, cfg, iters, rank, world, dev, dist)

    # config 4: the batch is split over the ranks (fixed total work, strong
    # scaling); configs 1-3: every rank solves its own tensor (replicas)
    if args.config == 4:
        mine = rank_share(w.batch, rank, world)
        scaling, units_total = "strong", w.batch
    else:
        mine = [rank]
        scaling, units_total = "weak", world
    mask = w.mask()
    targets = {b: w.target(b=b) for b in mine}
    obs = {b: targets[b] * mask for b in mine}
    S = P.Solver(w.dims, B, device=dev)

    def step():
        t = 0.0
        n = 0
        for b in mine:
            S.upload(obs[b], mask)          # H2D before the solve's timed region
            rep = S.run(cfg)                # device-resident solve, CUDA events
            t += rep.device_seconds
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

    # per-kernel times (live, CUDA events on the solver stream) for the roofline
    S.upload(obs[mine[0]], mask)
    S.set_profile(True)
    S.run(cfg)
    kt = S.kernel_times_ms()
    S.set_profile(False)
    S.close()

    # end to end through the public batch call, host buffers (every rank, its share)
    e2e = None
    if not args.no_e2e:
        Ms = [obs[b] for b in mine]
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        Ls, reps = P.icnnm_solve_batch(Ms, mask, B, cfg, devices=[dev])
        te = time.perf_counter() - t0
        te = max_over_ranks(dist, dev, te)
        n_mine = len(mine)
        e2e = {"value": w.m * iters * units_total / te, "unit": UNIT,
               "h2d_bytes_per_step": int(n_mine * (obs[mine[0]].nbytes + mask.nbytes)
                                         + B.K.nbytes),
               "d2h_bytes_per_step": int(n_mine * (Ls[0].nbytes + 3 * 8 * iters)),
               "seconds": te,
               "path": "icnnm_cuda_solve_batch C ABI on host f64 buffers: basis validation, "
                       "per-tensor input validation, allocation, H2D, %d solves, D2H of L and "
                       "the per-iteration reports, all inside the timed region (wall clock, "
                       "max over ranks)" % n_mine,
               "psnr_db_last": synth.psnr(targets[mine[-1]], Ls[-1])}

    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and w.m * w.k <= 3e8:
            cpu = cpu_baseline_sample(w, obs[mine[0]], mask, B)
        report_line(args, P, w, iters, world, value, t_max, kt, psnr, launches, clk, scaling,
                    e2e, cpu, n_per_rank=len(mine),
                    extra={"step_device_s": [round(x, 5) for x in dev_s]})
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def bench_sharded(args, w, B, cfg, iters, rank, world, dev, dist):
    """BASELINE config 5: one tensor H-sharded over the ranks (halo exchange +
    one NCCL all-reduce per iteration), strong scaling."""
    import paper_2604_17001_b200 as P
    import synthgen as synth
    local_slabs = 1
    if world == 1:
        need = w.m * ((w.k + 127) // 128 * 128) * 4
        if need > 150e9:
            if rank == 0:
                print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": 1,
                                  "unavailable": "config 5 W state (%.0f GB) exceeds one B200; "
                                                 "run with --gpus >= 2 or --dims" % (need / 1e9)}))
            return 0

    # every solve builds its own communicator, so every solve needs a fresh
    # unique id (an id bootstraps exactly one ncclCommInitRank)
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
    peaks = load_peaks()
    f16 = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops") or 1393.6
    achieved = 4.0 * w.m * w.k * w.k * iters * args.steps / t_max / 1e12
    roof = {"bound": "tensor", "kernel": "whole iteration (solve-level)",
            "achieved": achieved / world, "peak": f16 / 3.0, "unit": "TFLOP/s",
            "frac": achieved / world / (f16 / 3.0),
            "peak_source": "MEASURED_PEAKS.json dense bf16 sustained / 3 kind::f16 MMAs per "
                           "fp32 product; per GPU", "traffic": None}
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


def kernel_roofline(w, kt, peaks, engine, P, dev):
    """Per-kernel rooflines: algorithmic flops 2 m k^2 per launch (either
    contraction) on the pipe used (F16x3: 3 kind::f16 MMAs per fp32 product)
    and algorithmic bytes (forward: W read + written, 8 m k, + L~ 4 m; adjoint:
    W read 4 m k + adj written 4 m); each kernel's bound is the
    slower of the two at the measured peaks (sustained bf16: the kernels run
    inside a seconds-long solve)."""
    k, m = w.k, w.m
    flops = 2.0 * m * k * k
    hbm = peaks.get("hbm_gbs") or 6550.1
    if engine == "f16x3":
        tpeak = (peaks.get("bf16_tflops_sustained") or 1393.6) / 3.0
        src = "MEASURED_PEAKS.json bf16 sustained %.1f TFLOP/s / 3 kind::f16 MMAs per fp32 " \
              "product; HBM %.1f GB/s" % (tpeak * 3, hbm)
    elif engine == "tf32x3":
        tpeak = (peaks.get("bf16_tflops_sustained") or 1393.6) / 2.0 / 3.0
        src = "half the bf16 sustained rate (kind::tf32 K=8) / 3 MMAs per product"
    else:
        tpeak = P.probe_ffma_tflops(dev)
        src = "measured FFMA probe"
    out = {}
    for name, nbytes in (("forward", 8.0 * m * k + 4.0 * m), ("adjoint", 4.0 * m * k + 4.0 * m)):
        ms = kt[name]
        t_tensor = flops / (tpeak * 1e12) * 1e3
        t_hbm = nbytes / (hbm * 1e9) * 1e3
        bound = "hbm" if t_hbm > t_tensor else "tensor"
        if bound == "hbm":
            achieved, peak, unit = nbytes / (ms * 1e-3) / 1e9, hbm, "GB/s"
        else:
            achieved, peak, unit = flops / (ms * 1e-3) / 1e12, tpeak, "TFLOP/s"
        out[name] = {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak, "ms_per_launch": ms,
                     "algorithmic_bytes": nbytes, "algorithmic_flops": flops,
                     "roofline_ms": max(t_tensor, t_hbm)}
    return out, src


def report_line(args, P, w, iters, world, value, t_max, kt, psnr, launches, clk, scaling,
                e2e, cpu, n_per_rank, extra=None):
    peaks = load_peaks()
    per, src = kernel_roofline(w, kt, peaks, args.engine, P, 0)
    dom = "forward" if kt["forward"] >= kt["adjoint"] else "adjoint"
    d = per[dom]
    traffic, tsrc = load_ncu_traffic(args.config, args.engine)
    roof = {"bound": d["bound"], "kernel": dom, "achieved": d["achieved"], "peak": d["peak"],
            "unit": d["unit"], "frac": d["frac"],
            "traffic": (traffic or {}).get(dom),
            "traffic_source": tsrc,
            "peak_source": src,
            "per_kernel": per,
            "per_launch_ms": kt,
            # the whole iteration against its roofline (both contractions +
            # the elementwise kernels, vs the sum of the two kernels' bounds)
            "iteration_frac": (per["forward"]["roofline_ms"] + per["adjoint"]["roofline_ms"])
            / (t_max * 1e3 / (args.steps * n_per_rank * iters))}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (BASELINE.json generator, seeded)",
        "config": {"workload": f"BASELINE config {args.config}: "
                               + (f"batch of {w.batch} x " if args.config == 4 else "")
                               + f"{w.dims[0]}x{w.dims[1]}x{w.dims[2]} kernel "
                               f"{w.kernel[0]}x{w.kernel[1]}x{w.kernel[2]} (k={w.k}), "
                               f"{iters} iterations per solve",
                   "engine": args.engine,
                   "step": ("the rank's share of the %d-tensor batch (%d tensors), one full "
                            "ICNNM solve each from HBM" % (w.batch, n_per_rank))
                   if args.config == 4 else "one full ICNNM solve from HBM",
                   "l2": "inputs larger than L2 (W state %.2f GB per solve)" % (
                       w.m * ((w.k + 15) // 16 * 16) * 4 / 1e9),
                   "parallelism": ("batch split x%d (no communication)" % world)
                   if args.config == 4 else "replicas x%d" % world},
        "psnr_db": psnr,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "lib_sha16": lib_sha16(),
    }
    if extra:
        line["timing_detail"] = extra
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    sys.exit(main())
