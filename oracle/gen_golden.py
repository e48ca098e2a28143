"""Generate golden fixtures for the GPU parity tests (test infrastructure).

The reference ships no golden data (proj/test_output.txt is pass/fail only)
and cannot be built here (Eigen3/FFTW3 absent), so full-size fixtures come
from the pinned fp64 oracle (icnnm_oracle.py, itself checked against the
reference's known-answer tests in tests/test_oracle_pins.py).  Each fixture
stores the basis K it was solved with, so the GPU test feeds identical bits.
Inputs come from synthgen (the BASELINE recipes), never from the product.

  python -m oracle.gen_golden --config 2 [--threads 8] [--dims H W T] [--iters N]
  python -m oracle.gen_golden --config 4 --batch-index 21
  # config 3 at full size: m x k fp64 = 29.8 GB per matrix -> blocked loop with
  # Y, Z memory-mapped on disk (oracle/icnnm_oracle_blocked.py)
  python -m oracle.gen_golden --config 3 --iters 10 --blocked --store /tmp/cfg3
  # config-5 recipe at 128x128x64 (kernel 9x9x9), in-RAM blocked loop
  python -m oracle.gen_golden --config 5 --dims 128 128 64 --blocked
  # a full-size config-2 problem in a regime where the iteration recovers
  # signal (smooth low-rank video, 50% i.i.d. sampling, no noise)
  python -m oracle.gen_golden --config 2 --recover
"""
import argparse
import dataclasses
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# the "recovering" variant of a config's recipe: few sinusoids,
# no blobs, no noise -> a video of low convolution rank; 50% i.i.d. sampling;
# solved with init_fill = "mean" (solver.cpp:83-86)
RECOVER = dict(n_sin=4, n_blob=0, noise=0.0, mask_kind=0, mask_rate=0.5)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--dims", type=int, nargs=3, default=None)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--batch-index", type=int, default=0)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--blocked", action="store_true")
    ap.add_argument("--store", default=None, help="blocked: directory for memory-mapped Y, Z")
    ap.add_argument("--chunk", type=int, default=16)
    ap.add_argument("--slab-rows", type=int, default=8)
    ap.add_argument("--recover", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    os.environ["ICNNM_ORACLE_THREADS"] = str(a.threads)
    from threadpoolctl import threadpool_limits
    from oracle import icnnm_oracle as O
    import synthgen as synth
    O.WORKERS = a.threads
    w = synth.WORKLOADS[a.config]
    if a.dims:
        w = synth.scaled(w, tuple(a.dims), iters=a.iters or None)
    elif a.iters:
        w = synth.scaled(w, w.dims, iters=a.iters)
    if a.recover:
        w = dataclasses.replace(w, **RECOVER)
    X = w.target(b=a.batch_index)
    mask = w.mask()
    t0 = time.time()
    cfg = O.SolverConfig(max_iters=w.iters, tol_primal=1e-300, tol_change=1e-300,
                         init_fill="mean" if a.recover else "zero")

    def log(msg):
        print(f"[{time.time() - t0:8.1f} s] {msg}", flush=True)
    with threadpool_limits(limits=a.threads):
        B = O.learn_ensemble_basis(w.training(), w.kernel)
        log(f"basis learned (k = {w.k})")
        if a.blocked:
            from oracle import icnnm_oracle_blocked as OB
            L, rep = OB.icnnm_solve_blocked(X * mask, mask, B, cfg, store_dir=a.store,
                                            chunk=a.chunk, slab_rows=a.slab_rows,
                                            workers=a.threads, log=log)
        else:
            L, rep = O.icnnm_solve(X * mask, mask, B, cfg)
    dt = time.time() - t0
    tag = f"cfg{a.config}" + ("_recover" if a.recover else "") + \
          (f"_{'x'.join(map(str, w.dims))}" if a.dims else "") + \
          (f"_b{a.batch_index}" if a.batch_index else "") + f"_it{w.iters}"
    out = a.out or os.path.join(ROOT, "tests", "golden", tag + ".npz")
    pm = X * mask
    np.savez_compressed(out, L=L.astype(np.float32), K=B.K, eigenvalues=B.eigenvalues,
                        kernel=np.array(w.kernel), dims=np.array(w.dims), iters=w.iters,
                        config=a.config, batch_index=a.batch_index,
                        recover=int(a.recover), init_fill=cfg.init_fill,
                        psnr=O.psnr(X, L), psnr_zero_fill=O.psnr(X, pm),
                        objective=np.array(rep.objective),
                        primal_residual=np.array(rep.primal_residual),
                        l_change=np.array(rep.l_change),
                        seconds=dt, threads=a.threads, blocked=int(a.blocked))
    print(f"{out}: psnr={O.psnr(X, L):.4f} dB (zero fill {O.psnr(X, pm):.4f} dB), "
          f"{dt:.0f} s, {a.threads} threads", flush=True)


if __name__ == "__main__":
    main()
