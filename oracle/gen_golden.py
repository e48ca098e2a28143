"""Generate golden fixtures for the GPU parity tests (test infrastructure).

The reference ships no golden data (proj/test_output.txt is pass/fail only)
and cannot be built here (Eigen3/FFTW3 absent), so full-size fixtures come
from the pinned fp64 oracle (icnnm_oracle.py, itself checked against the
reference's known-answer tests in tests/test_oracle_pins.py).  Each fixture
stores the basis K it was solved with, so the GPU test feeds identical bits.

  python -m oracle.gen_golden --config 2 [--threads 8] [--dims H W T] [--iters N]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--dims", type=int, nargs=3, default=None)
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--batch-index", type=int, default=0)
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    os.environ["ICNNM_ORACLE_THREADS"] = str(a.threads)
    from threadpoolctl import threadpool_limits
    from oracle import icnnm_oracle as O
    from paper_2604_17001_b200 import synth
    O.WORKERS = a.threads
    w = synth.WORKLOADS[a.config]
    if a.dims:
        w = synth.scaled(w, tuple(a.dims), iters=a.iters or None)
    elif a.iters:
        w = synth.scaled(w, w.dims, iters=a.iters)
    X = w.target(b=a.batch_index)
    mask = w.mask()
    t0 = time.time()
    with threadpool_limits(limits=a.threads):
        B = O.learn_ensemble_basis(w.training(), w.kernel)
        L, rep = O.icnnm_solve(X * mask, mask, B,
                               O.SolverConfig(max_iters=w.iters, tol_primal=1e-300,
                                              tol_change=1e-300))
    dt = time.time() - t0
    tag = f"cfg{a.config}" + (f"_{'x'.join(map(str, w.dims))}" if a.dims else "") + \
          (f"_b{a.batch_index}" if a.batch_index else "") + f"_it{w.iters}"
    out = a.out or os.path.join(ROOT, "tests", "golden", tag + ".npz")
    np.savez_compressed(out, L=L.astype(np.float32), K=B.K, eigenvalues=B.eigenvalues,
                        kernel=np.array(w.kernel), dims=np.array(w.dims), iters=w.iters,
                        config=a.config, batch_index=a.batch_index,
                        psnr=O.psnr(X, L), objective=np.array(rep.objective),
                        seconds=dt, threads=a.threads)
    print(f"{out}: psnr={O.psnr(X, L):.4f} dB, {dt:.0f} s, {a.threads} threads")


if __name__ == "__main__":
    main()
