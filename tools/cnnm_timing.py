"""ICNNM vs the CNNM baseline on the GPU at a BASELINE config (the paper's
runtime-ordering claim, test_acceptance.cpp:288-300, at full scale).

usage: python tools/cnnm_timing.py [--config 2] [--iters 40]
Prints one JSON line with both solvers' loop time and PSNR.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2604_17001_b200 as P  # noqa: E402
from paper_2604_17001_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--iters", type=int, default=40)
    a = ap.parse_args()
    w = synth.WORKLOADS[a.config]
    X, mask = w.target(), w.mask()
    B = P.learn_ensemble_basis(w.training(), w.kernel)
    cfg = P.SolverConfig(max_iters=a.iters, tol_primal=1e-300, tol_change=1e-300)
    P.icnnm_solve(X * mask, mask, B, P.SolverConfig(max_iters=2))
    P.cnnm_solve(X * mask, mask, w.kernel, P.SolverConfig(max_iters=2))
    Li, ri = P.icnnm_solve(X * mask, mask, B, cfg)
    Lc, rc = P.cnnm_solve(X * mask, mask, w.kernel, cfg)
    print(json.dumps(dict(config=a.config, iters=a.iters, m=int(X.size), k=int(B.K.shape[0]),
                          icnnm_loop_s=ri.loop_seconds, cnnm_loop_s=rc.loop_seconds,
                          icnnm_wall_s=ri.wall_time_seconds, cnnm_wall_s=rc.wall_time_seconds,
                          cnnm_ms_per_iter=1e3 * rc.loop_seconds / a.iters,
                          icnnm_ms_per_iter=1e3 * ri.loop_seconds / a.iters,
                          psnr_icnnm=synth.psnr(X, Li), psnr_cnnm=synth.psnr(X, Lc))))


if __name__ == "__main__":
    main()
