"""Time the GPU `analyze` path (recovery diagnostics) on a BASELINE config.

usage: python tools/analyze_timing.py [--config 2]
Prints one JSON line: wall seconds of analyze_recovery and of its parts.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2604_17001_b200 import analysis as A, learn_ensemble_basis, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    w = synth.WORKLOADS[a.config]
    X, mask = w.target(), w.mask()
    b = learn_ensemble_basis(w.training(), w.kernel)
    A.relative_eigenvalues(X, b)  # warm-up (module load, smem attributes)
    t = {}
    t0 = time.perf_counter()
    s = A.relative_eigenvalues(X, b)
    t["relative_eigenvalues_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    alpha = A.spectral_corr_coeff(X, b)
    t["spectral_corr_coeff_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    cc = A.conv_coherence(X, w.kernel)
    t["conv_coherence_s"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    d = A.analyze_recovery(X, b, mask)
    t["analyze_recovery_s"] = time.perf_counter() - t0
    m, k = X.size, b.K.shape[0]
    # one fp64 implicit GEMM pass = 2 m k^2 flops
    print(json.dumps(dict(config=a.config, m=m, k=k, r_K=d.r_K, r0=d.r0, alpha_K=d.alpha_K,
                          mu1=d.mu1, mu2=d.mu2, tau=d.tau, certified=d.certified,
                          sigma_max=float(s.max()), alpha=alpha, cc_rank=cc.rank,
                          conv64_pass_flop=2.0 * m * k * k, **t)))


if __name__ == "__main__":
    main()
