"""Gram-accumulation kernel (north-star (e)) timing driver: conv_gram of one
training tensor of config C, and the measured DFMA peak.  Run under
`ncu --metrics gpu__time_duration.sum` for the kernel's own duration; the
roofline is flops = 2 m kh (2kw-1)(2kt-1) (half lag space, mirrored) over the
DFMA probe.

  python tools/gram_profile.py --config 2
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17001_b200 as P  # noqa: E402
import synthgen as synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
a = ap.parse_args()
w = synth.WORKLOADS[a.config]
X = w.training()[0]
kh, kw, kt = w.kernel
peak = P.probe_dfma_tflops(0)
P.conv_gram(X, w.kernel)
t0 = time.perf_counter()
P.conv_gram(X, w.kernel)
dt = time.perf_counter() - t0
flops_half = 2.0 * X.size * kh * (2 * kw - 1) * (2 * kt - 1)
flops_full = 2.0 * X.size * (2 * kh - 1) * (2 * kw - 1) * (2 * kt - 1)
print(f"config {a.config}: dims {X.shape} kernel {w.kernel} DFMA peak {peak:.2f} TFLOP/s; "
      f"conv_gram call (H2D + kernels + D2H + host Gram fill) {dt * 1e3:.2f} ms; "
      f"flops computed {flops_half:.3e} (full lag box {flops_full:.3e})")
