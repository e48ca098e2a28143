"""In-kernel pipeline counters of the tcgen05 kernels (set_profile tc_counters):
per-role wait / work cycles as fractions of the MMA thread's cycles.

  python tools/with_ab_lib.py tools/tc_counters.py --config 4 [--iters 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17001_b200 as P  # noqa: E402
import synthgen as synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--engine", default="f16x3")
a = ap.parse_args()
w = synth.WORKLOADS[a.config]
X, mask = w.target(), w.mask()
B = P.learn_ensemble_basis(w.training(), w.kernel)
S = P.Solver(X.shape, B)
S.upload(X * mask, mask)
cfg = P.SolverConfig(max_iters=a.iters, tol_primal=1e-300, tol_change=1e-300, engine=a.engine)
S.run(cfg)
S.set_profile(True)
S.run(cfg)
kt = S.kernel_times_ms()
S.set_profile(False, tc_counters=True)
S.run(cfg)
c = S.tc_counters()
nb = X.size // 128
print(f"config {a.config} k={w.k}: kernel ms {kt}")
for kind, d in c.items():
    tot = max(d["mma_total"], 1)
    frac = {n: round(v / tot, 3) for n, v in d.items()}
    print(kind, "MMA-thread cycles/CTA/launch %.0f" % (tot / 148 / (a.iters + 1)), frac,
          "(builder / epilogue: sums over lane 0 of the role's warps)")
