"""Where the end-to-end C-ABI solve spends its time (ICNNM_TIMING phase marks on
stderr) on BASELINE config 2; run twice so the second call is warm."""
import os, sys, time
os.environ.setdefault("ICNNM_TIMING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_17001_b200 as P
from paper_2604_17001_b200 import synth

w = synth.WORKLOADS[2]
X, mask = w.target(), w.mask()
B = P.learn_ensemble_basis(w.training(), w.kernel)
cfg = P.SolverConfig(max_iters=w.iters, tol_primal=1e-300, tol_change=1e-300)
M = np.ascontiguousarray(X * mask)
for rep in range(3):
    t0 = time.perf_counter()
    L, r = P.icnnm_solve(M, mask, B, cfg)
    t = time.perf_counter() - t0
    print(f"call {rep}: {t*1e3:.1f} ms python-wall, report wall {r.wall_time_seconds*1e3:.1f} ms, "
          f"device {r.device_seconds*1e3:.1f} ms", flush=True)
    sys.stderr.flush()
