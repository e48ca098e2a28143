"""Single failing case for debugger runs (k=1183 F16x3 solve, 2 iterations)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_17001_b200 as P
dims, ks, it = (32, 32, 24), (13, 13, 7), int(sys.argv[1]) if len(sys.argv) > 1 else 2
rng = np.random.default_rng(5)
X = rng.uniform(0, 1, size=dims); mask = (rng.uniform(size=dims) < 0.3).astype(float)
B = P.learn_ensemble_basis([rng.uniform(0, 1, size=dims)], ks)
L, r = P.icnnm_solve(X * mask, mask, B, P.SolverConfig(max_iters=it, engine="f16x3", tol_primal=1e-300, tol_change=1e-300))
print("solve ok", r.iterations, r.objective[-1])
