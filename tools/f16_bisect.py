"""Bisect the F16x3 solve failure at k=1183 (see tools/f16_debug.py)."""
import os, subprocess, sys
CASE = r'''
import sys, numpy as np
sys.path.insert(0, %r)
import paper_2604_17001_b200 as P
dims, ks, it = (32, 32, 24), (13, 13, 7), %d
rng = np.random.default_rng(5)
X = rng.uniform(0, 1, size=dims); mask = (rng.uniform(size=dims) < 0.3).astype(float)
B = P.learn_ensemble_basis([rng.uniform(0, 1, size=dims)], ks)
L, r = P.icnnm_solve(X * mask, mask, B, P.SolverConfig(max_iters=it, engine="f16x3", tol_primal=1e-300, tol_change=1e-300))
print("solve ok", r.iterations, r.objective[-1])
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for env in [{}, {"ICNNM_F16_OFF": "1"}, {"ICNNM_F16_OFF": "2"}, {"ICNNM_TC_SB": "4"},
            {"ICNNM_TC_SB": "3"}, {"CUDA_LAUNCH_BLOCKING": "1"}]:
    for it in (1, 2, 3, 8):
        for rep in range(2):
            try:
                p = subprocess.run([sys.executable, "-c", CASE % (root, it)], capture_output=True,
                                   text=True, timeout=60, env=dict(os.environ, **env))
                out = p.stdout.strip() + (" ERR " + p.stderr.strip().splitlines()[-1] if p.returncode else "")
            except subprocess.TimeoutExpired:
                out = "HANG"
            print(env, it, rep, "->", out, flush=True)
