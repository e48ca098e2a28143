"""Small solves/operators for compute-sanitizer (memcheck/racecheck) runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_17001_b200 as P
from paper_2604_17001_b200 import synth

for engine in ("f16x3", "tf32x3", "ffma"):
    X = synth.synth_video(16, 12, 16, 6, 1, 5)
    mask = synth.reference_bernoulli_mask(X.shape, 0.4, 2)
    B = P.learn_ensemble_basis([synth.synth_video(16, 12, 16, 6, 1, 6)], (3, 3, 3))
    L, rep = P.icnnm_solve(X * mask, mask, B, P.SolverConfig(max_iters=5, engine=engine,
                                                             tol_primal=1e-300, tol_change=1e-300))
    L2, rep2 = P.icnnm_solve(X * mask, mask, B, P.SolverConfig(max_iters=3, engine=engine,
                                                               exact_residual=True))
    r0, rows, rep3 = P.sharded_solve(X * mask, mask, B, P.SolverConfig(max_iters=3, engine=engine),
                                     local_slabs=2)
    out = P.BasisConvolver((7, 5, 9), (3, 2, 4), np.eye(24), engine=engine).apply(np.ones((7, 5, 9)))
    adj = P.conv_adjoint(np.ones((315, 24)), (3, 2, 4), (7, 5, 9), engine=engine)
    print(engine, "ok", rep.iterations, rep2.iterations, rep3.iterations, float(out.sum()), float(adj.sum()))
g = P.conv_gram(np.ones((6, 5, 4)), (2, 2, 2))
z = P.prox_l21(np.ones((10, 3)), 0.5)
print("ok")
