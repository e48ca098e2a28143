"""Per-kernel times (CUDA events on the solver stream) of one config-C solve.
With tools/with_ab_lib.py in front it runs the experiments build, whose A/B
knobs are read from the environment:
  ICNNM_TC_BMIX=0 python tools/with_ab_lib.py tools/ab_kernels.py --config 4
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17001_b200 as P
import synthgen as synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--engine", default="f16x3")
ap.add_argument("--iters", type=int, default=60)
ap.add_argument("--tag", default="")
a = ap.parse_args()
w = synth.WORKLOADS[a.config]
X, mask = w.target(), w.mask()
B = P.learn_ensemble_basis(w.training(), w.kernel)
S = P.Solver(X.shape, B)
S.upload(X * mask, mask)
cfg = P.SolverConfig(max_iters=a.iters, tol_primal=1e-300, tol_change=1e-300, engine=a.engine)
S.run(cfg)
r = S.run(cfg)
S.set_profile(True)
S.run(cfg)
kt = S.kernel_times_ms()
L = S.download()
print(json.dumps({"tag": a.tag, "config": a.config, "loop_ms_per_iter": r.loop_seconds * 1e3 / a.iters,
                  "kernels_ms": {k: round(v, 4) for k, v in kt.items()},
                  "psnr": synth.psnr(X, L), "knobs": {k: v for k, v in os.environ.items() if k.startswith("ICNNM_")}}))
