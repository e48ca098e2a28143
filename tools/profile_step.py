"""Small driver for ncu: one config-C solve with a few iterations."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17001_b200 as P
import synthgen as synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--engine", default="f16x3")
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--runs", type=int, default=1)
a = ap.parse_args()
w = synth.WORKLOADS[a.config]
X, mask = w.target(), w.mask()
B = P.learn_ensemble_basis(w.training(), w.kernel)
S = P.Solver(X.shape, B)
S.upload(X * mask, mask)
cfg = P.SolverConfig(max_iters=a.iters, tol_primal=1e-300, tol_change=1e-300, engine=a.engine)
for _ in range(a.runs):
    r = S.run(cfg)
print(f"config {a.config} engine {a.engine}: {a.iters} iters in {r.loop_seconds*1e3:.2f} ms (loop)")
if os.environ.get("ICNNM_TC_COUNTERS"):
    S.set_profile(False, tc_counters=True)
    r = S.run(cfg)
    import json
    c = S.tc_counters()
    nsm = 148
    nb = (X.size // 128)
    ntn = (w.k + 31) // 32 * 32
    import math
    nt_tiles = math.ceil(ntn / 128); nkc = ntn // 32
    mmas = nb * nt_tiles * nkc * 12
    for k, d in c.items():
        tot = max(d["mma_total"], 1)
        print(k, "MMA-thread cycles per CTA per launch: %.0f" % (tot / nsm / a.iters),
              "cycles per MMA issued: %.1f" % (tot / (mmas * a.iters)),
              "kernel time per launch (ms):", S.kernel_times_ms() if False else "")
        print(k, {n: round(v / tot, 3) for n, v in d.items()}, "(fractions of MMA-thread cycles; builder/epi: sums over the role's warps (lane 0))")
        bt = max(d["build_total"], 1)
        print(k, "builder warp time split: chunk waits %.3f, chunk work %.3f, per-brick prep %.3f, other %.3f"
              % (d["build_wait"] / bt, d["build_work"] / bt, d["build_prep"] / bt,
                 1 - (d["build_wait"] + d["build_work"] + d["build_prep"]) / bt))
