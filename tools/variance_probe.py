"""Per-solve device time with and without a concurrent nvidia-smi sampler."""
import os, sys, subprocess, threading, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17001_b200 as P
from paper_2604_17001_b200 import synth
w = synth.WORKLOADS[2]
X, mask = w.target(), w.mask()
B = P.learn_ensemble_basis(w.training(), w.kernel)
S = P.Solver(X.shape, B)
S.upload(X * mask, mask)
cfg = P.SolverConfig(max_iters=300, tol_primal=1e-300, tol_change=1e-300)
def run(n):
    return [round(S.run(cfg).device_seconds, 4) for _ in range(n)]
print("warm", run(3), flush=True)
print("no sampler", run(6), flush=True)
stop = threading.Event(); clocks = []
def sampler(period):
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        clocks.append(out); stop.wait(period)
for period in (0.2, 1.0):
    stop.clear(); clocks.clear()
    t = threading.Thread(target=sampler, args=(period,), daemon=True); t.start()
    r = run(6); stop.set(); t.join()
    print(f"sampler {period}s", r, clocks[:12], flush=True)
print("no sampler again", run(6), flush=True)
