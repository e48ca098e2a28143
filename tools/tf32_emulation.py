"""Numerics study: does a split-TF32 GEMM hold the 1e-4 / 0.01 dB tolerance?

Emulates the GPU restated iteration in numpy float32 with the
two contractions computed as sum of tf32 products (mantissa rounded to 10
bits, round-to-nearest like cvt.rna.tf32.f32), and compares with the fp64
oracle.  terms: 1 = hi*hi, 2 = hi*hi + lo*hi (B exact split not used),
3 = hi*hi + hi*lo + lo*hi.
"""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import icnnm_oracle as O
from paper_2604_17001_b200 import synth


def tf32(x):
    x = np.asarray(x, dtype=np.float32)
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + 0x1000) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def gemm(A, B, terms):
    if terms == 0:
        return A.astype(np.float32) @ B.astype(np.float32)
    Ah = tf32(A); Bh = tf32(B)
    out = Ah @ Bh
    if terms >= 2:
        Al = tf32(A.astype(np.float32) - Ah)
        out = out + Al @ Bh
    if terms >= 3:
        Bl = tf32(B.astype(np.float32) - Bh)
        out = out + Ah @ Bl
    return out


def im2col(L, ks):
    return np.stack([np.roll(L, s, axis=(0, 1, 2)).ravel() for s in O.kernel_offsets(ks)], axis=1)


def solve(M, mask, K, ks, iters, terms, lam=1000.0):
    k = K.shape[0]
    dims = M.shape
    pm = (M * mask).astype(np.float64)
    L = pm.copy()
    th = [min(1e-2 * np.abs(pm).max() * k, 1e10)]
    for _ in range(iters):
        th.append(min(th[-1] * 1.05, 1e10))
    K32 = K.astype(np.float32)
    W = gemm(im2col(L.astype(np.float32), ks), K32, terms)
    for it in range(iters):
        t = th[it]; r = t / th[it + 1]
        n = np.sqrt((W.astype(np.float64) ** 2).sum(0)); tau = 1 / t
        c = np.where(n > tau, tau / np.where(n > 0, n, 1), 1.0).astype(np.float32)
        U = gemm(W * c[None, :], K32.T, terms)
        adj = O.conv_adjoint(U.astype(np.float64), ks, dims)
        d = (lam * (pm - mask * L) - (t / k) * adj) / (lam * mask + t)
        Ln = L + d
        W = gemm(im2col((Ln + r * d).astype(np.float32), ks), K32, terms) + np.float32(r) * c[None, :] * W
        L = Ln
    return L


if __name__ == "__main__":
    dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (48, 48, 32)
    cfgn = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    w = synth.scaled(synth.WORKLOADS[cfgn], dims, n_train=4)
    iters = int(sys.argv[5]) if len(sys.argv) > 5 else w.iters
    X = w.target(); mask = w.mask()
    B = O.learn_ensemble_basis(w.training(), w.kernel)
    t0 = time.time()
    Lo, _ = O.icnnm_solve(X * mask, mask, B, O.SolverConfig(max_iters=iters, tol_primal=1e-300, tol_change=1e-300))
    print(f"dims={dims} k={w.k} iters={iters} oracle psnr={O.psnr(X, Lo):.4f} ({time.time()-t0:.0f}s)", flush=True)
    for terms in (0, 1, 2, 3):
        t0 = time.time()
        L = solve(X * mask, mask, B.K, w.kernel, iters, terms)
        print(f"terms={terms}: rel={O.rel_l2(L, Lo):.3e} dPSNR={abs(O.psnr(X, L) - O.psnr(X, Lo)):.2e} ({time.time()-t0:.0f}s)", flush=True)
