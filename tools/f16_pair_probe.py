"""First-contact check of the F16x3 CTA-pair (cta_group::2) kernels at operator level."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_17001_b200 as P
from oracle import icnnm_oracle as O


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


for dims, ks in [((16, 16, 16), (3, 3, 3)), ((32, 32, 8), (5, 5, 3)), ((16, 16, 32), (9, 9, 5)),
                 ((7, 5, 9), (3, 2, 4)), ((12, 11, 10), (4, 4, 8))]:
    k = int(np.prod(ks))
    L = np.random.default_rng(1).integers(-8, 9, size=dims).astype(np.float64)
    out = P.BasisConvolver(dims, ks, np.eye(k), engine="f16x3").apply(L)
    ref = O.conv_matrix(L, ks)
    print(dims, ks, "fwd K=I exact:", np.array_equal(out, ref), "maxdiff", np.abs(out - ref).max(), flush=True)
    m = L.size
    W = np.random.default_rng(4).integers(-4, 5, size=(m, k)).astype(np.float64)
    a1 = P.conv_adjoint(W, ks, dims, engine="f16x3")
    a0 = O.conv_adjoint(W, ks, dims)
    print("   adj int exact:", np.array_equal(a1, a0), "maxdiff", np.abs(a1 - a0).max(), flush=True)
    Lr = np.random.default_rng(2).uniform(-1, 1, size=dims)
    K = np.linalg.qr(np.random.default_rng(3).standard_normal((k, k)))[0]
    g1 = P.BasisConvolver(dims, ks, K, engine="f16x3").apply(Lr)
    r = O.BasisConvolver(dims, ks, K).apply(Lr)
    print("   fwd random K rel", rel(g1, r), flush=True)
