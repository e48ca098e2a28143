"""Input builders of the reference's analysis tests, shared by the oracle pins
(test_analysis_pins.py) and the GPU parity tests (test_gpu_analysis.py).

Restates /root/reference/proj/tests/test_util.hpp:81-89 (random_orthogonal),
test_analysis.cpp:31-39 (basis_from_matrix) and test_acceptance.cpp:56-83
(cosine_1d / cosine_2d / one_missing_mask).
"""
import numpy as np

from oracle import icnnm_oracle as O
from paper_2604_17001_b200 import synth


def Rng(seed):
    return synth.Rng(seed)


def random_orthogonal(n, rng):
    """Q of a Householder QR of an n x n standard-normal matrix filled row by
    row (LAPACK and Eigen share the Householder sign convention)."""
    M = rng.normal(0.0, 1.0, n * n).reshape(n, n)
    Q, _ = np.linalg.qr(M)
    return Q


def basis_from_matrix(ks, K):
    ks = tuple(ks)
    return O.EigenBasis(ks, np.asarray(K, dtype=np.float64), np.zeros(int(np.prod(ks))))


def cosine_1d(m, period):
    return np.cos(2.0 * np.pi * np.arange(m) / period)


def cosine_2d(n, period):
    c = np.cos(2.0 * np.pi * np.arange(n) / period)
    return np.outer(c, c)


def one_missing_mask(dims, missing_flat):
    t = np.ones(dims)
    t.reshape(-1)[missing_flat] = 0.0
    return t
