"""CPU ORACLE, blocked / out-of-core -- test infrastructure only (never the
product path).

The same literal fp64 restatement of the reference ADMM loop as
``icnnm_oracle.AdmmSolver`` (/root/reference/proj/core/src/solver.cpp:62-146,
operators conv_op.cpp:57-114), for problems whose m x k matrices do not fit
in host RAM (BASELINE config 3: m = 3,145,728, k = 1183 -> 29.8 GB per fp64
m x k matrix; the reference itself keeps ~12 of them).  Only
Y and Z are stored (in RAM or in memory-mapped files); every other m x k
quantity of the loop is produced and consumed in blocks:

* column chunks (the FFT side): A(L)K columns j0..j1 come from the k kernel
  spectra exactly as BasisConvolver::apply computes them (1 forward FFT of L,
  per-column inverse FFTs, conv_op.cpp:100-114); the prox (solver.cpp:42-50),
  the gap / residual / multiplier update (:123-126) and the objective's
  column norms (:128-129) are column-separable;
* H-slab row blocks (the GEMM + adjoint side): WK = (Y + theta Z) K^T
  (:110) is row-separable, and conv_adjoint (conv_op.cpp:57-77) adds each
  row block's contributions out[i] += WK[i + s, s] into the m-vector.

The two passes are the literal loop's order of operations; the only
difference from the in-core oracle is the order in which fp64 sums are
accumulated (adjoint: slab by slab; GEMM: the same dot products), i.e.
rounding at the 1e-16 level (checked against the in-core oracle in
tests/test_oracle_pins.py::test_blocked_oracle_matches_in_core).
"""
from __future__ import annotations

import os
import time
from typing import Optional

import numpy as np
import scipy.fft as sfft

from . import icnnm_oracle as O


class BlockedAdmm:
    """admm_solve (solver.cpp:62-146) with Y, Z stored as (k, m) arrays in RAM
    or in memory-mapped files under `store_dir`."""

    def __init__(self, M_obs: np.ndarray, mask: np.ndarray, basis: O.EigenBasis,
                 cfg: Optional[O.SolverConfig] = None, store_dir: Optional[str] = None,
                 chunk: int = 16, slab_rows: int = 8, workers: int = 1,
                 validate_basis: bool = True, log=None, spectra_budget: float = 16e9):
        cfg = cfg or O.SolverConfig()
        if validate_basis:
            basis.validate()                                      # solver.cpp:156
        cfg.validate()                                            # :66
        ks = tuple(int(x) for x in basis.kernel_shape)
        O.validate_kernel(ks, M_obs.shape)                        # :67
        if mask.shape != M_obs.shape:                             # :68-69
            raise ValueError("solve: mask dims != observation dims")
        if np.any((mask != 0.0) & (mask != 1.0)):                 # tensor.hpp:115-121
            raise ValueError("SamplingMask: entries must be 0 or 1")
        if int(mask.sum() + 0.5) == 0:                            # :70-71
            raise ValueError("solve: empty sampling set")
        if not np.all(np.isfinite(M_obs)):                        # :72
            raise ValueError("solve: observations: non-finite tensor entries")
        self.t_start = time.perf_counter()
        self.cfg, self.ks, self.K = cfg, ks, np.asarray(basis.K, dtype=np.float64)
        self.dims = tuple(int(d) for d in M_obs.shape)
        self.M_obs, self.mask = M_obs, mask
        self.k = k = int(np.prod(ks))
        self.m = m = int(np.prod(self.dims))
        self.chunk, self.slab_rows, self.workers = chunk, slab_rows, workers
        self.log = log or (lambda *a: None)
        self.pm = pm = M_obs * mask                               # :80
        L = pm.copy()                                             # :82
        if cfg.init_fill == "mean":                               # :83-86
            L = L + (1.0 - mask) * (pm.sum() / float(int(mask.sum() + 0.5)))
        self.L = L
        theta = cfg.theta0 if cfg.theta0 is not None else 1e-2 * np.max(np.abs(pm)) * k  # :88-89
        if theta <= 0:
            theta = 1e-2                                          # :90
        self.theta = min(theta, cfg.theta_max)                    # :91
        rs = np.sqrt(k) * np.linalg.norm(pm)                      # :97
        self.res_scale = rs if rs != 0 else 1.0                   # :98
        if store_dir:
            os.makedirs(store_dir, exist_ok=True)
            self.Y = np.lib.format.open_memmap(os.path.join(store_dir, "Y.npy"), mode="w+",
                                               dtype=np.float64, shape=(k, m))
            self.Z = np.lib.format.open_memmap(os.path.join(store_dir, "Z.npy"), mode="w+",
                                               dtype=np.float64, shape=(k, m))
        else:
            self.Y = np.zeros((k, m))                             # :102
            self.Z = np.empty((k, m))
        # kernel spectra (conv_op.cpp:92-97) kept when they fit the budget,
        # otherwise recomputed per column chunk (same bits either way)
        self._spec = self._spectra(0, k) if 16.0 * m * k <= spectra_budget else None
        self.report = O.SolveReport()
        self.report.termination = "max_iters"
        self.it = 0
        # AKL_0 = A(L_0) K (:100); Y_0 = 0 (:102); the first Z-update (:108)
        # happens in the same column pass
        self.Y[:] = 0.0
        self._zl21 = self._column_pass(first=True)

    # --- A(L) K, column chunk [j0, j1): BasisConvolver::apply (conv_op.cpp:100-114)
    def _spectra(self, j0: int, j1: int) -> np.ndarray:
        kern = self.K[:, j0:j1].T.reshape((j1 - j0,) + self.ks)
        padded = np.zeros((j1 - j0,) + self.dims)
        padded[(slice(None),) + tuple(slice(0, q) for q in self.ks)] = kern
        return sfft.fftn(padded, axes=tuple(range(1, len(self.dims) + 1)), workers=self.workers)

    def _akl_chunk(self, fl: np.ndarray, j0: int, j1: int) -> np.ndarray:
        axes = tuple(range(1, len(self.dims) + 1))
        spec = self._spec[j0:j1] if self._spec is not None else self._spectra(j0, j1)
        out = sfft.ifftn(fl[None] * spec, axes=axes, workers=self.workers).real
        return out.reshape(j1 - j0, -1)

    def _column_pass(self, first: bool) -> float:
        """Column chunks of AKL_t = A(L_t) K.  Unless `first`: the end of the
        previous iteration -- gap = Z - AKL (:123), ||gap|| (:124),
        Y += theta_prev gap (:125) -- then, for every call, the Z-update of
        the next iteration's :108 with the current theta.  Returns
        sum_j ||Z_j|| of the Z it produced (the objective's :128-129 term
        for that iteration)."""
        fl = sfft.fftn(self.L, workers=self.workers)
        th_prev, th = getattr(self, "_theta_prev", None), self.theta
        gap2 = 0.0
        zl21 = 0.0
        for j0 in range(0, self.k, self.chunk):
            j1 = min(self.k, j0 + self.chunk)
            akl = self._akl_chunk(fl, j0, j1)
            Y = np.array(self.Y[j0:j1])
            if not first:
                gap = np.array(self.Z[j0:j1]) - akl               # :123
                gap2 += float(np.einsum("ij,ij->", gap, gap))
                Y += th_prev * gap                                # :125
                self.Y[j0:j1] = Y
            W = akl - Y / th                                      # :108
            n = np.sqrt(np.einsum("ij,ij->i", W, W))
            scale = np.where(n > 1.0 / th, 1.0 - (1.0 / th) / np.where(n > 0, n, 1.0), 0.0)  # :42-50
            Z = W * scale[:, None]
            self.Z[j0:j1] = Z
            zl21 += float(np.sum(np.sqrt(np.einsum("ij,ij->i", Z, Z))))
        self._gap2 = gap2
        return zl21

    def _row_pass(self) -> np.ndarray:
        """adj = conv_adjoint((Y + theta Z) K^T) (:110-111), H-slab by H-slab."""
        dims = self.dims
        H = dims[0]
        rest = int(np.prod(dims[1:])) if len(dims) > 1 else 1
        offs = O.kernel_offsets(self.ks)
        adj = np.zeros(dims)
        th = self.theta
        for h0 in range(0, H, self.slab_rows):
            h1 = min(H, h0 + self.slab_rows)
            sl = slice(h0 * rest, h1 * rest)
            P = np.array(self.Y[:, sl]) + th * np.array(self.Z[:, sl])
            WKt = self.K @ P                                      # :110 (transposed)
            WKt = WKt.reshape((self.k, h1 - h0) + tuple(dims[1:]))
            for col, s in enumerate(offs):
                # out[i] += WK[(i + s) mod dims, s]  (conv_op.cpp:57-77): row h of
                # the slab lands on output row h - s_h
                c = WKt[col]
                if len(dims) > 1:
                    c = np.roll(c, shift=tuple(-int(x) for x in s[1:]),
                                axis=tuple(range(1, len(dims))))
                rows = (np.arange(h0, h1) - int(s[0])) % H
                adj[rows] += c
        return adj

    def step(self) -> bool:
        cfg, k, theta = self.cfg, self.k, self.theta
        zl21 = self._zl21                                         # ||Z_j|| of this iteration's :108
        adj = self._row_pass()                                    # :110-111
        numer = adj / k + cfg.lambda_ * self.pm                   # :112-113
        denom = cfg.lambda_ * self.mask + theta                   # :114-115
        L_new = numer / denom                                     # :116
        l_change = np.linalg.norm(L_new - self.L) / max(np.linalg.norm(self.L), 1e-300)  # :118-119
        self.L = L_new                                            # :120
        self._theta_prev = theta
        self.theta = min(theta * cfg.theta_growth, cfg.theta_max)  # :126
        # :121-125 (AKL = A(L) K, gap, residual, Y update) fused with the next
        # iteration's Z-update in one column pass
        self._zl21 = self._column_pass(first=False)
        residual = np.sqrt(self._gap2) / self.res_scale           # :124
        fit = float(np.sum(((self.L - self.M_obs) * self.mask) ** 2))  # :130
        rep = self.report
        rep.objective.append(zl21 + 0.5 * cfg.lambda_ * k * fit)  # :131-132
        rep.primal_residual.append(residual)
        rep.l_change.append(l_change)
        self.it += 1
        rep.iterations = self.it
        self.log(f"iteration {self.it}: objective {rep.objective[-1]:.10g} "
                 f"residual {residual:.4g} l_change {l_change:.4g}")
        if residual < cfg.tol_primal or l_change < cfg.tol_change:  # :136-139
            rep.termination = "converged"
            return True
        return False


def icnnm_solve_blocked(M_obs, mask, basis, cfg=None, **kw):
    """icnnm_solve (solver.cpp:150-159) through the blocked loop."""
    s = BlockedAdmm(M_obs, mask, basis, cfg, **kw)
    for _ in range(s.cfg.max_iters):
        if s.step():
            break
    s.report.wall_time_seconds = time.perf_counter() - s.t_start
    return s.L, s.report
