"""CPU ORACLE — test infrastructure only (never the product path).

A literal fp64 numpy/scipy restatement of the reference ICNNM solver path,
/root/reference/proj/core (Eigen3 + FFTW3, neither present in this image, so
the reference itself cannot be compiled here: see DESIGN.md §4).  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this module, and only as the checker / CPU baseline.

Each function cites the reference file:line it restates.  Parity pinning:
the reference ships no golden data files (proj/test_output.txt is pass/fail
only), so this oracle is pinned against every known-answer test of the
reference's own suites for this path (tests/test_oracle_pins.py), with the
reference tests' inputs rebuilt bit-for-bit from libstdc++'s mt19937_64
streams (proj/tests/test_util.hpp:27-49, proj/core/src/mask.cpp:49-59).

Conventions (tensor.hpp:64-68, fft.cpp:78-90, conv_op.cpp:42-44,94):
row-major tensors, kernel taps corner-anchored and flattened row-major,
periodic boundaries, K column j = eigen-kernel j.  Internally the m x k
operator matrices are stored transposed, as (k, *dims) arrays (column j of
the reference's matrix is row j here), so per-column FFTs are contiguous.
"""
from __future__ import annotations

import dataclasses
import itertools
import os
import time
from typing import List, Optional, Sequence, Tuple

import numpy as np
import scipy.fft as sfft

WORKERS = int(os.environ.get("ICNNM_ORACLE_THREADS", "1"))


def kernel_offsets(ks: Sequence[int]) -> List[Tuple[int, ...]]:
    """Row-major multi-indices of the kernel box (for_each_index,
    tensor.hpp:140-152)."""
    return list(itertools.product(*[range(int(k)) for k in ks]))


def validate_kernel(ks, dims) -> None:
    """KernelShape::validate_for (tensor.hpp:100-107)."""
    if len(ks) != len(dims):
        raise ValueError("KernelShape: order mismatch with tensor")
    for k, d in zip(ks, dims):
        if k < 1 or k > d:
            raise ValueError("KernelShape: kernel dim out of range")


def circular_shift(L: np.ndarray, s) -> np.ndarray:
    """circular_shift (conv_op.cpp:19-33): out[i] = L[(i - s) mod dims]."""
    return np.roll(L, shift=tuple(int(x) for x in s), axis=tuple(range(L.ndim)))


def conv_matrix(L: np.ndarray, ks) -> np.ndarray:
    """conv_matrix (conv_op.cpp:35-46): m x k, column s = vec(shift(L, s))."""
    validate_kernel(ks, L.shape)
    return np.stack([circular_shift(L, s).ravel() for s in kernel_offsets(ks)], axis=1)


def pad_to(X: np.ndarray, dims) -> np.ndarray:
    """pad_to (fft.cpp:78-90): corner-anchored zero padding."""
    out = np.zeros(tuple(dims))
    out[tuple(slice(0, k) for k in X.shape)] = X
    return out


def circular_convolve(L: np.ndarray, X: np.ndarray) -> np.ndarray:
    """circular_convolve (fft.cpp:92-107): (L*X)[i] = sum_s L[i-s] X[s]."""
    if X.ndim != L.ndim:
        raise ValueError("pad_to: order mismatch")
    if any(k > d for k, d in zip(X.shape, L.shape)):
        raise ValueError("pad_to: kernel dim exceeds tensor dim")
    fl = sfft.fftn(L, workers=WORKERS)
    fx = sfft.fftn(pad_to(X, L.shape), workers=WORKERS)
    return sfft.ifftn(fl * fx, workers=WORKERS).real


def circular_autocorrelation(L: np.ndarray) -> np.ndarray:
    """circular_autocorrelation (fft.cpp:109-118)."""
    fl = sfft.fftn(L, workers=WORKERS)
    return sfft.ifftn((fl * fl.conj()).real, workers=WORKERS).real


class BasisConvolver:
    """BasisConvolver (conv_op.cpp:85-114): k kernel spectra precomputed;
    apply(L) = A_k(L) K via 1 forward + k inverse c2c FFTs.  Returned
    transposed: (k, *dims)."""

    def __init__(self, dims, ks, K: np.ndarray, chunk: int = 64):
        validate_kernel(ks, dims)
        self.dims = tuple(int(d) for d in dims)
        self.ks = tuple(int(k) for k in ks)
        k = int(np.prod(self.ks))
        if K.shape != (k, k):
            raise ValueError("BasisConvolver: K must be k x k")
        self.K = np.asarray(K, dtype=np.float64)
        self.k = k
        self.chunk = chunk
        # kernel spectra (conv_op.cpp:92-97); computed lazily per chunk to
        # avoid the m x k complex cache of the reference when large.
        self._spec = None
        if int(np.prod(self.dims)) * k * 16 <= (8 << 30):
            self._spec = self._spectra(0, k)

    def _spectra(self, j0: int, j1: int) -> np.ndarray:
        kern = self.K[:, j0:j1].T.reshape((j1 - j0,) + self.ks)
        padded = np.zeros((j1 - j0,) + self.dims)
        padded[(slice(None),) + tuple(slice(0, q) for q in self.ks)] = kern
        return sfft.fftn(padded, axes=tuple(range(1, len(self.dims) + 1)), workers=WORKERS)

    def apply_t(self, L: np.ndarray) -> np.ndarray:
        if L.shape != self.dims:
            raise ValueError("BasisConvolver: tensor dims mismatch")
        fl = sfft.fftn(L, workers=WORKERS)
        out = np.empty((self.k,) + self.dims)
        axes = tuple(range(1, len(self.dims) + 1))
        for j0 in range(0, self.k, self.chunk):
            j1 = min(self.k, j0 + self.chunk)
            spec = self._spec[j0:j1] if self._spec is not None else self._spectra(j0, j1)
            out[j0:j1] = sfft.ifftn(fl[None] * spec, axes=axes, workers=WORKERS).real
        return out

    def apply(self, L: np.ndarray) -> np.ndarray:
        """m x k, as the reference returns it."""
        return self.apply_t(L).reshape(self.k, -1).T


def conv_adjoint_t(Wt: np.ndarray, ks, dims) -> np.ndarray:
    """conv_adjoint (conv_op.cpp:57-77) on a (k, *dims) array:
    out[i] = sum_s W[(i + s) mod dims, s], s-major then i row-major."""
    dims = tuple(int(d) for d in dims)
    validate_kernel(ks, dims)
    k = int(np.prod(ks))
    if Wt.shape[0] != k or Wt[0].size != int(np.prod(dims)):
        raise ValueError("conv_adjoint: W shape mismatch with dims/kernel")
    out = np.zeros(dims)
    axes = tuple(range(len(dims)))
    for col, s in enumerate(kernel_offsets(ks)):
        out += np.roll(Wt[col].reshape(dims), shift=tuple(-int(x) for x in s), axis=axes)
    return out


def conv_adjoint(W: np.ndarray, ks, dims) -> np.ndarray:
    """conv_adjoint on an m x k matrix."""
    m = int(np.prod(dims))
    k = int(np.prod(ks))
    if W.shape != (m, k):
        raise ValueError("conv_adjoint: W shape mismatch with dims/kernel")
    return conv_adjoint_t(np.ascontiguousarray(W.T), ks, dims)


def prox_l21(W: np.ndarray, tau: float) -> np.ndarray:
    """prox_l21 (solver.cpp:42-50): columns scaled by (n > tau) ? 1 - tau/n : 0."""
    if tau < 0:
        raise ValueError("prox_l21: tau must be >= 0")
    n = np.linalg.norm(W, axis=0)
    scale = np.where(n > tau, 1.0 - tau / np.where(n > 0, n, 1.0), 0.0)
    return W * scale[None, :]


def _prox_l21_t(Wt: np.ndarray, tau: float) -> Tuple[np.ndarray, np.ndarray]:
    k = Wt.shape[0]
    n = np.sqrt(np.einsum("ij,ij->i", Wt.reshape(k, -1), Wt.reshape(k, -1)))
    scale = np.where(n > tau, 1.0 - tau / np.where(n > 0, n, 1.0), 0.0)
    return Wt * scale.reshape((k,) + (1,) * (Wt.ndim - 1)), n


def conv_gram(L: np.ndarray, ks) -> np.ndarray:
    """conv_gram (spectral.cpp:54-81): G[s,t] = R[(s - t) mod dims]."""
    validate_kernel(ks, L.shape)
    R = circular_autocorrelation(L)
    offs = np.array(kernel_offsets(ks), dtype=np.int64)
    dims = np.array(L.shape, dtype=np.int64)
    diff = np.mod(offs[:, None, :] - offs[None, :, :], dims)
    return R[tuple(diff[..., j] for j in range(L.ndim))]


def fix_column_signs(M: np.ndarray) -> np.ndarray:
    """fix_column_signs (spectral.cpp:43-52)."""
    M = M.copy()
    for c in range(M.shape[1]):
        nz = np.nonzero(np.abs(M[:, c]) > 1e-12)[0]
        if nz.size and M[nz[0], c] < 0:
            M[:, c] = -M[:, c]
    return M


def psd_eig_sorted(G: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """psd_eig_sorted (spectral.cpp:87-98): descending, clamped, signs fixed."""
    w, V = np.linalg.eigh(G)
    w = np.maximum(0.0, w[::-1])
    V = fix_column_signs(V[:, ::-1])
    return w, V


@dataclasses.dataclass
class EigenBasis:
    kernel_shape: Tuple[int, ...]
    K: np.ndarray
    eigenvalues: np.ndarray
    degenerate: bool = False

    def validate(self) -> None:
        """EigenBasis::validate (spectral.cpp:25-41)."""
        k = int(np.prod(self.kernel_shape))
        if self.K.shape != (k, k):
            raise ValueError("EigenBasis: K must be k x k")
        if len(self.eigenvalues) != k:
            raise ValueError("EigenBasis: eigenvalue count mismatch")
        if np.max(np.abs(self.K.T @ self.K - np.eye(k))) > 1e-10:
            raise ValueError("EigenBasis: K is not orthogonal")
        ev = np.asarray(self.eigenvalues)
        if np.any(ev < 0):
            raise ValueError("EigenBasis: negative eigenvalue")
        if np.any(ev[1:] > ev[:-1] + 1e-12):
            raise ValueError("EigenBasis: eigenvalues not nonincreasing")


def learn_ensemble_basis(refs: Sequence[np.ndarray], ks) -> EigenBasis:
    """learn_ensemble_basis (spectral.cpp:133-161)."""
    if len(refs) == 0:
        raise ValueError("learn_ensemble_basis: empty reference list")
    dims = refs[0].shape
    validate_kernel(ks, dims)
    k = int(np.prod(ks))
    G = np.zeros((k, k))
    for r in refs:
        if r.shape != dims:
            raise ValueError("learn_ensemble_basis: dim mismatch among refs")
        G += conv_gram(r, ks)
    if np.max(np.abs(G)) == 0.0:
        return EigenBasis(tuple(ks), np.eye(k), np.zeros(k), True)
    w, V = psd_eig_sorted(G)
    return EigenBasis(tuple(ks), V, np.sqrt(w), False)


@dataclasses.dataclass
class SolverConfig:
    """SolverConfig (solver.hpp:29-43)."""
    lambda_: float = 1000.0
    theta0: Optional[float] = None
    theta_growth: float = 1.05
    theta_max: float = 1e10
    max_iters: int = 1000
    tol_primal: float = 1e-7
    tol_change: float = 1e-8
    rank_tol: float = 1e-8
    init_fill: str = "zero"

    def validate(self) -> None:
        """SolverConfig::validate (solver.cpp:26-40)."""
        if not self.lambda_ > 0:
            raise ValueError("SolverConfig: lambda must be > 0")
        if self.theta0 is not None and not self.theta0 > 0:
            raise ValueError("SolverConfig: theta0 must be > 0")
        if not self.theta_growth >= 1:
            raise ValueError("SolverConfig: theta_growth must be >= 1")
        if not self.theta_max > 0:
            raise ValueError("SolverConfig: theta_max must be > 0")
        if self.theta0 is not None and self.theta0 > self.theta_max:
            raise ValueError("SolverConfig: theta0 must be <= theta_max")
        if self.max_iters < 1:
            raise ValueError("SolverConfig: max_iters must be >= 1")
        if not (self.tol_primal > 0 and self.tol_change > 0 and self.rank_tol > 0):
            raise ValueError("SolverConfig: tolerances must be > 0")
        if self.init_fill not in ("zero", "mean"):
            raise ValueError("SolverConfig: init_fill must be 'zero' or 'mean'")


@dataclasses.dataclass
class SolveReport:
    iterations: int = 0
    objective: List[float] = dataclasses.field(default_factory=list)
    primal_residual: List[float] = dataclasses.field(default_factory=list)
    termination: str = "max_iters"
    wall_time_seconds: float = 0.0
    l_change: List[float] = dataclasses.field(default_factory=list)


class AdmmSolver:
    """admm_solve (solver.cpp:62-146) with the prox_l21 Z-update (or, for
    cnnm_solve, svt), literally; setup in __init__ (:66-102), one loop body
    per step() (:108-139)."""

    def __init__(self, M_obs: np.ndarray, mask: np.ndarray, basis: EigenBasis,
                 cfg: Optional[SolverConfig] = None, validate_basis: bool = True,
                 z_update=None):
        cfg = cfg or SolverConfig()
        self.z_update = z_update or (lambda Xt, tau: _prox_l21_t(Xt, tau)[0])
        if validate_basis:
            basis.validate()                                     # solver.cpp:156
        cfg.validate()                                           # :66
        ks = tuple(basis.kernel_shape)
        validate_kernel(ks, M_obs.shape)                         # :67
        if mask.shape != M_obs.shape:                            # :68-69
            raise ValueError("solve: mask dims != observation dims")
        if np.any((mask != 0.0) & (mask != 1.0)):                # tensor.hpp:115-121
            raise ValueError("SamplingMask: entries must be 0 or 1")
        if int(mask.sum() + 0.5) == 0:                           # :70-71
            raise ValueError("solve: empty sampling set")
        if not np.all(np.isfinite(M_obs)):                       # :72
            raise ValueError("solve: observations: non-finite tensor entries")
        self.t_start = time.perf_counter()
        self.cfg, self.ks, self.basis = cfg, ks, basis
        self.M_obs, self.mask = M_obs, mask
        self.dims = M_obs.shape
        self.k = k = int(np.prod(ks))
        self.pm = pm = M_obs * mask                              # :80
        L = pm.copy()                                            # :82
        if cfg.init_fill == "mean":                              # :83-86
            L = L + (1.0 - mask) * (pm.sum() / float(int(mask.sum() + 0.5)))
        self.L = L
        theta = cfg.theta0 if cfg.theta0 is not None else 1e-2 * np.max(np.abs(pm)) * k  # :88-89
        if theta <= 0:
            theta = 1e-2                                         # :90
        self.theta = min(theta, cfg.theta_max)                   # :91
        self.conv = BasisConvolver(self.dims, ks, basis.K)       # :93
        rs = np.sqrt(k) * np.linalg.norm(pm)                     # :97
        self.res_scale = rs if rs != 0 else 1.0                  # :98
        self.AKL = self.conv.apply_t(L)                          # :100  (k, *dims)
        self.Z = self.AKL.copy()                                 # :101
        self.Y = np.zeros_like(self.AKL)                         # :102
        self.report = SolveReport()
        self.report.termination = "max_iters"
        self.it = 0

    def step(self) -> bool:
        """One iteration; returns True when the stopping test fires."""
        cfg, k, theta = self.cfg, self.k, self.theta
        flat = (k, -1)
        self.Z = self.z_update(self.AKL - self.Y / theta, 1.0 / theta)  # :108
        # WK = (Y + theta Z) K^T  -> transposed: K (Y + theta Z)^T      (:110)
        WKt = (self.basis.K @ (self.Y + theta * self.Z).reshape(flat)).reshape(self.AKL.shape)
        adj = conv_adjoint_t(WKt, self.ks, self.dims)            # :111
        numer = adj / k + cfg.lambda_ * self.pm                  # :112-113
        denom = cfg.lambda_ * self.mask + theta                  # :114-115
        L_new = numer / denom                                    # :116
        l_change = np.linalg.norm(L_new - self.L) / max(np.linalg.norm(self.L), 1e-300)  # :118-119
        self.L = L_new                                           # :120
        self.AKL = self.conv.apply_t(self.L)                     # :121
        gap = self.Z - self.AKL                                  # :123
        residual = np.linalg.norm(gap) / self.res_scale          # :124
        self.Y += theta * gap                                    # :125
        self.theta = min(theta * cfg.theta_growth, cfg.theta_max)  # :126
        col_sum = float(np.sum(np.linalg.norm(self.Z.reshape(flat), axis=1)))  # :128-129
        fit = float(np.sum(((self.L - self.M_obs) * self.mask) ** 2))  # :130
        rep = self.report
        rep.objective.append(col_sum + 0.5 * cfg.lambda_ * k * fit)    # :131-132
        rep.primal_residual.append(residual)
        rep.l_change.append(l_change)
        self.it += 1
        rep.iterations = self.it
        if residual < cfg.tol_primal or l_change < cfg.tol_change:      # :136-139
            rep.termination = "converged"
            return True
        return False


def icnnm_solve(M_obs: np.ndarray, mask: np.ndarray, basis: EigenBasis,
                cfg: Optional[SolverConfig] = None, validate_basis: bool = True
                ) -> Tuple[np.ndarray, SolveReport]:
    """icnnm_solve (solver.cpp:150-159)."""
    s = AdmmSolver(M_obs, mask, basis, cfg, validate_basis)
    for _ in range(s.cfg.max_iters):                             # :107
        if s.step():
            break
    s.report.wall_time_seconds = time.perf_counter() - s.t_start
    return s.L, s.report


def svt(W: np.ndarray, tau: float) -> np.ndarray:
    """svt (solver.cpp:52-57): U max(S - tau, 0) V^T of a thin SVD."""
    if tau < 0:
        raise ValueError("svt: tau must be >= 0")
    U, S, Vt = np.linalg.svd(W, full_matrices=False)
    return (U * np.maximum(S - tau, 0.0)) @ Vt


def _svt_t(Wt: np.ndarray, tau: float) -> np.ndarray:
    # transposed storage (k, *dims): svt(W^T) = svt(W)^T
    k = Wt.shape[0]
    return svt(Wt.reshape(k, -1), tau).reshape(Wt.shape)


def cnnm_solve(M_obs: np.ndarray, mask: np.ndarray, ks, cfg: Optional[SolverConfig] = None
               ) -> Tuple[np.ndarray, SolveReport]:
    """cnnm_solve (solver.cpp:161-170): the shared ADMM loop with K = I and
    the singular-value-thresholding Z-update (the CNNM baseline)."""
    ks = tuple(int(d) for d in ks)
    k = int(np.prod(ks))
    validate_kernel(ks, M_obs.shape)
    s = AdmmSolver(M_obs, mask, EigenBasis(ks, np.eye(k), np.zeros(k)), cfg,
                   validate_basis=False, z_update=_svt_t)
    for _ in range(s.cfg.max_iters):
        if s.step():
            break
    s.report.wall_time_seconds = time.perf_counter() - s.t_start
    return s.L, s.report


def objective_icnnm(L, M_obs, mask, basis: EigenBasis, lam: float) -> float:
    """objective_icnnm (solver.cpp:172-187)."""
    basis.validate()
    conv = BasisConvolver(L.shape, basis.kernel_shape, basis.K)
    AKL = conv.apply_t(L).reshape(basis.K.shape[0], -1)
    col_sum = float(np.sum(np.linalg.norm(AKL, axis=1)))
    fit = float(np.sum(((L - M_obs) * mask) ** 2))
    return col_sum + 0.5 * lam * basis.K.shape[0] * fit


def mse(ref, est) -> float:
    """mse (metrics.cpp:28-32)."""
    return float(np.mean((np.asarray(ref) - np.asarray(est)) ** 2))


def psnr(ref, est, peak: float = 1.0) -> float:
    """psnr (metrics.cpp:34-38): +inf when MSE is 0."""
    e = mse(ref, est)
    if e == 0:
        return float("inf")
    return 10.0 * np.log10(peak * peak / e)


def rel_l2(a, b) -> float:
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


# ---------------------------------------------------------------------------
# Recovery-theory diagnostics (core/src/analysis.cpp) and the spectrum /
# generator helpers its tests use.
# ---------------------------------------------------------------------------
DEFAULT_RANK_TOL = 1e-8  # kDefaultRankTol (spectral.hpp:25)


@dataclasses.dataclass
class ConvSpectrum:
    singular_values: np.ndarray
    eigenvectors: np.ndarray
    rank: int
    degenerate: bool


def conv_spectrum(L: np.ndarray, ks, tol: float = DEFAULT_RANK_TOL) -> ConvSpectrum:
    """conv_spectrum (spectral.cpp:102-131): Gram eigen-decomposition with the
    k*eps*lambda_1 backward-error floor on the rank cut."""
    validate_kernel(ks, L.shape)
    k = int(np.prod(ks))
    if np.linalg.norm(L) == 0.0:
        return ConvSpectrum(np.zeros(k), np.eye(k), 0, True)
    w, V = psd_eig_sorted(conv_gram(L, ks))
    floor = k * np.finfo(float).eps * w[0]
    cut = max(tol * tol * w[0], floor)
    return ConvSpectrum(np.sqrt(w), V, int(np.sum(w > cut)), False)


def synth_low_conv_rank(dims, ks, target_rank: int, rng) -> np.ndarray:
    """synth_low_conv_rank (synth.cpp:27-93).  `rng` is an mt19937_64 stream
    seeded like the reference (uniform / uniform_int draws in the same order)."""
    dims = tuple(int(d) for d in dims)
    validate_kernel(ks, dims)
    k = int(np.prod(ks))
    if target_rank < 1 or target_rank > k:
        raise ValueError("synth_low_conv_rank: infeasible target rank")
    if target_rank >= k:
        return rng.uniform(-1.0, 1.0, int(np.prod(dims))).reshape(dims)
    if target_rank == 1:
        c = 0.0
        while abs(c) < 0.1:
            c = float(rng.uniform(-1.0, 1.0, 1)[0])
        return np.full(dims, c)
    use_dc = target_rank % 2 != 0
    n_cos = (target_rank - 1 if use_dc else target_rank) // 2
    out = np.zeros(dims)
    used = set()
    if use_dc:
        out[...] = float(rng.uniform(0.5, 1.5, 1)[0])
        used.add((0,) * len(dims))
    grids = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    for _ in range(n_cos):
        for attempt in itertools.count():
            if attempt > 1000:
                raise RuntimeError("synth_low_conv_rank: frequency sampling stuck")
            f = [int(rng.uniform_int(0, d - 1, 1)[0]) for d in dims]
            canon = tuple(min(fj, d - fj) for fj, d in zip(f, dims))
            if any(fj != 0 for fj in f) and canon not in used:
                used.add(canon)
                break
        A = float(rng.uniform(0.5, 1.5, 1)[0])
        phi = float(rng.uniform(0.0, 2.0 * np.pi, 1)[0])
        arg = np.full(dims, phi)
        for fj, d, g in zip(f, dims, grids):
            arg = arg + 2.0 * np.pi * fj * g / d
        out += A * np.cos(arg)
    if conv_spectrum(out, ks, 1e-8).rank > target_rank:
        raise RuntimeError("synth_low_conv_rank: rank check failed")
    return out


def relative_eigenvalues(L0: np.ndarray, basis: EigenBasis) -> np.ndarray:
    """relative_eigenvalues (analysis.cpp:29-38): ||L0 * kernel_i||_F."""
    basis.validate()
    validate_kernel(basis.kernel_shape, L0.shape)
    k = basis.K.shape[0]
    return np.array([np.linalg.norm(circular_convolve(L0, basis.K[:, i].reshape(basis.kernel_shape)))
                     for i in range(k)])


def support_from(sigma: np.ndarray, rank_tol: float) -> List[int]:
    """support_from (analysis.cpp:40-49)."""
    smax = float(np.max(sigma))
    if smax == 0:
        return []
    return [i for i in range(len(sigma)) if sigma[i] > rank_tol * smax]


def power_iteration_top_eig(S: np.ndarray) -> float:
    """power_iteration_top_eig (analysis.cpp:51-69)."""
    n = S.shape[0]
    v = np.ones(n) / np.sqrt(float(n))
    eig = 0.0
    for it in range(10000):
        w = S @ v
        nw = np.linalg.norm(w)
        if nw == 0:
            return 0.0
        w = w / nw
        new_eig = float(w @ (S @ w))
        done = abs(new_eig - eig) <= 1e-10 * max(1.0, abs(new_eig))
        eig = new_eig
        v = w
        if done and it > 0:
            break
    return eig


def relative_conv_rank(L0, basis: EigenBasis, rank_tol: float = DEFAULT_RANK_TOL):
    """relative_conv_rank (analysis.cpp:71-77)."""
    sup = support_from(relative_eigenvalues(L0, basis), rank_tol)
    return len(sup), sup


def spectral_corr_coeff(L0, basis: EigenBasis, rank_tol: float = DEFAULT_RANK_TOL) -> float:
    """spectral_corr_coeff (analysis.cpp:79-96)."""
    sigma = relative_eigenvalues(L0, basis)
    sup = support_from(sigma, rank_tol)
    if not sup:
        raise ValueError("spectral_corr_coeff: r_K = 0, undefined")
    G = conv_gram(L0, basis.kernel_shape)
    KD = basis.K[:, sup] / sigma[sup]
    S = KD.T @ G @ KD
    return float(np.sqrt(max(0.0, power_iteration_top_eig(S))))


def active_coherence(basis: EigenBasis, support_I: Sequence[int]) -> float:
    """active_coherence (analysis.cpp:98-109)."""
    if len(support_I) == 0:
        raise ValueError("active_coherence: empty support")
    k = basis.K.shape[0]
    rows = np.sum(basis.K[:, list(support_I)] ** 2, axis=1)
    return k / len(support_I) * float(np.max(rows))


@dataclasses.dataclass
class ConvCoherence:
    mu1: float
    mu2: float
    tau: float
    rank: int


def conv_coherence(L0: np.ndarray, ks, rank_tol: float = DEFAULT_RANK_TOL) -> ConvCoherence:
    """conv_coherence (analysis.cpp:111-135): thin SVD of the dense conv matrix."""
    if np.linalg.norm(L0) == 0:
        raise ValueError("conv_coherence: zero tensor")
    A = conv_matrix(L0, ks)
    U, s, Vt = np.linalg.svd(A, full_matrices=False)
    r = int(np.sum(s > rank_tol * s[0]))
    m, k = A.shape
    mu1 = m / r * float(np.max(np.sum(U[:, :r] ** 2, axis=1)))
    mu2 = k / r * float(np.max(np.sum(Vt[:r, :].T ** 2, axis=1)))
    return ConvCoherence(mu1, mu2, float(s[0] / s[r - 1]), r)


@dataclasses.dataclass
class ThresholdInputs:
    r_K: int = 0
    alpha_K: float = 0.0
    mu_K_I: float = 0.0
    mu1: float = 0.0
    mu2: float = 0.0
    r0: int = 0
    k: int = 0
    m: int = 0
    rho0: float = 0.0


def thresholds(inp: ThresholdInputs) -> dict:
    """thresholds (analysis.cpp:137-153)."""
    a2 = inp.alpha_K ** 2
    k, m, rk, r0 = float(inp.k), float(inp.m), float(inp.r_K), float(inp.r0)
    t = dict(
        rho_min_noiseless=1.0 - k / ((1.0 + a2) * inp.mu_K_I * rk * m),
        rho_min_noisy=1.0 - 0.64 * k / ((0.64 + a2) * inp.mu_K_I * rk * m),
        error_bound_factor=(18.0 * np.sqrt(k) + 2.0) * (inp.alpha_K + np.sqrt(1.0 + a2)) / inp.alpha_K,
        icnnm_ideal_bound=1.0 - 0.5 * k / (inp.mu2 * r0 * m),
        cnnm_bound=1.0 - 0.25 * k / (max(inp.mu1, inp.mu2) * r0 * m),
    )
    t["certified"] = inp.rho0 > t["rho_min_noiseless"]
    return t


def analyze_recovery(L0, basis: EigenBasis, mask, rank_tol: float = DEFAULT_RANK_TOL) -> dict:
    """analyze_recovery (analysis.cpp:155-185)."""
    if mask.shape != L0.shape:
        raise ValueError("analyze_recovery: mask dims != target dims")
    if np.any((mask != 0.0) & (mask != 1.0)):
        raise ValueError("SamplingMask: entries must be 0 or 1")
    rk, sup = relative_conv_rank(L0, basis, rank_tol)
    if rk == 0:
        raise ValueError("analyze_recovery: zero target, diagnostics undefined")
    d = dict(r_K=rk, support_I=sup)
    d["alpha_K"] = spectral_corr_coeff(L0, basis, rank_tol)
    d["mu_K_I"] = active_coherence(basis, sup)
    cc = conv_coherence(L0, basis.kernel_shape, rank_tol)
    d.update(mu1=cc.mu1, mu2=cc.mu2, tau=cc.tau, r0=cc.rank)
    d["rho0"] = int(np.sum(mask) + 0.5) / mask.size
    d.update(thresholds(ThresholdInputs(rk, d["alpha_K"], d["mu_K_I"], cc.mu1, cc.mu2, cc.rank,
                                        basis.K.shape[0], L0.size, d["rho0"])))
    return d
