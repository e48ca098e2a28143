"""Recovery-theory diagnostics on the GPU: mirror of the reference's
``icnnm/analysis.hpp`` (/root/reference/proj/core/include/icnnm/analysis.hpp:25-99,
core/src/analysis.cpp).  Same names, argument meaning and error behaviour;
the compute is the matrix-free fp64 path of ``csrc/icnnm_analysis.cu``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Sequence, Tuple

import numpy as np

from ._lib import (ConvCoherenceC, RecoveryDiagnosticsC, ThresholdInputsC, ThresholdValuesC,
                   check, dptr, lib, lptr)
from .api import EigenBasis, InvalidArgument, _check_basis_shape, _colmajor, _dims, _f64

DEFAULT_RANK_TOL = 1e-8  # kDefaultRankTol (spectral.hpp:25)


@dataclasses.dataclass
class ConvCoherence:
    """ConvCoherence (analysis.hpp:62-66)."""
    mu1: float = 0.0
    mu2: float = 0.0
    tau: float = 0.0
    rank: int = 0


@dataclasses.dataclass
class ThresholdInputs:
    """ThresholdInputs (analysis.hpp:72-82)."""
    r_K: int = 0
    alpha_K: float = 0.0
    mu_K_I: float = 0.0
    mu1: float = 0.0
    mu2: float = 0.0
    r0: int = 0
    k: int = 0
    m: int = 0
    rho0: float = 0.0


@dataclasses.dataclass
class Thresholds:
    """Thresholds (analysis.hpp:84-91)."""
    rho_min_noiseless: float = 0.0
    rho_min_noisy: float = 0.0
    error_bound_factor: float = 0.0
    cnnm_bound: float = 0.0
    icnnm_ideal_bound: float = 0.0
    certified: bool = False


@dataclasses.dataclass
class RecoveryDiagnostics:
    """RecoveryDiagnostics (analysis.hpp:29-44)."""
    r_K: int = 0
    support_I: List[int] = dataclasses.field(default_factory=list)
    alpha_K: float = 0.0
    mu_K_I: float = 0.0
    mu1: float = 0.0
    mu2: float = 0.0
    tau: float = 0.0
    r0: int = 0
    rho0: float = 0.0
    rho_min_noiseless: float = 0.0
    rho_min_noisy: float = 0.0
    error_bound_factor: float = 0.0
    cnnm_bound: float = 0.0
    icnnm_ideal_bound: float = 0.0
    certified: bool = False


def _basis_args(L0, basis: EigenBasis):
    L0 = _f64(L0)
    _check_basis_shape(basis, L0.shape)
    ev = None if basis.eigenvalues is None else _f64(basis.eigenvalues)
    return L0, _colmajor(basis.K), ev


def relative_eigenvalues(L0, basis: EigenBasis, device: int = 0) -> np.ndarray:
    """sigma^K_i = ||A(L0) K_i|| (analysis.cpp:29-38)."""
    L0, Kc, ev = _basis_args(L0, basis)
    out = np.empty(basis.k())
    check(lib().icnnm_cuda_relative_eigenvalues(
        L0.ndim, lptr(_dims(L0.shape)), dptr(L0), lptr(_dims(basis.kernel_shape)), dptr(Kc),
        None if ev is None else dptr(ev), device, dptr(out)))
    return out


def relative_conv_rank(L0, basis: EigenBasis, rank_tol: float = DEFAULT_RANK_TOL,
                       device: int = 0) -> Tuple[int, List[int]]:
    """relative_conv_rank (analysis.cpp:71-77): (r_K, support I)."""
    L0, Kc, ev = _basis_args(L0, basis)
    sup = np.zeros(basis.k(), dtype=np.int64)
    r = C.c_int64()
    check(lib().icnnm_cuda_relative_conv_rank(
        L0.ndim, lptr(_dims(L0.shape)), dptr(L0), lptr(_dims(basis.kernel_shape)), dptr(Kc),
        None if ev is None else dptr(ev), float(rank_tol), device, C.byref(r), lptr(sup)))
    return r.value, sup[: r.value].tolist()


def spectral_corr_coeff(L0, basis: EigenBasis, rank_tol: float = DEFAULT_RANK_TOL,
                        device: int = 0) -> float:
    """spectral_corr_coeff (analysis.cpp:79-96)."""
    L0, Kc, ev = _basis_args(L0, basis)
    out = C.c_double()
    check(lib().icnnm_cuda_spectral_corr_coeff(
        L0.ndim, lptr(_dims(L0.shape)), dptr(L0), lptr(_dims(basis.kernel_shape)), dptr(Kc),
        None if ev is None else dptr(ev), float(rank_tol), device, C.byref(out)))
    return out.value


def active_coherence(basis: EigenBasis, support_I: Sequence[int]) -> float:
    """active_coherence (analysis.cpp:98-109)."""
    sup = np.ascontiguousarray(np.asarray(list(support_I), dtype=np.int64))
    out = C.c_double()
    check(lib().icnnm_active_coherence(basis.k(), dptr(_colmajor(basis.K)), len(sup),
                                       lptr(sup) if len(sup) else None, C.byref(out)))
    return out.value


def conv_coherence(L0, kernel_shape, rank_tol: float = DEFAULT_RANK_TOL,
                   device: int = 0) -> ConvCoherence:
    """conv_coherence (analysis.cpp:111-135), matrix-free."""
    L0 = _f64(L0)
    kernel_shape = tuple(int(d) for d in kernel_shape)
    if len(kernel_shape) != L0.ndim:
        raise InvalidArgument("KernelShape: order mismatch with tensor")
    out = ConvCoherenceC()
    check(lib().icnnm_cuda_conv_coherence(L0.ndim, lptr(_dims(L0.shape)), dptr(L0),
                                          lptr(_dims(kernel_shape)), float(rank_tol), device,
                                          C.byref(out)))
    return ConvCoherence(out.mu1, out.mu2, out.tau, int(out.rank))


def thresholds(inp: ThresholdInputs) -> Thresholds:
    """thresholds (analysis.cpp:137-153)."""
    c = ThresholdInputsC(int(inp.r_K), inp.alpha_K, inp.mu_K_I, inp.mu1, inp.mu2, int(inp.r0),
                         int(inp.k), int(inp.m), inp.rho0)
    o = ThresholdValuesC()
    check(lib().icnnm_thresholds(C.byref(c), C.byref(o)))
    return Thresholds(o.rho_min_noiseless, o.rho_min_noisy, o.error_bound_factor, o.cnnm_bound,
                      o.icnnm_ideal_bound, bool(o.certified))


def _diag_from_c(d: RecoveryDiagnosticsC, sup: np.ndarray) -> RecoveryDiagnostics:
    return RecoveryDiagnostics(
        r_K=int(d.r_K), support_I=sup[: d.r_K].tolist(), alpha_K=d.alpha_K, mu_K_I=d.mu_K_I,
        mu1=d.mu1, mu2=d.mu2, tau=d.tau, r0=int(d.r0), rho0=d.rho0,
        rho_min_noiseless=d.rho_min_noiseless, rho_min_noisy=d.rho_min_noisy,
        error_bound_factor=d.error_bound_factor, cnnm_bound=d.cnnm_bound,
        icnnm_ideal_bound=d.icnnm_ideal_bound, certified=bool(d.certified))


def analyze_recovery(L0, basis: EigenBasis, mask, rank_tol: float = DEFAULT_RANK_TOL,
                     device: int = 0) -> RecoveryDiagnostics:
    """analyze_recovery (analysis.cpp:155-185)."""
    L0, Kc, ev = _basis_args(L0, basis)
    W = _f64(mask)
    if W.shape != L0.shape:
        raise InvalidArgument("analyze_recovery: mask dims != target dims")
    sup = np.zeros(basis.k(), dtype=np.int64)
    d = RecoveryDiagnosticsC()
    d.support_I = lptr(sup)
    check(lib().icnnm_cuda_analyze_recovery(
        L0.ndim, lptr(_dims(L0.shape)), dptr(L0), lptr(_dims(basis.kernel_shape)), dptr(Kc),
        None if ev is None else dptr(ev), dptr(W), float(rank_tol), device, C.byref(d)))
    return _diag_from_c(d, sup)


def diagnostics_to_json(d: RecoveryDiagnostics) -> str:
    """diagnostics_to_json (report_io.cpp:70-88) through the C ABI."""
    sup = np.ascontiguousarray(np.asarray(d.support_I, dtype=np.int64))
    c = RecoveryDiagnosticsC(int(d.r_K), lptr(sup) if len(sup) else None, d.alpha_K, d.mu_K_I,
                             d.mu1, d.mu2, d.tau, int(d.r0), d.rho0, d.rho_min_noiseless,
                             d.rho_min_noisy, d.error_bound_factor, d.cnnm_bound,
                             d.icnnm_ideal_bound, int(d.certified))
    n = lib().icnnm_diagnostics_to_json(C.byref(c), None, 0)
    buf = C.create_string_buffer(n + 1)
    lib().icnnm_diagnostics_to_json(C.byref(c), buf, n + 1)
    return buf.value.decode()
