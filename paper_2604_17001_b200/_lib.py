"""ctypes binding of the in-tree C-ABI library ``libicnnm_b200.so``.

The library is the product: every solver/operator call goes through it. If it
is missing (not built) any call raises immediately -- there is no CPU or
PyTorch fallback on the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libicnnm_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "icnnm_b200.h")

ICNNM_OK = 0
ICNNM_INVALID_ARGUMENT = 1
ICNNM_RUNTIME_ERROR = 2
ICNNM_CUDA_ERROR = 3


class IcnnmError(RuntimeError):
    """Base class of library failures."""


class InvalidArgument(IcnnmError, ValueError):
    """std::invalid_argument in the reference (solver.cpp:26-40,66-72)."""


class CudaError(IcnnmError):
    """CUDA / NCCL failure (no reference analogue)."""


class SolverConfigC(C.Structure):
    _fields_ = [
        ("lambda_", C.c_double),
        ("has_theta0", C.c_int),
        ("theta0", C.c_double),
        ("theta_growth", C.c_double),
        ("theta_max", C.c_double),
        ("max_iters", C.c_int),
        ("tol_primal", C.c_double),
        ("tol_change", C.c_double),
        ("rank_tol", C.c_double),
        ("init_fill", C.c_int),
        ("engine", C.c_int),
        ("exact_residual", C.c_int),
    ]


class SolveReportC(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("objective", C.POINTER(C.c_double)),
        ("primal_residual", C.POINTER(C.c_double)),
        ("l_change", C.POINTER(C.c_double)),
        ("termination", C.c_int),
        ("wall_time_seconds", C.c_double),
        ("loop_seconds", C.c_double),
        ("device_seconds", C.c_double),
    ]


class ConvCoherenceC(C.Structure):
    _fields_ = [("mu1", C.c_double), ("mu2", C.c_double), ("tau", C.c_double),
                ("rank", C.c_int64)]


class ThresholdInputsC(C.Structure):
    _fields_ = [("r_K", C.c_int64), ("alpha_K", C.c_double), ("mu_K_I", C.c_double),
                ("mu1", C.c_double), ("mu2", C.c_double), ("r0", C.c_int64),
                ("k", C.c_int64), ("m", C.c_int64), ("rho0", C.c_double)]


class ThresholdValuesC(C.Structure):
    _fields_ = [("rho_min_noiseless", C.c_double), ("rho_min_noisy", C.c_double),
                ("error_bound_factor", C.c_double), ("cnnm_bound", C.c_double),
                ("icnnm_ideal_bound", C.c_double), ("certified", C.c_int)]


class RecoveryDiagnosticsC(C.Structure):
    _fields_ = [("r_K", C.c_int64), ("support_I", C.POINTER(C.c_int64)),
                ("alpha_K", C.c_double), ("mu_K_I", C.c_double), ("mu1", C.c_double),
                ("mu2", C.c_double), ("tau", C.c_double), ("r0", C.c_int64),
                ("rho0", C.c_double), ("rho_min_noiseless", C.c_double),
                ("rho_min_noisy", C.c_double), ("error_bound_factor", C.c_double),
                ("cnnm_bound", C.c_double), ("icnnm_ideal_bound", C.c_double),
                ("certified", C.c_int)]


_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)

# name -> (restype, argtypes); the full exported surface of include/icnnm_b200.h
SIGNATURES = {
    "icnnm_default_config": (None, [C.POINTER(SolverConfigC)]),
    "icnnm_validate_config": (C.c_int, [C.POINTER(SolverConfigC)]),
    "icnnm_last_error": (C.c_char_p, []),
    "icnnm_version": (C.c_char_p, []),
    "icnnm_device_count": (C.c_int, []),
    "icnnm_empty_cache": (C.c_int, []),
    "icnnm_cuda_solve": (C.c_int, [C.c_int, _lp, _dp, _dp, _lp, _dp, _dp,
                                   C.POINTER(SolverConfigC), C.c_int, _dp,
                                   C.POINTER(SolveReportC)]),
    "icnnm_cuda_solve_batch": (C.c_int, [C.c_int, C.c_int, _lp, C.POINTER(_dp), C.POINTER(_dp),
                                         _lp, _dp, _dp, C.POINTER(SolverConfigC),
                                         C.POINTER(C.c_int), C.c_int, C.POINTER(_dp),
                                         C.POINTER(SolveReportC)]),
    "icnnm_solver_create": (C.c_int, [C.c_int, _lp, _lp, _dp, _dp, C.c_int,
                                      C.POINTER(C.c_void_p)]),
    "icnnm_solver_upload": (C.c_int, [C.c_void_p, _dp, _dp]),
    "icnnm_solver_run": (C.c_int, [C.c_void_p, C.POINTER(SolverConfigC),
                                   C.POINTER(SolveReportC)]),
    "icnnm_solver_download": (C.c_int, [C.c_void_p, _dp]),
    "icnnm_solver_last_launches": (C.c_int64, [C.c_void_p]),
    "icnnm_solver_device_bytes": (C.c_int64, [C.c_void_p]),
    "icnnm_solver_set_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "icnnm_solver_kernel_times": (C.c_int, [C.c_void_p, _dp]),
    "icnnm_solver_destroy": (None, [C.c_void_p]),
    "icnnm_solver_tc_counters": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "icnnm_cuda_conv_forward": (C.c_int, [C.c_int, _lp, _dp, _lp, _dp, C.c_int, _dp]),
    "icnnm_cuda_conv_adjoint": (C.c_int, [C.c_int, _lp, _lp, _dp, C.c_int, _dp]),
    "icnnm_cuda_conv_forward_ex": (C.c_int, [C.c_int, _lp, _dp, _lp, _dp, C.c_int, C.c_int, _dp]),
    "icnnm_cuda_conv_adjoint_ex": (C.c_int, [C.c_int, _lp, _lp, _dp, C.c_int, C.c_int, _dp]),
    "icnnm_cuda_prox_l21": (C.c_int, [C.c_int64, C.c_int64, _dp, C.c_double, C.c_int, _dp]),
    "icnnm_cuda_conv_gram": (C.c_int, [C.c_int, _lp, _dp, _lp, C.c_int, _dp]),
    "icnnm_cuda_learn_basis": (C.c_int, [C.c_int, C.c_int, _lp, C.POINTER(_dp), _lp,
                                         C.c_int, _dp, _dp, C.POINTER(C.c_int)]),
    "icnnm_host_symeig": (C.c_int, [C.c_int, _dp, _dp, _dp]),
    "icnnm_cuda_objective": (C.c_int, [C.c_int, _lp, _dp, _dp, _dp, _lp, _dp,
                                       C.c_double, C.c_int, _dp]),
    "icnnm_dist_unique_id": (C.c_int, [C.c_char_p]),
    "icnnm_sharded_solve": (C.c_int, [C.c_int, _lp, _dp, _dp, _lp, _dp,
                                      C.POINTER(SolverConfigC), C.c_int, C.c_int,
                                      C.c_int, C.c_char_p, C.c_int, _dp, _lp, _lp,
                                      C.POINTER(SolveReportC)]),
    "icnnm_sharded_rows": (C.c_int, [C.c_int, _lp, _lp, C.c_int, C.c_int, C.c_int, _lp, _lp]),
    "icnnm_sharded_solve_local": (C.c_int, [C.c_int, _lp, C.c_int64, C.c_int64, _dp, _dp, _lp,
                                            _dp, C.POINTER(SolverConfigC), C.c_int, C.c_int,
                                            C.c_int, C.c_char_p, C.c_int, _dp,
                                            C.POINTER(SolveReportC)]),
    "icnnm_shard_plan": (C.c_int, [C.c_int64, C.c_int, C.c_int64, C.c_int, _lp, _lp]),
    "icnnm_probe_ffma_tflops": (C.c_int, [C.c_int, _dp]),
    "icnnm_probe_dfma_tflops": (C.c_int, [C.c_int, _dp]),
    "icnnm_io_last_error": (C.c_char_p, []),
    "icnnm_write_tnsr": (C.c_int, [C.c_char_p, C.c_int, _lp, _dp]),
    "icnnm_read_tnsr": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), _lp, _dp]),
    "icnnm_write_ebas": (C.c_int, [C.c_char_p, C.c_int, _lp, _dp, _dp]),
    "icnnm_read_ebas": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), _lp, _dp, _dp]),
    "icnnm_config_from_json": (C.c_int, [C.c_char_p, C.POINTER(SolverConfigC)]),
    "icnnm_report_to_json": (C.c_int64, [C.POINTER(SolveReportC), C.c_char_p, C.c_int64]),
    "icnnm_cuda_cnnm_solve": (C.c_int, [C.c_int, _lp, _dp, _dp, _lp, C.POINTER(SolverConfigC),
                                        C.c_int, _dp, C.POINTER(SolveReportC)]),
    "icnnm_diagnostics_to_json": (C.c_int64, [C.POINTER(RecoveryDiagnosticsC), C.c_char_p,
                                              C.c_int64]),
    "icnnm_cuda_relative_eigenvalues": (C.c_int, [C.c_int, _lp, _dp, _lp, _dp, _dp, C.c_int,
                                                  _dp]),
    "icnnm_cuda_relative_conv_rank": (C.c_int, [C.c_int, _lp, _dp, _lp, _dp, _dp, C.c_double,
                                                C.c_int, _lp, _lp]),
    "icnnm_cuda_spectral_corr_coeff": (C.c_int, [C.c_int, _lp, _dp, _lp, _dp, _dp, C.c_double,
                                                 C.c_int, _dp]),
    "icnnm_active_coherence": (C.c_int, [C.c_int64, _dp, C.c_int64, _lp, _dp]),
    "icnnm_cuda_conv_coherence": (C.c_int, [C.c_int, _lp, _dp, _lp, C.c_double, C.c_int,
                                            C.POINTER(ConvCoherenceC)]),
    "icnnm_thresholds": (C.c_int, [C.POINTER(ThresholdInputsC), C.POINTER(ThresholdValuesC)]),
    "icnnm_cuda_analyze_recovery": (C.c_int, [C.c_int, _lp, _dp, _lp, _dp, _dp, _dp,
                                              C.c_double, C.c_int,
                                              C.POINTER(RecoveryDiagnosticsC)]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the C-ABI library; raise loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise IcnnmError(
                    f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    " or `make -C paper_2604_17001_b200/csrc`")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(status: int) -> None:
    """Map a status code to the reference's exception classes."""
    if status == ICNNM_OK:
        return
    msg = lib().icnnm_last_error().decode(errors="replace")
    if status == ICNNM_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if status == ICNNM_CUDA_ERROR:
        raise CudaError(msg)
    raise IcnnmError(msg)


CLI_PATH = os.path.join(_HERE, "icnnm_b200")


def check_io(status: int) -> None:
    if status == ICNNM_OK:
        return
    msg = lib().icnnm_io_last_error().decode(errors="replace")
    if status == ICNNM_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    raise IcnnmError(msg)


def dptr(a):
    return a.ctypes.data_as(_dp)


def lptr(a):
    return a.ctypes.data_as(_lp)
