"""Host-side mirror of the reference's ICNNM C++ API over the C ABI.

Same names, argument meaning and error behaviour as
``/root/reference/proj/core/include/icnnm/{solver,conv_op,spectral}.hpp``:

=============================  ===============================================
reference (C++)                here (Python, numpy float64 arrays)
=============================  ===============================================
SolverConfig (solver.hpp:29)   :class:`SolverConfig`
SolveReport  (solver.hpp:46)   :class:`SolveReport`
EigenBasis   (spectral.hpp:30) :class:`EigenBasis`
icnnm_solve  (solver.hpp:64)   :func:`icnnm_solve`
learn_ensemble_basis (:72)     :func:`learn_ensemble_basis`
BasisConvolver::apply          :meth:`BasisConvolver.apply`
conv_adjoint (conv_op.hpp:54)  :func:`conv_adjoint`
prox_l21     (solver.hpp:56)   :func:`prox_l21`
conv_gram    (spectral.hpp:63) :func:`conv_gram`
objective_icnnm (solver.hpp:77):func:`objective_icnnm`
=============================  ===============================================

Tensors are numpy arrays (row-major, last index fastest, as DenseTensor);
m x k operator matrices are (m, k) arrays; K is the k x k matrix whose column
j is the row-major flattened eigen-kernel j.  ``std::invalid_argument`` maps
to :class:`InvalidArgument` (a ``ValueError``).  All compute runs on the GPU
through ``libicnnm_b200.so``.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

from ._lib import (SolveReportC, SolverConfigC, check, dptr, lib, lptr,
                   InvalidArgument)

ENGINES = {"ffma": 0, "tf32x3": 1, "f16x3": 2, "f64": 3, "auto": 4}


@dataclasses.dataclass
class SolverConfig:
    """icnnm::SolverConfig (solver.hpp:29-43); same defaults."""
    lambda_: float = 1000.0
    theta0: Optional[float] = None
    theta_growth: float = 1.05
    theta_max: float = 1e10
    max_iters: int = 1000
    tol_primal: float = 1e-7
    tol_change: float = 1e-8
    rank_tol: float = 1e-8
    init_fill: str = "zero"
    engine: str = "auto"        # include/icnnm_b200.h ICNNM_ENGINE_AUTO
    exact_residual: bool = False

    def to_c(self) -> SolverConfigC:
        if self.init_fill not in ("zero", "mean"):
            raise InvalidArgument("SolverConfig: init_fill must be 'zero' or 'mean'")
        if self.engine not in ENGINES:
            raise InvalidArgument("SolverConfig: unknown engine")
        c = SolverConfigC()
        c.lambda_ = float(self.lambda_)
        c.has_theta0 = 0 if self.theta0 is None else 1
        c.theta0 = 0.0 if self.theta0 is None else float(self.theta0)
        c.theta_growth = float(self.theta_growth)
        c.theta_max = float(self.theta_max)
        c.max_iters = int(self.max_iters)
        c.tol_primal = float(self.tol_primal)
        c.tol_change = float(self.tol_change)
        c.rank_tol = float(self.rank_tol)
        c.init_fill = 0 if self.init_fill == "zero" else 1
        c.engine = ENGINES[self.engine]
        c.exact_residual = 1 if self.exact_residual else 0
        return c

    def validate(self) -> None:
        """SolverConfig::validate (solver.cpp:26-40)."""
        c = self.to_c()
        check(lib().icnnm_validate_config(C.byref(c)))


@dataclasses.dataclass
class SolveReport:
    """icnnm::SolveReport (solver.hpp:46-52) plus l_change / loop_seconds."""
    iterations: int = 0
    objective: List[float] = dataclasses.field(default_factory=list)
    primal_residual: List[float] = dataclasses.field(default_factory=list)
    termination: str = "max_iters"
    wall_time_seconds: float = 0.0
    l_change: List[float] = dataclasses.field(default_factory=list)
    loop_seconds: float = 0.0
    device_seconds: float = 0.0


@dataclasses.dataclass
class EigenBasis:
    """icnnm::EigenBasis (spectral.hpp:30-44)."""
    kernel_shape: Tuple[int, ...]
    K: np.ndarray
    eigenvalues: np.ndarray
    degenerate: bool = False

    def k(self) -> int:
        return int(np.prod(self.kernel_shape))

    def kernel(self, i: int) -> np.ndarray:
        return self.K[:, i].reshape(self.kernel_shape)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _dims(shape) -> np.ndarray:
    return np.asarray(list(shape), dtype=np.int64)


def _colmajor(K: np.ndarray) -> np.ndarray:
    # column-major bytes of K == C-order bytes of K^T
    return np.ascontiguousarray(np.asarray(K, dtype=np.float64).T)


def _report_buffers(n: int):
    obj = np.zeros(n)
    res = np.zeros(n)
    lc = np.zeros(n)
    rep = SolveReportC()
    rep.objective = dptr(obj)
    rep.primal_residual = dptr(res)
    rep.l_change = dptr(lc)
    return rep, obj, res, lc


def _report_from_c(rep, obj, res, lc) -> SolveReport:
    n = rep.iterations
    return SolveReport(
        iterations=n,
        objective=obj[:n].tolist(),
        primal_residual=res[:n].tolist(),
        termination="converged" if rep.termination == 1 else "max_iters",
        wall_time_seconds=rep.wall_time_seconds,
        l_change=lc[:n].tolist(),
        loop_seconds=rep.loop_seconds,
        device_seconds=rep.device_seconds,
    )


def _check_basis_shape(basis: EigenBasis, dims) -> None:
    if len(basis.kernel_shape) != len(dims):
        raise InvalidArgument("KernelShape: order mismatch with tensor")
    k = basis.k()
    if basis.K.shape != (k, k):
        raise InvalidArgument("EigenBasis: K must be k x k")
    if basis.eigenvalues is not None and len(basis.eigenvalues) != k:
        raise InvalidArgument("EigenBasis: eigenvalue count mismatch")


def icnnm_solve(M_obs, mask, basis: EigenBasis, cfg: Optional[SolverConfig] = None,
                device: int = 0) -> Tuple[np.ndarray, SolveReport]:
    """icnnm_solve (solver.hpp:64-67; solver.cpp:150-159) on the GPU."""
    cfg = cfg or SolverConfig()
    M = _f64(M_obs)
    W = _f64(mask)
    if M.shape != W.shape:
        raise InvalidArgument("solve: mask dims != observation dims")
    _check_basis_shape(basis, M.shape)
    c = cfg.to_c()
    L = np.empty_like(M)
    rep, obj, res, lc = _report_buffers(max(int(cfg.max_iters), 1))
    Kc = _colmajor(basis.K)
    ev = _f64(basis.eigenvalues) if basis.eigenvalues is not None else None
    check(lib().icnnm_cuda_solve(M.ndim, lptr(_dims(M.shape)), dptr(M), dptr(W),
                                 lptr(_dims(basis.kernel_shape)), dptr(Kc),
                                 dptr(ev) if ev is not None else None, C.byref(c),
                                 device, dptr(L), C.byref(rep)))
    return L, _report_from_c(rep, obj, res, lc)


def icnnm_solve_batch(M_obs: Sequence[np.ndarray], masks, basis: EigenBasis,
                      cfg: Optional[SolverConfig] = None, devices: Sequence[int] = (0,)
                      ) -> Tuple[List[np.ndarray], List[SolveReport]]:
    """A batch of independent icnnm_solve calls sharing one basis and config
    (BASELINE config 4), split in contiguous blocks over `devices` inside one
    library call (icnnm_cuda_solve_batch).  `masks` is one mask per tensor or
    a single mask shared by all.  Returns the recovered tensors and one
    SolveReport per tensor."""
    cfg = cfg or SolverConfig()
    Ms = [_f64(x) for x in M_obs]
    n = len(Ms)
    if n == 0:
        return [], []
    if isinstance(masks, np.ndarray) and masks.shape == Ms[0].shape:
        Ws = [_f64(masks)] * n
    else:
        Ws = [_f64(x) for x in masks]
    if len(Ws) != n:
        raise InvalidArgument("solve_batch: one mask per tensor (or one shared mask)")
    shape = Ms[0].shape
    for M, W in zip(Ms, Ws):
        if M.shape != shape or W.shape != shape:
            raise InvalidArgument("solve_batch: all tensors and masks must share dims")
    _check_basis_shape(basis, shape)
    c = cfg.to_c()
    Ls = [np.empty_like(M) for M in Ms]
    bufs = [_report_buffers(max(int(cfg.max_iters), 1)) for _ in range(n)]
    reps = (SolveReportC * n)()
    for i, (rep, _, _, _) in enumerate(bufs):
        reps[i] = rep
    Kc = _colmajor(basis.K)
    ev = _f64(basis.eigenvalues) if basis.eigenvalues is not None else None
    pM = (C.POINTER(C.c_double) * n)(*[dptr(x) for x in Ms])
    pW = (C.POINTER(C.c_double) * n)(*[dptr(x) for x in Ws])
    pL = (C.POINTER(C.c_double) * n)(*[dptr(x) for x in Ls])
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    check(lib().icnnm_cuda_solve_batch(n, len(shape), lptr(_dims(shape)), pM, pW,
                                       lptr(_dims(basis.kernel_shape)), dptr(Kc),
                                       dptr(ev) if ev is not None else None, C.byref(c),
                                       devs, len(devices), pL, reps))
    out = [_report_from_c(reps[i], b[1], b[2], b[3]) for i, b in enumerate(bufs)]
    return Ls, out


class Solver:
    """Handle API: basis bound once (BasisConvolver's precompute-once
    pattern, conv_op.hpp:61-81); problems are uploaded to HBM and solved
    from there.  ``run`` is the device-resident hot path."""

    def __init__(self, dims, basis: EigenBasis, device: int = 0):
        _check_basis_shape(basis, dims)
        self.dims = tuple(int(d) for d in dims)
        self.device = device
        Kc = _colmajor(basis.K)
        ev = _f64(basis.eigenvalues) if basis.eigenvalues is not None else None
        h = C.c_void_p()
        check(lib().icnnm_solver_create(len(self.dims), lptr(_dims(self.dims)),
                                        lptr(_dims(basis.kernel_shape)), dptr(Kc),
                                        dptr(ev) if ev is not None else None, device,
                                        C.byref(h)))
        self._h = h

    def upload(self, M_obs, mask) -> None:
        M = _f64(M_obs)
        W = _f64(mask)
        if M.shape != self.dims or W.shape != self.dims:
            raise InvalidArgument("solve: tensor dims mismatch")
        check(lib().icnnm_solver_upload(self._h, dptr(M), dptr(W)))

    def run(self, cfg: Optional[SolverConfig] = None) -> SolveReport:
        cfg = cfg or SolverConfig()
        c = cfg.to_c()
        rep, obj, res, lc = _report_buffers(max(int(cfg.max_iters), 1))
        check(lib().icnnm_solver_run(self._h, C.byref(c), C.byref(rep)))
        return _report_from_c(rep, obj, res, lc)

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is not None:
            if (not isinstance(out, np.ndarray) or out.shape != tuple(self.dims)
                    or out.dtype != np.float64 or not out.flags.c_contiguous
                    or not out.flags.writeable):
                raise InvalidArgument("download: out must be a writeable C-contiguous "
                                      f"float64 array of shape {tuple(self.dims)}")
            L = out
        else:
            L = np.empty(self.dims)
        check(lib().icnnm_solver_download(self._h, dptr(L)))
        return L

    def set_profile(self, on, tc_counters: bool = False) -> None:
        check(lib().icnnm_solver_set_profile(self._h, (1 if on else 0) | (2 if tc_counters else 0)))

    def tc_counters(self) -> dict:
        out = (C.c_uint64 * 20)()
        check(lib().icnnm_solver_tc_counters(self._h, out))
        names = ["build_wait", "build_work", "mma_wait_a", "mma_wait_b", "mma_wait_acc",
                 "epi_wait", "epi_work", "load_wait", "mma_total", "build_prep"]
        return {"forward": dict(zip(names, out[:10])), "adjoint": dict(zip(names, out[10:]))}

    def kernel_times_ms(self) -> dict:
        out = np.zeros(4)
        check(lib().icnnm_solver_kernel_times(self._h, dptr(out)))
        return {"forward": out[0], "adjoint": out[1], "update": out[2], "coef": out[3]}

    @property
    def last_launches(self) -> int:
        return int(lib().icnnm_solver_last_launches(self._h))

    @property
    def device_bytes(self) -> int:
        return int(lib().icnnm_solver_device_bytes(self._h))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().icnnm_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class BasisConvolver:
    """BasisConvolver (conv_op.hpp:65-81): apply(L) = A_k(L) K (m x k)."""

    def __init__(self, tensor_dims, kernel_shape, K, device: int = 0, engine: str = "ffma"):
        if engine not in ENGINES:
            raise InvalidArgument("unknown engine")
        self.engine = ENGINES[engine]
        self.dims = tuple(int(d) for d in tensor_dims)
        self.kernel_shape = tuple(int(d) for d in kernel_shape)
        k = int(np.prod(self.kernel_shape))
        K = np.asarray(K, dtype=np.float64)
        if K.shape != (k, k):
            raise InvalidArgument("BasisConvolver: K must be k x k")
        if len(self.kernel_shape) != len(self.dims):
            raise InvalidArgument("KernelShape: order mismatch with tensor")
        self._Kc = _colmajor(K)
        self.device = device

    def k(self) -> int:
        return int(np.prod(self.kernel_shape))

    def apply(self, L) -> np.ndarray:
        L = _f64(L)
        if L.shape != self.dims:
            raise InvalidArgument("BasisConvolver: tensor dims mismatch")
        m, k = L.size, self.k()
        out = np.empty((k, m))
        check(lib().icnnm_cuda_conv_forward_ex(L.ndim, lptr(_dims(self.dims)), dptr(L),
                                               lptr(_dims(self.kernel_shape)), dptr(self._Kc),
                                               self.engine, self.device, dptr(out)))
        return out.T


def conv_adjoint(W, kernel_shape, dims, device: int = 0, engine: str = "ffma") -> np.ndarray:
    """conv_adjoint (conv_op.cpp:57-77): out[i] = sum_s W[(i+s) mod dims, s]."""
    dims = tuple(int(d) for d in dims)
    kernel_shape = tuple(int(d) for d in kernel_shape)
    W = np.asarray(W, dtype=np.float64)
    m, k = int(np.prod(dims)), int(np.prod(kernel_shape))
    if len(kernel_shape) != len(dims):
        raise InvalidArgument("KernelShape: order mismatch with tensor")
    if W.ndim != 2 or W.shape != (m, k):
        raise InvalidArgument("conv_adjoint: W shape mismatch with dims/kernel")
    Wc = np.ascontiguousarray(W.T)
    out = np.empty(dims)
    if engine not in ENGINES:
        raise InvalidArgument("unknown engine")
    check(lib().icnnm_cuda_conv_adjoint_ex(len(dims), lptr(_dims(dims)), lptr(_dims(kernel_shape)),
                                           dptr(Wc), ENGINES[engine], device, dptr(out)))
    return out


def prox_l21(W, tau: float, device: int = 0) -> np.ndarray:
    """prox_l21 (solver.cpp:42-50): column shrinkage."""
    W = np.asarray(W, dtype=np.float64)
    if tau < 0:
        raise InvalidArgument("prox_l21: tau must be >= 0")
    rows, cols = W.shape
    Wc = np.ascontiguousarray(W.T)
    Z = np.empty_like(Wc)
    check(lib().icnnm_cuda_prox_l21(rows, cols, dptr(Wc), float(tau), device, dptr(Z)))
    return Z.T


def conv_gram(L, kernel_shape, device: int = 0) -> np.ndarray:
    """conv_gram (spectral.cpp:54-81): A_k(L)^T A_k(L) via autocorrelation."""
    L = _f64(L)
    kernel_shape = tuple(int(d) for d in kernel_shape)
    k = int(np.prod(kernel_shape))
    G = np.empty((k, k))
    check(lib().icnnm_cuda_conv_gram(L.ndim, lptr(_dims(L.shape)), dptr(L),
                                     lptr(_dims(kernel_shape)), device, dptr(G)))
    return G.T.copy()


def learn_ensemble_basis(refs: Sequence[np.ndarray], kernel_shape, device: int = 0) -> EigenBasis:
    """learn_ensemble_basis (spectral.cpp:133-161): GPU Gram, host eigensolve."""
    if len(refs) == 0:
        raise InvalidArgument("learn_ensemble_basis: empty reference list")
    refs = [_f64(r) for r in refs]
    dims = refs[0].shape
    for r in refs:
        if r.shape != dims:
            raise InvalidArgument("learn_ensemble_basis: dim mismatch among refs")
    kernel_shape = tuple(int(d) for d in kernel_shape)
    k = int(np.prod(kernel_shape))
    ptrs = (C.POINTER(C.c_double) * len(refs))(*[dptr(r) for r in refs])
    Kc = np.empty((k, k))
    ev = np.empty(k)
    deg = C.c_int(0)
    check(lib().icnnm_cuda_learn_basis(len(refs), len(dims), lptr(_dims(dims)), ptrs,
                                       lptr(_dims(kernel_shape)), device, dptr(Kc), dptr(ev),
                                       C.byref(deg)))
    return EigenBasis(kernel_shape, Kc.T.copy(), ev, bool(deg.value))


def objective_icnnm(L, M_obs, mask, basis: EigenBasis, lam: float, device: int = 0) -> float:
    """objective_icnnm (solver.cpp:172-187)."""
    L, M, W = _f64(L), _f64(M_obs), _f64(mask)
    if L.shape != M.shape or W.shape != L.shape:
        raise InvalidArgument("objective_icnnm: dim mismatch")
    _check_basis_shape(basis, L.shape)
    out = C.c_double()
    check(lib().icnnm_cuda_objective(L.ndim, lptr(_dims(L.shape)), dptr(L), dptr(M), dptr(W),
                                     lptr(_dims(basis.kernel_shape)), dptr(_colmajor(basis.K)),
                                     float(lam), device, C.byref(out)))
    return out.value


def symeig(G) -> Tuple[np.ndarray, np.ndarray]:
    """Host eigensolver of learn_basis: (eigenvalues desc, eigenvectors cols)."""
    G = _f64(G)
    n = G.shape[0]
    ev = np.empty(n)
    V = np.empty((n, n))
    check(lib().icnnm_host_symeig(n, dptr(np.ascontiguousarray(G.T)), dptr(ev), dptr(V)))
    return ev, V.T.copy()


# --------------------------------------------------------------------------
# Sharded solve (H slabs; NCCL across processes)
# --------------------------------------------------------------------------
def dist_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().icnnm_dist_unique_id(buf))
    return buf.raw


def shard_plan(H: int, G: int, kh: int, g: int) -> Tuple[int, int]:
    s = C.c_int64()
    c = C.c_int64()
    check(lib().icnnm_shard_plan(int(H), int(G), int(kh), int(g), C.byref(s), C.byref(c)))
    return s.value, c.value


def sharded_solve(M_obs, mask, basis: EigenBasis, cfg: Optional[SolverConfig] = None,
                  local_slabs: int = 1, world: int = 1, rank: int = 0,
                  nccl_id: Optional[bytes] = None, device: int = 0):
    """H-sharded solve; returns (row0, L_rows (nrows, ...), report)."""
    cfg = cfg or SolverConfig()
    M, W = _f64(M_obs), _f64(mask)
    if M.shape != W.shape:
        raise InvalidArgument("solve: mask dims != observation dims")
    _check_basis_shape(basis, M.shape)
    c = cfg.to_c()
    out = np.empty_like(M)
    r0 = C.c_int64()
    nr = C.c_int64()
    rep, obj, res, lc = _report_buffers(max(int(cfg.max_iters), 1))
    idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    check(lib().icnnm_sharded_solve(M.ndim, lptr(_dims(M.shape)), dptr(M), dptr(W),
                                    lptr(_dims(basis.kernel_shape)), dptr(_colmajor(basis.K)),
                                    C.byref(c), int(local_slabs), int(world), int(rank), idbuf,
                                    device, dptr(out), C.byref(r0), C.byref(nr), C.byref(rep)))
    H = M.shape[0] if M.ndim == 3 else 1
    inner = M.size // H
    rows = out.reshape(-1)[: nr.value * inner].reshape((nr.value,) + M.shape[1:])
    return r0.value, rows.copy(), _report_from_c(rep, obj, res, lc)


def sharded_rows(dims, kernel_shape, local_slabs: int = 1, world: int = 1, rank: int = 0):
    """(row0, nrows): the H rows a rank owns in the sharded solve."""
    r0 = C.c_int64()
    nr = C.c_int64()
    check(lib().icnnm_sharded_rows(len(dims), lptr(_dims(dims)), lptr(_dims(kernel_shape)),
                                   int(local_slabs), int(world), int(rank), C.byref(r0),
                                   C.byref(nr)))
    return r0.value, nr.value


def sharded_solve_local(dims, M_rows, mask_rows, basis: EigenBasis,
                        cfg: Optional[SolverConfig] = None, local_slabs: int = 1,
                        world: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None,
                        device: int = 0):
    """H-sharded solve from slab-local inputs: M_rows / mask_rows are this
    rank's rows (sharded_rows) of the full `dims` tensor; no process holds
    the whole tensor.  Returns (L_rows, report)."""
    cfg = cfg or SolverConfig()
    dims = tuple(int(d) for d in dims)
    M, W = _f64(M_rows), _f64(mask_rows)
    if M.shape != W.shape:
        raise InvalidArgument("solve: mask dims != observation dims")
    _check_basis_shape(basis, dims)
    r0, nr = sharded_rows(dims, basis.kernel_shape, local_slabs, world, rank)
    if M.shape != (nr,) + dims[1:]:
        raise InvalidArgument(f"sharded solve: rank {rank} owns rows [{r0}, {r0 + nr}) -> "
                              f"inputs of shape {(nr,) + dims[1:]}, got {M.shape}")
    c = cfg.to_c()
    out = np.empty_like(M)
    rep, obj, res, lc = _report_buffers(max(int(cfg.max_iters), 1))
    idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
    check(lib().icnnm_sharded_solve_local(len(dims), lptr(_dims(dims)), r0, nr, dptr(M), dptr(W),
                                          lptr(_dims(basis.kernel_shape)),
                                          dptr(_colmajor(basis.K)), C.byref(c),
                                          int(local_slabs), int(world), int(rank), idbuf,
                                          device, dptr(out), C.byref(rep)))
    return out, _report_from_c(rep, obj, res, lc)


def cnnm_solve(M_obs, mask, kernel_shape, cfg: Optional[SolverConfig] = None,
               device: int = 0) -> Tuple[np.ndarray, SolveReport]:
    """cnnm_solve (solver.cpp:161-170): the CNNM baseline (K = I, SVT
    Z-update) on the GPU in fp64."""
    cfg = cfg or SolverConfig()
    M, W = _f64(M_obs), _f64(mask)
    if M.shape != W.shape:
        raise InvalidArgument("solve: mask dims != observation dims")
    kernel_shape = tuple(int(d) for d in kernel_shape)
    if len(kernel_shape) != M.ndim:
        raise InvalidArgument("KernelShape: order mismatch with tensor")
    c = cfg.to_c()
    out = np.empty_like(M)
    rep, obj, res, lc = _report_buffers(max(int(cfg.max_iters), 1))
    check(lib().icnnm_cuda_cnnm_solve(M.ndim, lptr(_dims(M.shape)), dptr(M), dptr(W),
                                      lptr(_dims(kernel_shape)), C.byref(c), device, dptr(out),
                                      C.byref(rep)))
    return out, _report_from_c(rep, obj, res, lc)


def device_count() -> int:
    return int(lib().icnnm_device_count())


def empty_cache() -> None:
    """Return the library's cached device blocks to the driver."""
    check(lib().icnnm_empty_cache())


def probe_ffma_tflops(device: int = 0) -> float:
    out = C.c_double()
    check(lib().icnnm_probe_ffma_tflops(device, C.byref(out)))
    return out.value


def probe_dfma_tflops(device: int = 0) -> float:
    out = C.c_double()
    check(lib().icnnm_probe_dfma_tflops(device, C.byref(out)))
    return out.value
