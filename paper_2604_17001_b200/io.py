"""Reference file formats through the C ABI (tensor_io.cpp:86-128,
report_io.cpp:39-68): TNSR tensors, EBAS bases, SolverConfig JSON."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import SolverConfigC, check_io, dptr, lib, lptr
from .api import EigenBasis


def write_tnsr(path: str, t) -> None:
    t = np.ascontiguousarray(np.asarray(t, dtype=np.float64))
    check_io(lib().icnnm_write_tnsr(path.encode(), t.ndim, lptr(np.array(t.shape, np.int64)),
                                    dptr(t)))


def read_tnsr(path: str) -> np.ndarray:
    order = C.c_int()
    dims = np.zeros(16, np.int64)
    check_io(lib().icnnm_read_tnsr(path.encode(), C.byref(order), lptr(dims), None))
    out = np.empty(tuple(dims[: order.value]))
    check_io(lib().icnnm_read_tnsr(path.encode(), C.byref(order), lptr(dims), dptr(out)))
    return out


def write_ebas(path: str, basis: EigenBasis) -> None:
    kd = np.array(basis.kernel_shape, np.int64)
    Kc = np.ascontiguousarray(np.asarray(basis.K, np.float64).T)
    ev = np.ascontiguousarray(np.asarray(basis.eigenvalues, np.float64))
    check_io(lib().icnnm_write_ebas(path.encode(), len(kd), lptr(kd), dptr(ev), dptr(Kc)))


def read_ebas(path: str) -> EigenBasis:
    order = C.c_int()
    kd = np.zeros(16, np.int64)
    check_io(lib().icnnm_read_ebas(path.encode(), C.byref(order), lptr(kd), None, None))
    ks = tuple(int(x) for x in kd[: order.value])
    k = int(np.prod(ks))
    ev = np.empty(k)
    Kc = np.empty((k, k))
    check_io(lib().icnnm_read_ebas(path.encode(), C.byref(order), lptr(kd), dptr(ev), dptr(Kc)))
    return EigenBasis(ks, Kc.T.copy(), ev)


def config_from_json(text: str) -> SolverConfigC:
    c = SolverConfigC()
    check_io(lib().icnnm_config_from_json(text.encode(), C.byref(c)))
    return c
