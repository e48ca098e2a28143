"""BASELINE.json workloads: seeded synthetic inputs.

TEST / BENCH INPUT INFRASTRUCTURE, not the product.  The generator is host
C++ (std::mt19937_64, libstdc++ distributions) in its own library,
``synthgen/libicnnm_synth.so`` (include/icnnm_synth.h), so that the oracle
and the reference arm of bench.py generate inputs without loading the
product library ``libicnnm_b200.so``; this module pins the recipe of each
config.  No
public dataset is involved: the paper's datasets (Kodak, UCF-101, ...) are
not available, and BASELINE.json defines these synthetic stand-ins.

Pinned generator details (open in BASELINE.json, fixed here):
  * sinusoid amplitude U[0.5, 1.5], integer frequencies 0..4 per axis,
    phase U[0, 2pi); blobs: amplitude U[0.5, 1.5], sigma 4 px, start
    U[0,H) x U[0,W), direction U[0, 2pi), 1 px/frame, periodic;
  * min-max scaled to [0, 1], then texture noise N(0, sigma^2) (cfg 2, 3);
  * seeds: target 1000 + 10*cfg (+b for batch tensor b), training tensors
    2000 + 100*cfg + i, mask 3000 + cfg.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libicnnm_synth.so")
_dp = C.POINTER(C.c_double)
_lp = C.POINTER(C.c_int64)
_SIG = {
    "icnnm_synth_video": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int,
                                    C.c_double, C.c_double, C.c_uint64, _dp]),
    "icnnm_synth_mask": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_double,
                                   C.c_int, C.c_uint64, _dp]),
    "icnnm_rng_create": (C.c_void_p, [C.c_uint64]),
    "icnnm_rng_destroy": (None, [C.c_void_p]),
    "icnnm_rng_uniform": (None, [C.c_void_p, C.c_double, C.c_double, C.c_int64, _dp]),
    "icnnm_rng_uniform_int": (None, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, _lp]),
    "icnnm_rng_normal": (None, [C.c_void_p, C.c_double, C.c_double, C.c_int64, _dp]),
    "icnnm_reference_bernoulli_mask": (C.c_int, [C.c_int64, C.c_double, C.c_uint64, _dp]),
}
_lib = None


def lib():
    """The generator library (built by `make -C synthgen`)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is not built; run `make -C synthgen`")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise ValueError("synthgen: invalid generator arguments")


def dptr(a):
    return a.ctypes.data_as(_dp)


def lptr(a):
    return a.ctypes.data_as(_lp)


MASK_IID, MASK_EXACT, MASK_T_FRAMES, MASK_T_PREFIX, MASK_IID_BOXES = 0, 1, 2, 3, 4


def synth_video(H: int, W: int, T: int, n_sin: int, n_blob: int, seed: int,
                blob_sigma: float = 4.0, noise_sigma: float = 0.0) -> np.ndarray:
    out = np.empty((H, W, T))
    check(lib().icnnm_synth_video(H, W, T, n_sin, n_blob, blob_sigma, noise_sigma,
                                  C.c_uint64(seed), dptr(out)))
    return out


def synth_mask(H: int, W: int, T: int, kind: int, rate: float, seed: int,
               n_boxes: int = 0) -> np.ndarray:
    out = np.empty((H, W, T))
    check(lib().icnnm_synth_mask(H, W, T, kind, float(rate), n_boxes, C.c_uint64(seed),
                                 dptr(out)))
    return out


def reference_bernoulli_mask(dims, rate: float, seed: int) -> np.ndarray:
    """generate_mask(dims, {kBernoulli, rate, seed}) of mask.cpp:49-59."""
    out = np.empty(tuple(dims))
    check(lib().icnnm_reference_bernoulli_mask(out.size, float(rate), C.c_uint64(seed),
                                               dptr(out)))
    return out


class Rng:
    """A std::mt19937_64 stream with libstdc++ distributions, for rebuilding
    the reference tests' inputs (proj/tests/test_util.hpp:27-49)."""

    def __init__(self, seed: int):
        self._h = lib().icnnm_rng_create(C.c_uint64(seed))

    def uniform(self, lo: float, hi: float, n: int) -> np.ndarray:
        out = np.empty(n)
        lib().icnnm_rng_uniform(self._h, lo, hi, n, dptr(out))
        return out

    def uniform_int(self, lo: int, hi: int, n: int = 1) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        lib().icnnm_rng_uniform_int(self._h, lo, hi, n, lptr(out))
        return out

    def normal(self, mean: float, sd: float, n: int) -> np.ndarray:
        out = np.empty(n)
        lib().icnnm_rng_normal(self._h, mean, sd, n, dptr(out))
        return out

    # test_util.hpp helpers
    def random_tensor(self, dims) -> np.ndarray:
        dims = tuple(int(d) for d in dims)
        return self.uniform(-1.0, 1.0, int(np.prod(dims))).reshape(dims)

    def random_dims(self, max_order: int = 3, max_dim: int = 6) -> Tuple[int, ...]:
        order = int(self.uniform_int(1, max_order)[0])
        return tuple(int(self.uniform_int(2, max_dim)[0]) for _ in range(order))

    def random_kernel_dims(self, dims) -> Tuple[int, ...]:
        return tuple(int(self.uniform_int(1, d)[0]) for d in dims)

    def close(self):
        if self._h:
            lib().icnnm_rng_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclasses.dataclass
class Workload:
    cfg: int
    dims: Tuple[int, int, int]
    kernel: Tuple[int, int, int]
    iters: int
    batch: int
    n_sin: int
    n_blob: int
    noise: float
    n_train: int
    mask_kind: int
    mask_rate: float
    n_boxes: int = 0

    @property
    def m(self) -> int:
        return int(np.prod(self.dims))

    @property
    def k(self) -> int:
        return int(np.prod(self.kernel))

    def target(self, b: int = 0) -> np.ndarray:
        H, W, T = self.dims
        return synth_video(H, W, T, self.n_sin, self.n_blob, 1000 + 10 * self.cfg + b,
                           4.0, self.noise)

    def training(self) -> List[np.ndarray]:
        H, W, T = self.dims
        return [synth_video(H, W, T, self.n_sin, self.n_blob, 2000 + 100 * self.cfg + i,
                            4.0, self.noise) for i in range(self.n_train)]

    def mask(self) -> np.ndarray:
        H, W, T = self.dims
        return synth_mask(H, W, T, self.mask_kind, self.mask_rate, 3000 + self.cfg,
                          self.n_boxes)


# BASELINE.json:configs, in order.
WORKLOADS = {
    1: Workload(1, (32, 32, 8), (5, 5, 3), 200, 1, 8, 1, 0.0, 4, MASK_IID, 0.5),
    2: Workload(2, (128, 128, 32), (9, 9, 5), 300, 1, 16, 3, 0.01, 8, MASK_EXACT, 0.2),
    3: Workload(3, (256, 256, 48), (13, 13, 7), 300, 1, 16, 3, 0.01, 8, MASK_T_PREFIX, 40),
    4: Workload(4, (128, 128, 32), (7, 7, 5), 200, 64, 16, 3, 0.0, 8, MASK_T_FRAMES, 0.0),
    5: Workload(5, (1024, 1024, 64), (9, 9, 9), 100, 1, 32, 8, 0.0, 8, MASK_IID_BOXES, 0.3,
                200),
}


def scaled(w: Workload, dims: Tuple[int, int, int], iters: Optional[int] = None,
           n_train: Optional[int] = None) -> Workload:
    """Same recipe at smaller dims (parity cases for the large configs)."""
    return dataclasses.replace(w, dims=tuple(dims), iters=iters or w.iters,
                               n_train=n_train or w.n_train)


def psnr(ref: np.ndarray, est: np.ndarray, peak: float = 1.0) -> float:
    """psnr (metrics.cpp:34-38)."""
    e = float(np.mean((np.asarray(ref) - np.asarray(est)) ** 2))
    if e == 0:
        return float("inf")
    return 10.0 * np.log10(peak * peak / e)
