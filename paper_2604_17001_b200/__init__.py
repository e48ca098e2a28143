"""B200-native ICNNM hot path (arXiv 2604.17001) behind the reference's API.

See DESIGN.md.  The compute lives in ``libicnnm_b200.so`` (hand-written
sm_100a kernels + C++ host driver, C ABI in include/icnnm_b200.h); this
package is the Python mirror of the reference's solver/operator interface.
"""
from ._lib import IcnnmError, InvalidArgument, CudaError, LIB_PATH, lib
from .api import (SolverConfig, SolveReport, EigenBasis, Solver, BasisConvolver,
                  icnnm_solve, icnnm_solve_batch, cnnm_solve, learn_ensemble_basis, conv_adjoint, prox_l21, conv_gram,
                  objective_icnnm, symeig, sharded_solve, sharded_solve_local, sharded_rows, shard_plan, dist_unique_id,
                  device_count, empty_cache, probe_ffma_tflops, probe_dfma_tflops)
from . import synth, analysis

__all__ = [
    "IcnnmError", "InvalidArgument", "CudaError", "LIB_PATH", "lib",
    "SolverConfig", "SolveReport", "EigenBasis", "Solver", "BasisConvolver",
    "icnnm_solve", "icnnm_solve_batch", "cnnm_solve", "learn_ensemble_basis", "conv_adjoint", "prox_l21", "conv_gram",
    "objective_icnnm", "symeig", "sharded_solve", "sharded_solve_local", "sharded_rows", "shard_plan", "dist_unique_id",
    "device_count", "empty_cache", "probe_ffma_tflops", "probe_dfma_tflops", "synth", "analysis",
]
