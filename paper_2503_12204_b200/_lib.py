"""ctypes binding of the C-ABI in include/d4orm_cuda.h (libd4orm_b200.so).

The product path has no fallback: if the sm_100a library is missing or no GPU
is visible, every call raises.  PyTorch is not needed on this path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("D4ORM_LIB", str(_PKG / "libd4orm_b200.so")))

D4ORM_OK, D4ORM_E_INVALID, D4ORM_E_RUNTIME, D4ORM_E_CUDA, D4ORM_E_NCCL, D4ORM_E_UNSUPPORTED = range(6)
PREC_F32, PREC_F64 = 0, 1
NOISE_PHILOX, NOISE_HOST = 0, 1
FROM_SCRATCH, DEFORMATION = 0, 1

# every symbol include/d4orm_cuda.h declares (checked by tests on CPU)
EXPORTS = (
    "d4orm_cuda_create", "d4orm_cuda_nccl_id", "d4orm_cuda_destroy", "d4orm_cuda_last_error",
    "d4orm_cuda_version", "d4orm_cuda_set_problem", "d4orm_cuda_set_options", "d4orm_cuda_set_noise_fn",
    "d4orm_cuda_run_denoising", "d4orm_cuda_denoise_step", "d4orm_cuda_rollout_fitness",
    "d4orm_cuda_score_weights", "d4orm_cuda_philox_noise", "d4orm_cuda_bench_steps",
    "d4orm_cuda_launches_per_step", "d4orm_cuda_solve", "d4orm_cuda_mppi_solve", "d4orm_cuda_cem_solve",
    "d4orm_cuda_weighted_mean", "d4orm_cuda_set_exchange_fn",
)


class Problem_C(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("dx", C.c_int), ("du", C.c_int), ("pdim", C.c_int),
        ("robots", C.c_int), ("horizon", C.c_int), ("dt", C.c_double),
        ("lower", C.c_double * 3), ("upper", C.c_double * 3),
        ("starts", C.POINTER(C.c_double)), ("goals", C.POINTER(C.c_double)),
        ("n_obstacles", C.c_int), ("obs_centers", C.POINTER(C.c_double)), ("obs_radii", C.POINTER(C.c_double)),
        ("w_t", C.c_double), ("epsilon", C.c_double), ("robot_radius", C.c_double),
        ("goal_tolerance", C.c_double), ("obstacle_weight", C.c_double), ("effort_weight", C.c_double),
    ]


class DenoiserConfig_C(C.Structure):
    _fields_ = [("steps", C.c_int), ("batch", C.c_int64), ("lambda_", C.c_double),
                ("alpha_bar_final", C.c_double), ("seed", C.c_uint64), ("mode", C.c_int),
                ("alpha_bar", C.POINTER(C.c_double))]


class TraceRec_C(C.Structure):
    _fields_ = [("step", C.c_int), ("best_reward", C.c_double), ("mean_reward", C.c_double),
                ("weight_entropy", C.c_double)]


ITER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_uint64)


class SolveConfig_C(C.Structure):
    _fields_ = [("max_iterations", C.c_int), ("stop_on_success", C.c_int), ("deadline_seconds", C.c_double),
                ("denoiser", DenoiserConfig_C), ("on_iteration", ITER_FN), ("on_iteration_user", C.c_void_p)]


class IterationRec_C(C.Structure):
    _fields_ = [("reward", C.c_double), ("objective", C.c_double), ("success", C.c_int), ("elapsed", C.c_double)]


class MppiConfig_C(C.Structure):
    _fields_ = [("batch", C.c_int64), ("lambda_", C.c_double), ("sigma", C.c_double), ("iterations", C.c_int),
                ("seed", C.c_uint64), ("stop_on_success", C.c_int), ("deadline_seconds", C.c_double)]


class CemConfig_C(C.Structure):
    _fields_ = [("batch", C.c_int64), ("elite_fraction", C.c_double), ("initial_std", C.c_double),
                ("min_std", C.c_double), ("iterations", C.c_int), ("seed", C.c_uint64),
                ("stop_on_success", C.c_int), ("deadline_seconds", C.c_double)]


NOISE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.POINTER(C.c_double))
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)

_lib = None


def lib() -> C.CDLL:
    """Load libd4orm_b200.so; raise loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2503_12204_b200.build` "
                          "(the sm_100a CUDA library is the only implementation; there is no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, i32, i64, dp = C.c_void_p, C.c_int, C.c_int64, C.POINTER(C.c_double)
    L.d4orm_cuda_create.argtypes = [i32, i32, i32, vp, C.POINTER(vp)]
    L.d4orm_cuda_nccl_id.argtypes = [vp]
    L.d4orm_cuda_destroy.argtypes = [vp]
    L.d4orm_cuda_destroy.restype = None
    L.d4orm_cuda_last_error.argtypes = [vp]
    L.d4orm_cuda_last_error.restype = C.c_char_p
    L.d4orm_cuda_version.restype = C.c_char_p
    L.d4orm_cuda_set_problem.argtypes = [vp, C.POINTER(Problem_C)]
    L.d4orm_cuda_set_options.argtypes = [vp, i32, i32, i32]
    L.d4orm_cuda_set_noise_fn.argtypes = [vp, NOISE_FN, vp]
    L.d4orm_cuda_set_exchange_fn.argtypes = [vp, EXCHANGE_FN, vp]
    L.d4orm_cuda_run_denoising.argtypes = [vp, dp, C.POINTER(DenoiserConfig_C), dp, C.POINTER(TraceRec_C)]
    L.d4orm_cuda_denoise_step.argtypes = [vp, dp, dp, dp, i32, C.POINTER(DenoiserConfig_C), dp, dp, dp,
                                          C.POINTER(TraceRec_C)]
    L.d4orm_cuda_rollout_fitness.argtypes = [vp, dp, i64, dp, dp, dp, C.POINTER(C.c_int64)]
    L.d4orm_cuda_score_weights.argtypes = [vp, dp, i64, C.c_double, dp, dp]
    L.d4orm_cuda_philox_noise.argtypes = [vp, C.c_uint64, i32, i64, i64, C.POINTER(C.c_float)]
    L.d4orm_cuda_weighted_mean.argtypes = [vp, dp, dp, i64, i64, dp]
    L.d4orm_cuda_bench_steps.argtypes = [vp, dp, C.POINTER(DenoiserConfig_C), i32, i32, dp, dp]
    L.d4orm_cuda_launches_per_step.argtypes = [vp]
    L.d4orm_cuda_fitness_path.argtypes = [vp]
    L.d4orm_cuda_k5_regen.argtypes = [vp]
    L.d4orm_cuda_last_fit_kernel.argtypes = [vp]
    L.d4orm_cuda_last_w32.argtypes = [vp, C.POINTER(C.c_float), i64]
    L.d4orm_cuda_mppi_solve.argtypes = [vp, C.POINTER(MppiConfig_C), dp, dp, C.POINTER(IterationRec_C),
                                        C.POINTER(i32), dp, C.POINTER(i32)]
    L.d4orm_cuda_cem_solve.argtypes = [vp, C.POINTER(CemConfig_C), dp, dp, C.POINTER(IterationRec_C),
                                       C.POINTER(i32), dp, C.POINTER(i32)]
    L.d4orm_cuda_solve.argtypes = [vp, C.POINTER(SolveConfig_C), dp, dp, C.POINTER(IterationRec_C),
                                   C.POINTER(TraceRec_C), C.POINTER(i32), dp, C.POINTER(i32)]
    _lib = L
    return L


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


class D4ormError(RuntimeError):
    """Error raised by the CUDA path; `code` is the C-ABI status."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(D4ormError, ValueError):
    """std::invalid_argument in the reference."""


def raise_for(code: int, msg: str):
    if code == D4ORM_OK:
        return
    if code == D4ORM_E_INVALID:
        raise InvalidArgument(code, msg)
    raise D4ormError(code, msg)
