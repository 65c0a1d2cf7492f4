"""d4orm-b200: B200-native denoise-step hot path of D4orm (arXiv 2503.12204).

The compute is the sm_100a library libd4orm_b200.so (C-ABI: include/d4orm_cuda.h);
this package is the host-side mirror of the reference planner interface.
"""
from ._lib import (DEFORMATION, FROM_SCRATCH, NOISE_HOST, NOISE_PHILOX, PREC_F32, PREC_F64, D4ormError,
                   InvalidArgument, lib)
from .planner import DenoiserConfig, GpuDenoiser, SolveResult, make_schedule
from .scenarios import (DIFFDRIVE, HOLO2D, HOLO2D_VEL, HOLO3D, HOLO3D_VEL, UNICYCLE, Problem, RunConfig,
                        antipodal_circle, antipodal_sphere, baseline_config, cube_corners, random_obstacles,
                        random_square, validate)

__all__ = [
    "DEFORMATION", "FROM_SCRATCH", "NOISE_HOST", "NOISE_PHILOX", "PREC_F32", "PREC_F64", "D4ormError",
    "InvalidArgument", "lib", "DenoiserConfig", "GpuDenoiser", "SolveResult", "make_schedule", "DIFFDRIVE", "HOLO2D",
    "HOLO2D_VEL", "HOLO3D", "HOLO3D_VEL", "UNICYCLE", "Problem", "RunConfig", "antipodal_circle",
    "antipodal_sphere", "baseline_config", "cube_corners", "random_obstacles", "random_square", "validate",
]
