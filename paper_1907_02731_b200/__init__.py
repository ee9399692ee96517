"""B200-native (sm_100a) SFSeg power iteration.

A drop-in for the hot path of the reference SFSeg library (arxiv 1907.02731):
``sfseg::run`` and the engine entry points it is built from, re-implemented as
fused TMA-fed CUDA stencil kernels behind a C ABI (include/sfseg_cuda.h).
"""
from .engine import (CapacityError, Context, DegenerateSolutionError, Error, FeatureSet,
                     IterationRecord, KernelConfig, ParameterError, RunResult, RunTrace,
                     SeparableKernel3D, SfsegConfig, ShapeError, ValidationError,
                     convolve_separable, default_context, make_gaussian_kernel, normalize_l2,
                     project_binary, run, separable_convolution_count, sfseg_step,
                     sfseg_step_channel, threshold_final)

__all__ = [
    "CapacityError", "Context", "DegenerateSolutionError", "Error", "FeatureSet",
    "IterationRecord", "KernelConfig", "ParameterError", "RunResult", "RunTrace",
    "SeparableKernel3D", "SfsegConfig", "ShapeError", "ValidationError", "convolve_separable",
    "default_context", "make_gaussian_kernel", "normalize_l2", "project_binary", "run",
    "separable_convolution_count", "sfseg_step", "sfseg_step_channel", "threshold_final",
]
