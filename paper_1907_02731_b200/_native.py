"""ctypes binding of the C ABI in include/sfseg_cuda.h (libsfseg_cuda.so).

The library is built in-tree (paper_1907_02731_b200/lib/) by
``__graft_entry__.build()``. There is no fallback: if the shared object is
missing or no sm_100 device is present every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "lib"
CUDA_LIB = LIB_DIR / "libsfseg_cuda.so"
SYNTH_LIB = LIB_DIR / "libsfseg_synth.so"

# status codes (sfseg_cuda.h) -> exception classes named after errors.hpp:17-68
SFSEG_OK = 0
SFSEG_ERR_PARAMETER = 1
SFSEG_ERR_SHAPE = 2
SFSEG_ERR_VALIDATION = 3
SFSEG_ERR_DEGENERATE = 4
SFSEG_ERR_CAPACITY = 5
SFSEG_ERR_CUDA = 6
SFSEG_ERR_STATE = 7
SFSEG_ERR_IO = 8
SFSEG_ERR_FORMAT = 9
SFSEG_ERR_CORRUPTION = 10
SFSEG_SHARD_EXPORT_BYTES = 176

SFSEG_ARITH_EXACT = 0
SFSEG_ARITH_FAST = 1
SFSEG_MEM_HOST = 0
SFSEG_MEM_DEVICE = 1
SFSEG_CONV_STEP, SFSEG_CONV_ANGLE = 0, 1  # enum sfseg_conv
SFSEG_AFFINITY_EXACT, SFSEG_AFFINITY_TAYLOR, SFSEG_AFFINITY_TAYLOR_CHANNEL_SUM = 0, 1, 2


class Error(RuntimeError):
    """sfseg::Error (errors.hpp:17-20)."""


class ParameterError(Error):
    pass


class ShapeError(Error):
    pass


class ValidationError(Error):
    pass


class DegenerateSolutionError(Error):
    pass


class CapacityError(Error):
    pass


class CudaError(Error):
    pass


class IoError(Error):
    pass


class FormatError(Error):
    pass


class CorruptionError(Error):
    pass


_EXC = {
    SFSEG_ERR_PARAMETER: ParameterError,
    SFSEG_ERR_SHAPE: ShapeError,
    SFSEG_ERR_VALIDATION: ValidationError,
    SFSEG_ERR_DEGENERATE: DegenerateSolutionError,
    SFSEG_ERR_CAPACITY: CapacityError,
    SFSEG_ERR_CUDA: CudaError,
    SFSEG_ERR_STATE: Error,
    SFSEG_ERR_IO: IoError,
    SFSEG_ERR_FORMAT: FormatError,
    SFSEG_ERR_CORRUPTION: CorruptionError,
}


class Params(C.Structure):
    """sfseg_params — mirrors SfsegConfig (engine.hpp:22-57)."""

    _fields_ = [
        ("alpha", C.c_double),
        ("p", C.c_double),
        ("radii", C.c_int32 * 3),
        ("sigmas", C.c_double * 3),
        ("iterations", C.c_int32),
        ("temporal_window", C.c_int32),
        ("binarize_start", C.c_int32),
        ("sigmoid_slope0", C.c_double),
        ("slope_growth", C.c_double),
        ("threshold_frac", C.c_double),
        ("final_threshold", C.c_double),
        ("allow_negative_affinity", C.c_int32),
        ("arith", C.c_int32),
    ]


class IterRecord(C.Structure):
    _fields_ = [
        ("iter", C.c_int32),
        ("l2_norm_pre_normalize", C.c_double),
        ("angle_deg", C.c_double),
        ("iou", C.c_double),
        ("wall_time_s", C.c_double),
    ]


class Timing(C.Structure):
    _fields_ = [
        ("solve_ms", C.c_double),
        ("step_kernel_ms", C.c_double),
        ("step_launches", C.c_int32),
        ("total_launches", C.c_int32),
        ("bytes_per_launch", C.c_double),
    ]


class ShardIO(C.Structure):
    _fields_ = [
        ("send_lo", C.c_void_p), ("send_hi", C.c_void_p),
        ("recv_lo", C.c_void_p), ("recv_hi", C.c_void_p),
        ("send_lo_bytes", C.c_uint64), ("send_hi_bytes", C.c_uint64),
        ("recv_lo_bytes", C.c_uint64), ("recv_hi_bytes", C.c_uint64),
        ("frame_sum", C.c_void_p), ("frame_max", C.c_void_p),
        ("out_frames", C.c_int32), ("halo", C.c_int32),
    ]


class Clip(C.Structure):
    """sfseg_clip — one entry of sfseg_run_batch (include/sfseg_cuda.h)."""

    _fields_ = [
        ("frames", C.c_uint32), ("height", C.c_uint32), ("width", C.c_uint32),
        ("channels", C.c_int32),
        ("unary", C.c_void_p), ("pairwise", C.c_void_p), ("x0", C.c_void_p),
        ("soft", C.c_void_p), ("mask", C.c_void_p), ("records", C.c_void_p),
        ("status", C.c_int32), ("worker", C.c_int32), ("wall_ms", C.c_double),
    ]


_lib = None

_P = C.c_void_p
_FP = C.POINTER(C.c_float)
_U32 = C.c_uint32
_I32 = C.c_int32

_SIGS = {
    "sfseg_params_default": (None, [C.POINTER(Params)]),
    "sfseg_params_validate": (C.c_int, [C.POINTER(Params)]),
    "sfseg_make_kernel": (C.c_int, [C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_double),
                                     C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "sfseg_last_error": (C.c_char_p, []),
    "sfseg_build_info": (C.c_char_p, []),
    "sfseg_ctx_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "sfseg_ctx_destroy": (C.c_int, [_P]),
    "sfseg_ctx_set_timing": (C.c_int, [_P, C.c_int]),
    "sfseg_ctx_set_tap_trim": (C.c_int, [_P, C.c_int]),
    "sfseg_effective_radii": (C.c_int, [C.POINTER(Params), C.POINTER(C.c_int32)]),
    "sfseg_ctx_get_timing": (C.c_int, [_P, C.POINTER(Timing)]),
    "sfseg_ctx_synchronize": (C.c_int, [_P]),
    "sfseg_ctx_kernel_time": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_int32)]),
    "sfseg_ctx_stream": (C.c_void_p, [_P]),
    "sfseg_load": (C.c_int, [_P, _U32, _U32, _U32, _I32, _P, _P, _P, _I32]),
    "sfseg_load_files": (C.c_int, [_P, C.c_char_p, _P, _I32, C.c_char_p]),
    "sfseg_affinity_matvec": (C.c_int, [_P, _U32, _U32, _U32, _I32, _P, _P, C.POINTER(Params), _I32,
                                        _P, _P, _I32]),
    "sfseg_affinity_power_iteration": (C.c_int, [_P, _U32, _U32, _U32, _I32, _P, _P,
                                                 C.POINTER(Params), _I32, _P, _I32, C.c_double, _P,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_int32), _I32]),
    "sfseg_solve": (C.c_int, [_P, C.POINTER(Params), _I32, _I32, C.POINTER(IterRecord)]),
    "sfseg_solve_until": (C.c_int, [_P, C.POINTER(Params), _I32, _I32, _I32, C.c_double,
                                    C.POINTER(C.c_int32), C.POINTER(IterRecord)]),
    "sfseg_download": (C.c_int, [_P, C.c_double, _P, _P, _I32]),
    "sfseg_metrics": (C.c_int, [_P, _P, _P, C.c_double, C.POINTER(C.c_double),
                                C.POINTER(C.c_double), _I32]),
    "sfseg_probe_fp32_peak": (C.c_int, [C.c_int, C.POINTER(C.c_double)]),
    "sfseg_unit_range": (C.c_int, [_P, _U32, _U32, _U32, _P, _P, _I32]),
    "sfseg_multi_create": (C.c_int, [C.c_int32, _P, C.POINTER(_P)]),
    "sfseg_multi_destroy": (C.c_int, [_P]),
    "sfseg_multi_size": (C.c_int, [_P]),
    "sfseg_multi_run": (C.c_int, [_P, _U32, _U32, _U32, _I32, _P, _P, _P, C.POINTER(Params), _P, _P,
                                  _P, _I32]),
    "sfseg_run": (C.c_int, [_P, _U32, _U32, _U32, _I32, _P, _P, _P, C.POINTER(Params), _P, _P,
                            C.POINTER(IterRecord), _I32]),
    "sfseg_run_batch": (C.c_int, [_P, _I32, C.POINTER(Clip), _I32, C.POINTER(Params), _I32]),
    "sfseg_step": (C.c_int, [_P, _U32, _U32, _U32, _I32, _P, _P, _P, C.POINTER(Params), _P, _I32]),
    "sfseg_step_channel": (C.c_int, [_P, _U32, _U32, _U32, _P, _P, _P, C.POINTER(Params), _P, _I32]),
    "sfseg_normalize_l2": (C.c_int, [_P, _U32, _U32, _U32, _P, _P, C.POINTER(C.c_double), _I32]),
    "sfseg_project_binary": (C.c_int, [_P, _U32, _U32, _U32, _P, _I32, C.POINTER(Params), _P, _I32]),
    "sfseg_threshold_final": (C.c_int, [_P, _U32, _U32, _U32, _P, C.c_double, _P, _I32]),
    "sfseg_convolve_separable": (C.c_int, [_P, _U32, _U32, _U32, _P, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_double), _P, _I32]),
    "sfseg_separable_convolution_count": (C.c_uint64, []),
    "sfseg_convolve_separable_taps": (C.c_int, [_P, _U32, _U32, _U32, _P, C.POINTER(C.c_int32),
                                                _P, _P, _P, _P, _I32]),
    "sfseg_convolve_direct_taps": (C.c_int, [_P, _U32, _U32, _U32, _P, C.POINTER(C.c_int32),
                                             _P, _P, _P, _P, _I32]),
    "sfseg_shard_load": (C.c_int, [_P, _U32, _U32, _U32, _I32, _I32, _I32, _I32, _P, _P, _P, _I32]),
    "sfseg_shard_step": (C.c_int, [_P, C.POINTER(Params), _I32, C.POINTER(ShardIO)]),
    "sfseg_shard_finalize": (C.c_int, [_P, C.POINTER(Params), _I32, _P, _P,
                                       C.POINTER(C.c_double), _I32]),
    "sfseg_shard_download": (C.c_int, [_P, C.c_double, _P, _P, _I32]),
    "sfseg_shard_norms": (C.c_int, [_P, _I32, C.POINTER(C.c_double)]),
    "sfseg_shard_export": (C.c_int, [_P, _I32, _P]),
    "sfseg_shard_set_peers": (C.c_int, [_P, _P, _P]),
    "sfseg_synth_generate_device": (C.c_int, [_P, _P, _P, _P, _P]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def load_library(path: os.PathLike | str | None = None) -> C.CDLL:
    """Loads libsfseg_cuda.so (raises if it was never built: no fallback)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # SFSEG_CUDA_LIB: another build of the same library (development aid for
    # comparing kernel variants; still the CUDA library, never a fallback)
    p = Path(path) if path else Path(os.environ.get("SFSEG_CUDA_LIB", CUDA_LIB))
    if not p.exists():
        raise CudaError(
            f"{p} is missing: run __graft_entry__.build() (nvcc, sm_100a); "
            "there is no CPU fallback")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def check(rc: int) -> None:
    if rc != SFSEG_OK:
        msg = load_library().sfseg_last_error().decode(errors="replace")
        raise _EXC.get(rc, Error)(msg or f"sfseg status {rc}")
