"""Python mirror of the reference solve API (proj/include/sfseg/engine.hpp).

Same names, argument meaning and error behaviour as the C++ reference:

=====================  ===========================================
reference (C++)         here
=====================  ===========================================
SfsegConfig             SfsegConfig (engine.hpp:22-57)
KernelConfig            KernelConfig (conv3d.hpp:20-23)
sfseg_step_channel      sfseg_step_channel (engine.hpp:63-64)
sfseg_step              sfseg_step (engine.hpp:67-68)
normalize_l2            normalize_l2 (engine.hpp:72)
project_binary          project_binary (engine.hpp:78)
threshold_final         threshold_final (engine.hpp:82)
run                     run (engine.hpp:104-109)
make_gaussian_kernel    make_gaussian_kernel (conv3d.hpp:55-57)
convolve_separable      convolve_separable (conv3d.hpp:62-63)
=====================  ===========================================

Volumes are float32 arrays of shape (T, H, W) in the reference's linear order
(volume.hpp:32-36): numpy arrays (host memory) or CUDA torch tensors (device
memory, used in place). Every call goes through the C ABI in
include/sfseg_cuda.h to the sm_100a kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native as N
from ._native import (CapacityError, CorruptionError, DegenerateSolutionError, Error,
                      FormatError, IoError, ParameterError, ShapeError, ValidationError)

__all__ = [
    "KernelConfig", "SfsegConfig", "FeatureSet", "IterationRecord", "RunTrace", "RunResult",
    "SeparableKernel3D", "make_gaussian_kernel", "convolve_separable", "convolve_direct", "sfseg_step",
    "sfseg_step_channel", "normalize_l2", "project_binary", "threshold_final", "run",
    "run_once", "run_batch",
    "separable_convolution_count", "Context", "default_context", "Error", "ParameterError",
    "ShapeError", "ValidationError", "DegenerateSolutionError", "CapacityError", "IoError",
    "FormatError", "CorruptionError", "run_files", "volume_shape", "affinity_matvec",
    "power_iteration",
]

ARITH_EXACT = N.SFSEG_ARITH_EXACT
ARITH_FAST = N.SFSEG_ARITH_FAST


@dataclass
class KernelConfig:
    """Per-axis radii/sigmas, axis order (t, y, x) (conv3d.hpp:20-23)."""

    radii: tuple = (1, 3, 3)
    sigmas: tuple = (0.5, 1.5, 1.5)


@dataclass
class SfsegConfig:
    """Solver configuration; defaults of engine.hpp:22-49.

    ``arith`` selects the kernel arithmetic (not in the reference): "exact"
    reproduces the reference's rounding order bit for bit; "fast" uses fused
    multiply-adds (within the north-star tolerance). Default: $SFSEG_ARITH or
    "exact". ``threads`` is accepted and ignored, as on the GPU it has no
    meaning (README.md:174-189 makes results thread-count invariant).
    """

    alpha: float = 1.0
    p: float = 0.1
    kernel: KernelConfig = field(default_factory=KernelConfig)
    iterations: int = 5
    temporal_window: int = -1
    binarize_start: int = 3
    sigmoid_slope0: float = 10.0
    slope_growth: float = 2.0
    threshold_frac: float = 0.5
    final_threshold: float = 0.5
    allow_negative_affinity: bool = False
    threads: int = 0
    arith: str = field(default_factory=lambda: os.environ.get("SFSEG_ARITH", "exact"))

    def resolved_temporal_window(self) -> int:
        return self.kernel.radii[0] if self.temporal_window < 0 else self.temporal_window

    def to_params(self) -> N.Params:
        p = N.Params()
        p.alpha = float(self.alpha)
        p.p = float(self.p)
        for a in range(3):
            p.radii[a] = int(self.kernel.radii[a])
            p.sigmas[a] = float(self.kernel.sigmas[a])
        p.iterations = int(self.iterations)
        p.temporal_window = int(self.temporal_window)
        p.binarize_start = int(self.binarize_start)
        p.sigmoid_slope0 = float(self.sigmoid_slope0)
        p.slope_growth = float(self.slope_growth)
        p.threshold_frac = float(self.threshold_frac)
        p.final_threshold = float(self.final_threshold)
        p.allow_negative_affinity = int(bool(self.allow_negative_affinity))
        if self.arith not in ("exact", "fast"):
            raise ParameterError("arith must be 'exact' or 'fast'")
        p.arith = ARITH_EXACT if self.arith == "exact" else ARITH_FAST
        return p

    def validate(self) -> None:
        """SfsegConfig::validate (engine.cpp:21-42); raises ParameterError."""
        lib = N.load_library()
        p = self.to_params()
        N.check(lib.sfseg_params_validate(C.byref(p)))


@dataclass
class FeatureSet:
    """Unary S plus >= 1 pairwise channels, all (T, H, W) (volume.hpp:90-96)."""

    unary: object
    pairwise: list

    def shape(self):
        return tuple(self.unary.shape)


@dataclass
class IterationRecord:
    iter: int
    l2_norm_pre_normalize: float
    angle_deg: Optional[float] = None
    iou: Optional[float] = None
    wall_time_s: float = 0.0


@dataclass
class RunTrace:
    iterations: list = field(default_factory=list)


@dataclass
class RunResult:
    soft: np.ndarray
    mask: np.ndarray
    trace: RunTrace
    worker: int = 0       # run_batch: index of the context that ran the clip
    wall_ms: float = 0.0  # run_batch: host time of the clip's load + solve + download


@dataclass
class SeparableKernel3D:
    taps_t: np.ndarray
    taps_y: np.ndarray
    taps_x: np.ndarray
    radii: tuple
    sigmas: tuple

    def tap_count(self) -> int:
        return len(self.taps_t) + len(self.taps_y) + len(self.taps_x)


# ---------------------------------------------------------------------------
class Context:
    """One CUDA device + stream + resident buffers (sfseg_ctx)."""

    def __init__(self, device: int = 0):
        self._lib = N.load_library()
        h = C.c_void_p()
        N.check(self._lib.sfseg_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device
        # re-entrant: an IterationObserver may call the engine functions on
        # the same context from inside run(); the library runs those on the
        # context's scratch buffers, never on the resident problem
        self.lock = threading.RLock()

    def close(self) -> None:
        if self.handle:
            self._lib.sfseg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, on: bool) -> None:
        N.check(self._lib.sfseg_ctx_set_timing(self.handle, int(on)))

    def set_tap_trim(self, on: bool) -> None:
        """FAST arithmetic only, off by default: drop the outermost taps that
        are at most 2^-24 of their axis's largest tap and run the kernel of the
        remaining support (sfseg_ctx_set_tap_trim, include/sfseg_cuda.h)."""
        N.check(self._lib.sfseg_ctx_set_tap_trim(self.handle, int(on)))

    def timing(self) -> N.Timing:
        t = N.Timing()
        N.check(self._lib.sfseg_ctx_get_timing(self.handle, C.byref(t)))
        return t

    def synchronize(self) -> None:
        N.check(self._lib.sfseg_ctx_synchronize(self.handle))


_ctx_lock = threading.Lock()
_contexts: dict = {}


def default_context(device: Optional[int] = None) -> Context:
    if device is None:
        device = int(os.environ.get("SFSEG_DEVICE", "0"))
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def _is_torch_cuda(a) -> bool:
    return hasattr(a, "is_cuda") and bool(getattr(a, "is_cuda"))


class _Buf:
    """A volume argument as (pointer, mem kind), keeping host copies alive."""

    def __init__(self, a, shape=None, writable=False, dtype=np.float32):
        if _is_torch_cuda(a):
            import torch

            want = torch.float32 if dtype == np.float32 else torch.uint8
            if a.dtype != want or not a.is_contiguous():
                raise ValidationError("device volumes must be contiguous " + str(want))
            self.arr = a
            self.ptr = C.c_void_p(a.data_ptr())
            self.mem = N.SFSEG_MEM_DEVICE
            self.shape = tuple(a.shape)
        else:
            arr = np.asarray(a)
            if arr.dtype != dtype or not arr.flags.c_contiguous:
                if writable:
                    raise ValidationError("output buffer must be a contiguous %s array" % dtype)
                arr = np.ascontiguousarray(arr, dtype=dtype)
            self.arr = arr
            self.ptr = C.c_void_p(arr.ctypes.data)
            self.mem = N.SFSEG_MEM_HOST
            self.shape = tuple(arr.shape)
        if shape is not None and self.shape != tuple(shape):
            raise ShapeError("shape mismatch: %s vs %s" % (self.shape, tuple(shape)))


def _shape3(shape) -> tuple:
    if len(shape) != 3:
        raise ShapeError("volumes are (T, H, W)")
    return tuple(int(s) for s in shape)


def _empty_like(buf: _Buf, dtype=np.float32):
    if buf.mem == N.SFSEG_MEM_DEVICE:
        import torch

        return torch.empty(buf.shape, dtype=torch.float32 if dtype == np.float32 else torch.uint8,
                           device=buf.arr.device)
    return np.empty(buf.shape, dtype=dtype)


def _same_mem(bufs: Sequence[_Buf]) -> int:
    kinds = {b.mem for b in bufs}
    if len(kinds) != 1:
        raise ValidationError("mixing host and device volumes in one call")
    return kinds.pop()


# ---------------------------------------------------------------------------
def effective_radii(cfg: "SfsegConfig") -> tuple:
    """Radii a tap-trimmed FAST step runs for cfg's kernel (Context.set_tap_trim);
    equal to cfg's radii when every tap is above fp32 resolution."""
    out = (C.c_int32 * 3)()
    q = cfg.to_params()
    N.check(N.load_library().sfseg_effective_radii(C.byref(q), out))
    return tuple(int(v) for v in out)


def make_gaussian_kernel(sigmas, radii) -> SeparableKernel3D:
    """make_gaussian_kernel (conv3d.cpp:40-58); fp64 taps, mass folded into taps_t."""
    lib = N.load_library()
    r = (C.c_int32 * 3)(*[int(v) for v in radii])
    s = (C.c_double * 3)(*[float(v) for v in sigmas])
    if any(v < 0 for v in radii):
        raise ParameterError("kernel radius must be nonnegative")
    tt = np.zeros(2 * int(radii[0]) + 1)
    ty = np.zeros(2 * int(radii[1]) + 1)
    tx = np.zeros(2 * int(radii[2]) + 1)
    dp = C.POINTER(C.c_double)
    N.check(lib.sfseg_make_kernel(r, s, tt.ctypes.data_as(dp), ty.ctypes.data_as(dp),
                                  tx.ctypes.data_as(dp)))
    return SeparableKernel3D(tt, ty, tx, tuple(radii), tuple(sigmas))


def convolve_separable(v, kernel: KernelConfig | SeparableKernel3D, threads: int = 1,
                       ctx: Optional[Context] = None):
    """convolve_separable (conv3d.cpp:171-185): x, y then t pass, zero padded."""
    ctx = ctx or default_context()
    b = _Buf(v)
    T, H, W = _shape3(b.shape)
    out = _empty_like(b)
    ob = _Buf(out, writable=True)
    r = (C.c_int32 * 3)(*[int(x) for x in kernel.radii])
    s = (C.c_double * 3)(*[float(x) for x in kernel.sigmas])
    with ctx.lock:
        N.check(ctx._lib.sfseg_convolve_separable(ctx.handle, T, H, W, b.ptr, r, s, ob.ptr, b.mem))
    return out


def convolve_direct(v, kernel: KernelConfig | SeparableKernel3D, ctx: Optional[Context] = None):
    """convolve_direct (conv3d.cpp:187-243): the dense (2rt+1)(2ry+1)(2rx+1)
    triple sum in fp64 with the reference's weight products and summation
    order, cast to float — the check convolve_separable is tested against
    (test_conv3d.cpp:159-176)."""
    ctx = ctx or default_context()
    k = kernel if isinstance(kernel, SeparableKernel3D) else make_gaussian_kernel(kernel.sigmas,
                                                                                  kernel.radii)
    b = _Buf(v)
    T, H, W = _shape3(b.shape)
    out = _empty_like(b)
    ob = _Buf(out, writable=True)
    r = (C.c_int32 * 3)(*[int(x) for x in k.radii])
    tt, ty, tx = (np.ascontiguousarray(a, np.float64) for a in (k.taps_t, k.taps_y, k.taps_x))
    with ctx.lock:
        N.check(ctx._lib.sfseg_convolve_direct_taps(
            ctx.handle, T, H, W, b.ptr, r, C.c_void_p(tt.ctypes.data), C.c_void_p(ty.ctypes.data),
            C.c_void_p(tx.ctypes.data), ob.ptr, b.mem))
    return out


def separable_convolution_count() -> int:
    """separable_convolution_count (conv3d.cpp:64-66), counted by this library."""
    return int(N.load_library().sfseg_separable_convolution_count())


def _channel_ptrs(bufs: Sequence[_Buf]):
    arr = (C.c_void_p * len(bufs))(*[b.ptr.value for b in bufs])
    return arr


def sfseg_step(x, features: FeatureSet, cfg: SfsegConfig, ctx: Optional[Context] = None):
    """sfseg_step (engine.cpp:141-166): sum of per-channel steps, unnormalised."""
    ctx = ctx or default_context()
    p = cfg.to_params()
    N.check(ctx._lib.sfseg_params_validate(C.byref(p)))
    if len(features.pairwise) == 0:
        raise ParameterError("sfseg_step needs at least one pairwise channel")
    xb = _Buf(x)
    shape = _shape3(xb.shape)
    try:
        sb = _Buf(features.unary, shape)
    except ShapeError:
        raise ShapeError("shape mismatch: solution vs unary")
    fbs = []
    for f in features.pairwise:
        try:
            fbs.append(_Buf(f, shape))
        except ShapeError:
            raise ShapeError("shape mismatch: solution vs pairwise")
    mem = _same_mem([xb, sb] + fbs)
    out = _empty_like(xb)
    ob = _Buf(out, writable=True)
    T, H, W = shape
    with ctx.lock:
        N.check(ctx._lib.sfseg_step(ctx.handle, T, H, W, len(fbs), xb.ptr, sb.ptr,
                                    C.cast(_channel_ptrs(fbs), C.c_void_p), C.byref(p), ob.ptr, mem))
    return out


def sfseg_step_channel(x, s, f, cfg: SfsegConfig, ctx: Optional[Context] = None):
    """sfseg_step_channel (engine.cpp:131-139)."""
    ctx = ctx or default_context()
    p = cfg.to_params()
    N.check(ctx._lib.sfseg_params_validate(C.byref(p)))
    xb = _Buf(x)
    shape = _shape3(xb.shape)
    try:
        sb = _Buf(s, shape)
    except ShapeError:
        raise ShapeError("shape mismatch: solution vs unary")
    try:
        fb = _Buf(f, shape)
    except ShapeError:
        raise ShapeError("shape mismatch: solution vs pairwise")
    mem = _same_mem([xb, sb, fb])
    out = _empty_like(xb)
    ob = _Buf(out, writable=True)
    T, H, W = shape
    with ctx.lock:
        N.check(ctx._lib.sfseg_step_channel(ctx.handle, T, H, W, xb.ptr, sb.ptr, fb.ptr,
                                            C.byref(p), ob.ptr, mem))
    return out


def normalize_l2(x, ctx: Optional[Context] = None):
    """normalize_l2 (engine.cpp:168-183) -> (unit volume, norm)."""
    ctx = ctx or default_context()
    xb = _Buf(x)
    T, H, W = _shape3(xb.shape)
    out = _empty_like(xb)
    ob = _Buf(out, writable=True)
    norm = C.c_double()
    with ctx.lock:
        N.check(ctx._lib.sfseg_normalize_l2(ctx.handle, T, H, W, xb.ptr, ob.ptr, C.byref(norm),
                                            xb.mem))
    return out, norm.value


def project_binary(x, it: int, cfg: SfsegConfig, ctx: Optional[Context] = None):
    """project_binary (engine.cpp:185-205)."""
    ctx = ctx or default_context()
    p = cfg.to_params()
    xb = _Buf(x)
    T, H, W = _shape3(xb.shape)
    out = _empty_like(xb)
    ob = _Buf(out, writable=True)
    with ctx.lock:
        N.check(ctx._lib.sfseg_project_binary(ctx.handle, T, H, W, xb.ptr, int(it), C.byref(p),
                                              ob.ptr, xb.mem))
    return out


def threshold_final(x, frac: float, ctx: Optional[Context] = None):
    """threshold_final (engine.cpp:207-214): uint8 mask of x > float(frac*max)."""
    ctx = ctx or default_context()
    xb = _Buf(x)
    T, H, W = _shape3(xb.shape)
    out = _empty_like(xb, np.uint8)
    ob = _Buf(out, writable=True, dtype=np.uint8)
    with ctx.lock:
        N.check(ctx._lib.sfseg_threshold_final(ctx.handle, T, H, W, xb.ptr, float(frac), ob.ptr,
                                               xb.mem))
    return out


IterationObserver = Callable[[int, np.ndarray], None]


def run(features: FeatureSet, cfg: SfsegConfig, x0=None, reference=None, ground_truth=None,
        transform=None, observer: Optional[IterationObserver] = None,
        ctx: Optional[Context] = None) -> RunResult:
    """sfseg::run (engine.cpp:247-348) on the GPU.

    The per-frame windowed sweep of the reference is replaced by one global
    step per iteration (bit-equal, test_engine.cpp:276-297). ``transform``
    (FrameTransform) is supported only as None: a non-empty hook needs the
    windowed host round trip and lives in the C++ drop-in shim.
    """
    if transform is not None:
        raise ParameterError("FrameTransform hooks are handled by the C++ drop-in shim")
    ctx = ctx or default_context()
    p = cfg.to_params()
    N.check(ctx._lib.sfseg_params_validate(C.byref(p)))
    sb = _Buf(features.unary)
    shape = _shape3(sb.shape)
    if len(features.pairwise) == 0:
        raise ValidationError("feature set needs at least one pairwise channel")
    fbs = []
    for f in features.pairwise:
        try:
            fbs.append(_Buf(f, shape))
        except ShapeError:
            raise ShapeError("pairwise channel shape differs from unary shape")
    bufs = [sb] + fbs
    x0b = None
    if x0 is not None:
        try:
            x0b = _Buf(x0, shape)
        except ShapeError:
            raise ShapeError("x0 shape differs from features")
        bufs.append(x0b)
    refb = gtb = None
    if reference is not None:
        try:
            refb = _Buf(reference, shape)
        except ShapeError:
            raise ShapeError("reference shape differs from features")
    if ground_truth is not None:
        try:
            gtb = _Buf(ground_truth, shape, dtype=np.uint8)
        except ShapeError:
            raise ShapeError("ground truth shape differs from features")
    mem = _same_mem(bufs + [b for b in (refb, gtb) if b is not None])
    T, H, W = shape
    lib = ctx._lib
    soft = _empty_like(sb)
    mask = _empty_like(sb, np.uint8)
    trace = RunTrace()
    with ctx.lock:
        N.check(lib.sfseg_load(ctx.handle, T, H, W, len(fbs), sb.ptr,
                               C.cast(_channel_ptrs(fbs), C.c_void_p),
                               x0b.ptr if x0b else None, mem))
        per_iter = observer is not None or refb is not None or gtb is not None
        if not per_iter:
            recs = (N.IterRecord * cfg.iterations)()
            N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, cfg.iterations, recs))
            for r in recs:
                trace.iterations.append(IterationRecord(r.iter, r.l2_norm_pre_normalize,
                                                        wall_time_s=r.wall_time_s))
        else:
            x_it = _empty_like(sb)
            xib = _Buf(x_it, writable=True)
            for it in range(1, cfg.iterations + 1):
                rec = N.IterRecord()
                N.check(lib.sfseg_solve(ctx.handle, C.byref(p), it, it, C.byref(rec)))
                r = IterationRecord(rec.iter, rec.l2_norm_pre_normalize,
                                    wall_time_s=rec.wall_time_s)
                if refb is not None or gtb is not None:
                    ang, iou = C.c_double(), C.c_double()
                    N.check(lib.sfseg_metrics(ctx.handle, refb.ptr if refb else None,
                                              gtb.ptr if gtb else None, float(cfg.threshold_frac),
                                              C.byref(ang), C.byref(iou), mem))
                    if refb is not None:
                        r.angle_deg = ang.value
                    if gtb is not None:
                        r.iou = iou.value
                trace.iterations.append(r)
                if observer is not None:
                    N.check(lib.sfseg_download(ctx.handle, 0.5, xib.ptr, None, mem))
                    observer(it, x_it)
        ob, mb = _Buf(soft, writable=True), _Buf(mask, writable=True, dtype=np.uint8)
        N.check(lib.sfseg_download(ctx.handle, float(cfg.final_threshold), ob.ptr, mb.ptr, mem))
    return RunResult(soft, mask, trace)


def run_batch(clips: Sequence[FeatureSet], cfg: SfsegConfig, x0s: Optional[Sequence] = None,
              ctxs: Optional[Sequence[Context]] = None, outputs: Optional[Sequence] = None):
    """A batch of independent videos (BASELINE configs[3]): the reference runs
    one video per run() call (engine.cpp:247), so a batch is a loop of calls;
    sfseg_run_batch runs that loop over ``ctxs`` — largest clip first, each
    context on its own host thread. Contexts on one device overlap one clip's
    transfers with another's solve; contexts on several devices shard the
    batch (no collective). Every result equals run_once() of that clip alone.

    ``outputs``: optional list of (soft, mask) host arrays to fill (e.g. pinned
    buffers); otherwise numpy arrays are allocated. Returns a list of
    RunResult in batch order; the first failing clip raises its error."""
    if ctxs is None:
        ctxs = [default_context()]
    lib = ctxs[0]._lib
    p = cfg.to_params()
    N.check(lib.sfseg_params_validate(C.byref(p)))
    n = len(clips)
    arr = (N.Clip * max(n, 1))()
    keep = []
    results = []
    mem = None
    for i, fs in enumerate(clips):
        sb = _Buf(fs.unary)
        shape = _shape3(sb.shape)
        if len(fs.pairwise) == 0:
            raise ValidationError("feature set needs at least one pairwise channel")
        fbs = [sb if f is fs.unary else _Buf(f, shape) for f in fs.pairwise]
        x0b = _Buf(x0s[i], shape) if x0s is not None and x0s[i] is not None else None
        m = _same_mem([sb] + fbs + ([x0b] if x0b else []))
        if mem is not None and m != mem:
            raise ValidationError("mixing host and device volumes in one call")
        mem = m
        if outputs is not None:
            soft, mask = outputs[i]
        else:
            soft, mask = _empty_like(sb), _empty_like(sb, np.uint8)
        ob, mb = _Buf(soft, shape, writable=True), _Buf(mask, shape, writable=True, dtype=np.uint8)
        recs = (N.IterRecord * cfg.iterations)()
        fp = _channel_ptrs(fbs)
        keep.append((sb, fbs, x0b, ob, mb, recs, fp))
        T, H, W = shape
        c = arr[i]
        c.frames, c.height, c.width, c.channels = T, H, W, len(fbs)
        c.unary = sb.ptr
        c.pairwise = C.cast(fp, C.c_void_p)
        c.x0 = x0b.ptr if x0b else None
        c.soft, c.mask = ob.ptr, mb.ptr
        c.records = C.cast(recs, C.c_void_p)
        results.append((soft, mask, recs))
    handles = (C.c_void_p * len(ctxs))(*[c.handle.value for c in ctxs])
    locks = [c.lock for c in ctxs]
    for lk in locks:
        lk.acquire()
    try:
        N.check(lib.sfseg_run_batch(C.cast(handles, C.c_void_p), len(ctxs), arr, n, C.byref(p),
                                    mem if mem is not None else N.SFSEG_MEM_HOST))
    finally:
        for lk in locks:
            lk.release()
    out = []
    for i, (soft, mask, recs) in enumerate(results):
        trace = RunTrace([IterationRecord(r.iter, r.l2_norm_pre_normalize, wall_time_s=r.wall_time_s)
                          for r in recs])
        res = RunResult(soft, mask, trace)
        res.worker = int(arr[i].worker)
        res.wall_ms = float(arr[i].wall_ms)
        out.append(res)
    return out


def run_once(features: FeatureSet, cfg: SfsegConfig, x0=None,
             ctx: Optional[Context] = None) -> RunResult:
    """sfseg::run (engine.cpp:247-348) as ONE C-ABI call, sfseg_run: load (S^p
    computed under the channels' DMA), solve 1..iterations, download. This is
    the entry point bench.py's e2e times. A channel that is the unary array
    itself (f = S, as in BASELINE c0/c1/c3) is passed as the same pointer and
    crosses the bus once."""
    ctx = ctx or default_context()
    p = cfg.to_params()
    N.check(ctx._lib.sfseg_params_validate(C.byref(p)))
    sb = _Buf(features.unary)
    shape = _shape3(sb.shape)
    if len(features.pairwise) == 0:
        raise ValidationError("feature set needs at least one pairwise channel")
    fbs = [sb if f is features.unary else _Buf(f, shape) for f in features.pairwise]
    x0b = _Buf(x0, shape) if x0 is not None else None
    mem = _same_mem([sb] + fbs + ([x0b] if x0b else []))
    T, H, W = shape
    soft = _empty_like(sb)
    mask = _empty_like(sb, np.uint8)
    ob, mb = _Buf(soft, writable=True), _Buf(mask, writable=True, dtype=np.uint8)
    recs = (N.IterRecord * cfg.iterations)()
    with ctx.lock:
        N.check(ctx._lib.sfseg_run(ctx.handle, T, H, W, len(fbs), sb.ptr,
                                   C.cast(_channel_ptrs(fbs), C.c_void_p),
                                   x0b.ptr if x0b else None, C.byref(p), ob.ptr, mb.ptr, recs, mem))
    trace = RunTrace()
    for r in recs:
        trace.iterations.append(IterationRecord(r.iter, r.l2_norm_pre_normalize,
                                                wall_time_s=r.wall_time_s))
    return RunResult(soft, mask, trace)


def run_until_converged(features: FeatureSet, cfg: SfsegConfig, tol: float,
                        criterion: str = "angle", max_iterations: Optional[int] = None,
                        x0=None, ctx: Optional[Context] = None):
    """Power iteration with an early exit (sfseg_solve_until).

    The reference's run() always performs cfg.iterations; its power_iteration
    stops once ||x_k - x_{k-1}||_2 < tol (oracle.cpp:234-242, criterion
    "step") and bench.cpp's converged_conv once angle(x_k, x_{k-1}) < tol
    degrees (bench.cpp:75-80, criterion "angle"). Returns (RunResult,
    iterations_done); the result's trace has one record per iteration run.
    """
    crit = {"step": N.SFSEG_CONV_STEP, "angle": N.SFSEG_CONV_ANGLE}.get(criterion)
    if crit is None:
        raise ParameterError("criterion must be 'step' or 'angle'")
    ctx = ctx or default_context()
    p = cfg.to_params()
    N.check(ctx._lib.sfseg_params_validate(C.byref(p)))
    max_it = int(max_iterations if max_iterations is not None else cfg.iterations)
    sb = _Buf(features.unary)
    shape = _shape3(sb.shape)
    if len(features.pairwise) == 0:
        raise ValidationError("feature set needs at least one pairwise channel")
    fbs = [_Buf(f, shape) for f in features.pairwise]
    bufs = [sb] + fbs
    x0b = _Buf(x0, shape) if x0 is not None else None
    if x0b is not None:
        bufs.append(x0b)
    mem = _same_mem(bufs)
    T, H, W = shape
    lib = ctx._lib
    soft = _empty_like(sb)
    mask = _empty_like(sb, np.uint8)
    trace = RunTrace()
    recs = (N.IterRecord * max_it)()
    done = C.c_int32()
    with ctx.lock:
        N.check(lib.sfseg_load(ctx.handle, T, H, W, len(fbs), sb.ptr,
                               C.cast(_channel_ptrs(fbs), C.c_void_p),
                               x0b.ptr if x0b else None, mem))
        N.check(lib.sfseg_solve_until(ctx.handle, C.byref(p), 1, max_it, crit, float(tol),
                                      C.byref(done), recs))
        for r in recs[:done.value]:
            trace.iterations.append(IterationRecord(r.iter, r.l2_norm_pre_normalize,
                                                    wall_time_s=r.wall_time_s))
        ob, mb = _Buf(soft, writable=True), _Buf(mask, writable=True, dtype=np.uint8)
        N.check(lib.sfseg_download(ctx.handle, float(cfg.final_threshold), ob.ptr, mb.ptr, mem))
    return RunResult(soft, mask, trace), done.value


def volume_shape(path) -> tuple:
    """(T, H, W) from an SFSV container header (volume.hpp:111-121)."""
    with open(path, "rb") as f:
        h = f.read(32)
    if len(h) < 32:
        raise CorruptionError(f"file shorter than the container header: {path}")
    return tuple(int.from_bytes(h[o:o + 4], "little") for o in (8, 12, 16))


def run_files(unary_path, pairwise_paths: Sequence, cfg: SfsegConfig, x0_path=None,
              ctx: Optional[Context] = None) -> RunResult:
    """run() on volumes stored as SFSV containers (load_volume,
    volume.cpp:142-184), streamed from the files into device memory by
    sfseg_load_files (two pinned buffers, reads overlapped with the DMA);
    the files' headers are checked first and load_volume's errors surface
    as IoError / FormatError / CorruptionError / ValidationError."""
    ctx = ctx or default_context()
    p = cfg.to_params()
    N.check(ctx._lib.sfseg_params_validate(C.byref(p)))
    paths = [os.fsencode(x) for x in pairwise_paths]
    arr = (C.c_char_p * max(1, len(paths)))(*paths)
    lib = ctx._lib
    trace = RunTrace()
    recs = (N.IterRecord * cfg.iterations)()
    with ctx.lock:
        N.check(lib.sfseg_load_files(ctx.handle, os.fsencode(unary_path), C.cast(arr, C.c_void_p),
                                     len(paths), os.fsencode(x0_path) if x0_path else None))
        T, H, W = volume_shape(unary_path)
        N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, cfg.iterations, recs))
        for r in recs:
            trace.iterations.append(IterationRecord(r.iter, r.l2_norm_pre_normalize,
                                                    wall_time_s=r.wall_time_s))
        soft = np.empty((T, H, W), np.float32)
        mask = np.empty((T, H, W), np.uint8)
        N.check(lib.sfseg_download(ctx.handle, float(cfg.final_threshold),
                                   soft.ctypes.data_as(C.c_void_p), mask.ctypes.data_as(C.c_void_p),
                                   N.SFSEG_MEM_HOST))
    return RunResult(soft, mask, trace)


_AFFINITY_KINDS = {"exact": N.SFSEG_AFFINITY_EXACT, "taylor": N.SFSEG_AFFINITY_TAYLOR,
                   "taylor_channel_sum": N.SFSEG_AFFINITY_TAYLOR_CHANNEL_SUM}


def _affinity_operands(features: FeatureSet, cfg: SfsegConfig, kind: str):
    if kind not in _AFFINITY_KINDS:
        raise ParameterError("kind must be 'exact', 'taylor' or 'taylor_channel_sum'")
    S = np.ascontiguousarray(features.unary, np.float32)
    if len(features.pairwise) == 0:
        raise ValidationError("feature set needs at least one pairwise channel")
    F = [np.ascontiguousarray(f, np.float32) for f in features.pairwise]
    for f in F:
        if f.shape != S.shape:
            raise ShapeError("pairwise channel shape differs from unary shape")
    ptrs = (C.c_void_p * len(F))(*[f.ctypes.data for f in F])
    return S, F, ptrs, cfg.to_params(), _AFFINITY_KINDS[kind]


def affinity_matvec(features: FeatureSet, cfg: SfsegConfig, x, kind: str = "taylor",
                    ctx: Optional[Context] = None) -> np.ndarray:
    """y = M x for the reference's explicit affinity (oracle.hpp:76-107,
    oracle.cpp:191-207), matrix-free in fp64 on the GPU and without the
    1e6-node cap (sfseg_affinity_matvec)."""
    ctx = ctx or default_context()
    S, F, ptrs, p, k = _affinity_operands(features, cfg, kind)
    x = np.ascontiguousarray(x, np.float64)
    if x.shape != S.shape:
        raise ShapeError("matvec operand length mismatch")
    y = np.empty_like(x)
    T, H, W = S.shape
    with ctx.lock:
        N.check(ctx._lib.sfseg_affinity_matvec(ctx.handle, T, H, W, len(F), S.ctypes.data,
                                               C.cast(ptrs, C.c_void_p), C.byref(p), k,
                                               x.ctypes.data, y.ctypes.data, N.SFSEG_MEM_HOST))
    return y


def power_iteration(features: FeatureSet, cfg: SfsegConfig, x0, max_iters: int, tol: float,
                    kind: str = "taylor", ctx: Optional[Context] = None):
    """The reference's power_iteration + cluster_score (oracle.cpp:219-258)
    on the GPU: returns (eigenvector, eigenvalue, iterations_used)."""
    ctx = ctx or default_context()
    S, F, ptrs, p, k = _affinity_operands(features, cfg, kind)
    x0 = np.ascontiguousarray(x0, np.float64)
    if x0.shape != S.shape:
        raise ShapeError("x0 length does not match matrix size")
    vec = np.empty_like(x0)
    val, used = C.c_double(), C.c_int32()
    T, H, W = S.shape
    with ctx.lock:
        N.check(ctx._lib.sfseg_affinity_power_iteration(
            ctx.handle, T, H, W, len(F), S.ctypes.data, C.cast(ptrs, C.c_void_p), C.byref(p), k,
            x0.ctypes.data, int(max_iters), float(tol), vec.ctypes.data, C.byref(val),
            C.byref(used), N.SFSEG_MEM_HOST))
    return vec, val.value, used.value
