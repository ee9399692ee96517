"""Seeded synthetic problems for BASELINE.json's five configurations.

Wraps libsfseg_synth.so (include/sfseg_synth.h). BASELINE.json's workloads
are synthetic (moving ellipses with noise), so seeded inputs of exactly those
shapes and value distributions stand in for video data; see DESIGN.md §6.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from ._native import SYNTH_LIB
from .engine import FeatureSet, KernelConfig, SfsegConfig

NOISE_NONE, NOISE_UNIFORM, NOISE_GAUSSIAN = 0, 1, 2
FEAT_SAME, FEAT_MEAN_OF_F, FEAT_NOISY_F = 0, 1, 2

BOX = 1e30  # sigma that makes every raw tap exactly 1.0 (box filter)


class SynthSpec(C.Structure):
    _fields_ = [
        ("frames", C.c_uint32), ("height", C.c_uint32), ("width", C.c_uint32),
        ("channels", C.c_int32), ("objects", C.c_int32),
        ("semi_min", C.c_double), ("semi_max", C.c_double), ("area_frac", C.c_double),
        ("speed_min", C.c_double), ("speed_max", C.c_double),
        ("inside", C.c_double * 8), ("outside", C.c_double),
        ("noise", C.c_int32), ("noise_level", C.c_double),
        ("feature_mode", C.c_int32), ("feature_sigma", C.c_double),
        ("seed", C.c_uint64),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not SYNTH_LIB.exists():
            raise RuntimeError(f"{SYNTH_LIB} missing: run __graft_entry__.build()")
        _lib = C.CDLL(str(SYNTH_LIB))
        _lib.sfseg_synth_generate.restype = C.c_int
        _lib.sfseg_synth_generate.argtypes = [C.POINTER(SynthSpec), C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_int]
        _lib.sfseg_synth_generate_frames.restype = C.c_int
        _lib.sfseg_synth_generate_frames.argtypes = [C.POINTER(SynthSpec), C.c_uint32, C.c_uint32,
                                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_int]
        _lib.sfseg_synth_xoshiro_u64.argtypes = [C.c_uint64, C.c_void_p, C.c_size_t]
        _lib.sfseg_synth_xoshiro_gaussian.argtypes = [C.c_uint64, C.c_void_p, C.c_size_t]
    return _lib


@dataclass
class Problem:
    name: str
    shape: Tuple[int, int, int]
    channels: int
    spec: SynthSpec
    cfg: SfsegConfig

    def voxels(self) -> int:
        T, H, W = self.shape
        return T * H * W

    def generate(self, threads: int = 0, out=None, mask: bool = False, frame_range=None):
        """Returns (FeatureSet of numpy arrays, mask or None). ``out`` may hold
        preallocated (S, [F_c]) float32 arrays (e.g. pinned host memory).
        ``frame_range=(t0, t1)`` generates only those frames (bit-identical to
        the same frames of the whole volume; a time shard's slab)."""
        lib = _load()
        T, H, W = self.shape
        t0, t1 = frame_range if frame_range is not None else (0, T)
        T = t1 - t0
        if out is None:
            S = np.empty((T, H, W), np.float32)
            F = [np.empty((T, H, W), np.float32) for _ in range(self.channels)]
        else:
            S, F = out
        fptr = (C.c_void_p * self.channels)(*[_ptr(f) for f in F])
        m = np.empty((T, H, W), np.uint8) if mask else None
        rc = lib.sfseg_synth_generate_frames(C.byref(self.spec), int(t0), int(t1), C.c_void_p(_ptr(S)),
                                             C.cast(fptr, C.c_void_p),
                                             C.c_void_p(m.ctypes.data) if m is not None else None,
                                             int(threads))
        if rc != 0:
            raise ValueError("bad synthetic spec")
        return FeatureSet(S, list(F)), m

    def generate_device(self, device="cuda", mask: bool = False):
        """The same problem generated in HBM by sfseg_synth_generate_device
        (libsfseg_cuda.so, include/sfseg_cuda.h): returns (S, [F_c], mask or
        None) as torch tensors on ``device``. Bit-identical to generate()
        except gaussian draws (device log/cos: a rare value one float ulp off)."""
        import torch

        from ._native import load_library

        lib = load_library()
        T, H, W = self.shape
        dev = torch.device(device)
        S = torch.empty((T, H, W), dtype=torch.float32, device=dev)
        F = [torch.empty((T, H, W), dtype=torch.float32, device=dev) for _ in range(self.channels)]
        m = torch.empty((T, H, W), dtype=torch.uint8, device=dev) if mask else None
        fptr = (C.c_void_p * self.channels)(*[f.data_ptr() for f in F])
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream().cuda_stream
            rc = lib.sfseg_synth_generate_device(C.byref(self.spec), C.c_void_p(S.data_ptr()),
                                                 C.cast(fptr, C.c_void_p),
                                                 C.c_void_p(m.data_ptr()) if m is not None else None,
                                                 C.c_void_p(stream))
        if rc == -1:
            raise ValueError("bad synthetic spec")
        if rc != 0:
            raise RuntimeError("sfseg_synth_generate_device: CUDA failure")
        return S, F, m


def _ptr(a) -> int:
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def _spec(T, H, W, C_, *, objects=1, semi=(10.0, 20.0), area_frac=0.0, speed=(1.0, 2.0),
          inside=(0.9,), outside=0.1, noise=NOISE_UNIFORM, level=0.1, mode=FEAT_SAME,
          fsigma=0.0, seed=1) -> SynthSpec:
    s = SynthSpec()
    s.frames, s.height, s.width, s.channels = T, H, W, C_
    s.objects = objects
    s.semi_min, s.semi_max = semi
    s.area_frac = area_frac
    s.speed_min, s.speed_max = speed
    for i, v in enumerate(inside):
        s.inside[i] = v
    s.outside = outside
    s.noise, s.noise_level = noise, level
    s.feature_mode, s.feature_sigma = mode, fsigma
    s.seed = seed
    return s


def _cfg(radii, sigmas, iters) -> SfsegConfig:
    # throughput / eigenvector runs: pure power iteration (binarisation off,
    # binarize_start = iterations + 1); alpha = 1, p = 0.1
    return SfsegConfig(alpha=1.0, p=0.1, kernel=KernelConfig(tuple(radii), tuple(sigmas)),
                       iterations=iters, binarize_start=iters + 1)


def config(idx: int, seed: int = 20190708, frames: Optional[int] = None) -> List[Problem]:
    """BASELINE.json configs[idx] as Problem(s). ``frames`` crops T (parity
    runs on a T-cropped instance of the large configs). c3 returns 14 clips."""
    if idx == 0:
        T = frames or 8
        return [Problem("c0", (T, 64, 64), 1,
                        _spec(T, 64, 64, 1, semi=(10, 20), speed=(1, 2), noise=NOISE_UNIFORM,
                              level=0.1, seed=seed),
                        _cfg((1, 3, 3), (BOX, BOX, BOX), 20))]
    if idx == 1:
        T = frames or 80
        return [Problem("c1", (T, 480, 854), 1,
                        _spec(T, 480, 854, 1, area_frac=0.25, speed=(1, 2), noise=NOISE_GAUSSIAN,
                              level=0.1, seed=seed + 1),
                        _cfg((2, 5, 5), (0.5, 1.5, 1.5), 30))]
    if idx == 2:
        T = frames or 80
        return [Problem("c2", (T, 480, 854), 8,
                        _spec(T, 480, 854, 8, area_frac=0.25, speed=(1, 2), noise=NOISE_NONE,
                              mode=FEAT_MEAN_OF_F, fsigma=0.15, seed=seed + 2),
                        _cfg((3, 7, 7), (BOX, 5.0, 5.0), 30))]
    if idx == 3:
        rng = np.random.Generator(np.random.PCG64(seed + 3))
        clips = []
        for k in range(14):
            T = int(rng.integers(21, 280))
            H, W = [(240, 320), (360, 640)][int(rng.integers(0, 2))]
            if frames:
                T = min(T, frames)
            clips.append(Problem(f"c3.{k}", (T, H, W), 1,
                                 _spec(T, H, W, 1, area_frac=float(rng.uniform(0.05, 0.25)),
                                       speed=(1, 2), noise=NOISE_GAUSSIAN, level=0.1,
                                       seed=seed + 300 + k),
                                 _cfg((2, 4, 4), (0.5, 1.5, 1.5), 25)))
        return clips
    if idx == 4:
        T = frames or 1024
        return [Problem("c4", (T, 1080, 1920), 3,
                        _spec(T, 1080, 1920, 3, objects=3, area_frac=0.08, speed=(1, 2),
                              inside=(0.9, 0.7, 0.5), noise=NOISE_NONE, mode=FEAT_NOISY_F,
                              fsigma=0.1, seed=seed + 4),
                        _cfg((4, 10, 10), (0.5, 1.5, 1.5), 20))]
    raise ValueError("configs are 0..4")


def xoshiro_u64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    _load().sfseg_synth_xoshiro_u64(seed, out.ctypes.data, n)
    return out


def xoshiro_gaussian(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.float64)
    _load().sfseg_synth_xoshiro_gaussian(seed, out.ctypes.data, n)
    return out
