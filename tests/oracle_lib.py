"""Test-side loaders for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``    — oracle/_ref/liboracle.so, our C restatement (oracle/sfseg_oracle.c)
* ``Reference`` — oracle/_ref/libsfseg_ref.so, the reference library compiled
                  unchanged from /root/reference/proj/src (oracle/Makefile)

Both take the same sfseg_params struct as the product C ABI.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_1907_02731_b200._native import Params

ROOT = Path(__file__).resolve().parents[1]
REF_DIR = ROOT / "oracle" / "_ref"

_F = np.float32


def _vp(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _chans(F):
    return (C.c_void_p * len(F))(*[f.ctypes.data for f in F])


def params(cfg) -> Params:
    return cfg.to_params()


class _Base:
    def __init__(self, path: Path):
        self.lib = C.CDLL(str(path))


class Oracle(_Base):
    def __init__(self):
        super().__init__(REF_DIR / "liboracle.so")

    def make_kernel(self, radii, sigmas):
        r = (C.c_int32 * 3)(*radii)
        s = (C.c_double * 3)(*sigmas)
        out = [np.zeros(2 * v + 1) for v in radii]
        rc = self.lib.oracle_make_kernel(r, s, *[_vp(o) for o in out])
        assert rc == 0
        return out

    def convolve_separable(self, v, radii, sigmas):
        v = np.ascontiguousarray(v, _F)
        out = np.empty_like(v)
        T, H, W = v.shape
        rc = self.lib.oracle_convolve_separable(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), _vp(v),
                                                (C.c_int32 * 3)(*radii),
                                                (C.c_double * 3)(*sigmas), _vp(out))
        assert rc == 0
        return out

    def step(self, x, S, F, cfg):
        x, S = np.ascontiguousarray(x, _F), np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        out = np.empty_like(x)
        T, H, W = x.shape
        p = params(cfg)
        rc = self.lib.oracle_step(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), C.c_int32(len(F)),
                                  _vp(x), _vp(S), C.cast(_chans(F), C.c_void_p), C.byref(p),
                                  _vp(out))
        if rc:
            raise RuntimeError(f"oracle_step rc={rc}")
        return out

    def normalize_l2(self, x):
        x = np.ascontiguousarray(x, _F)
        out = np.empty_like(x)
        norm = C.c_double()
        rc = self.lib.oracle_normalize_l2(_vp(x), C.c_size_t(x.size), _vp(out), C.byref(norm))
        return out, norm.value, rc

    def project_binary(self, x, it, cfg):
        x = np.ascontiguousarray(x, _F)
        out = np.empty_like(x)
        p = params(cfg)
        self.lib.oracle_project_binary(_vp(x), C.c_size_t(x.size), C.c_int32(it), C.byref(p),
                                       _vp(out))
        return out

    def threshold_final(self, x, frac):
        x = np.ascontiguousarray(x, _F)
        out = np.empty(x.shape, np.uint8)
        self.lib.oracle_threshold_final(_vp(x), C.c_size_t(x.size), C.c_double(frac), _vp(out))
        return out

    def run(self, S, F, cfg, x0=None, checkpoints=()):
        S = np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        T, H, W = S.shape
        soft = np.empty_like(S)
        mask = np.empty(S.shape, np.uint8)
        norms = np.zeros(cfg.iterations)
        ck = np.asarray(checkpoints, np.int32)
        ck_out = np.empty((len(ck),) + S.shape, _F)
        p = params(cfg)
        rc = self.lib.oracle_run(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), C.c_int32(len(F)),
                                 _vp(S), C.cast(_chans(F), C.c_void_p),
                                 _vp(np.ascontiguousarray(x0, _F)) if x0 is not None else None,
                                 C.byref(p), _vp(soft), _vp(mask), _vp(norms),
                                 _vp(ck) if len(ck) else None, C.c_int32(len(ck)),
                                 _vp(ck_out) if len(ck) else None)
        if rc:
            raise RuntimeError(f"oracle_run rc={rc}")
        return soft, mask, norms, ck_out

    def xoshiro_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.oracle_xoshiro_u64(C.c_uint64(seed), _vp(out), C.c_size_t(n))
        return out


class Reference(_Base):
    """The reference library itself, built from /root/reference (test-only)."""

    def __init__(self):
        super().__init__(REF_DIR / "libsfseg_ref.so")
        self.lib.sfref_last_error.restype = C.c_char_p

    def _chk(self, rc):
        if rc:
            raise RuntimeError(f"reference rc={rc}: {self.lib.sfref_last_error().decode()}")

    def validate(self, cfg):
        p = params(cfg)
        return self.lib.sfref_validate(C.byref(p))

    def make_kernel(self, radii, sigmas):
        out = [np.zeros(2 * v + 1) for v in radii]
        self._chk(self.lib.sfref_make_kernel((C.c_int32 * 3)(*radii), (C.c_double * 3)(*sigmas),
                                             *[_vp(o) for o in out]))
        return out

    def convolve_separable(self, v, radii, sigmas, threads=1):
        v = np.ascontiguousarray(v, _F)
        out = np.empty_like(v)
        T, H, W = v.shape
        self._chk(self.lib.sfref_convolve_separable(
            C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), _vp(v), (C.c_int32 * 3)(*radii),
            (C.c_double * 3)(*sigmas), C.c_int(threads), _vp(out)))
        return out


    def convolve_direct(self, v, radii, sigmas):
        v = np.ascontiguousarray(v, _F)
        out = np.empty_like(v)
        T, H, W = v.shape
        self._chk(self.lib.sfref_convolve_direct(
            C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), _vp(v), (C.c_int32 * 3)(*radii),
            (C.c_double * 3)(*sigmas), _vp(out)))
        return out
    def step(self, x, S, F, cfg, threads=1):
        x, S = np.ascontiguousarray(x, _F), np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        out = np.empty_like(x)
        T, H, W = x.shape
        p = params(cfg)
        self._chk(self.lib.sfref_step(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W),
                                      C.c_int32(len(F)), _vp(x), _vp(S),
                                      C.cast(_chans(F), C.c_void_p), C.byref(p), C.c_int(threads),
                                      _vp(out)))
        return out

    def normalize_l2(self, x):
        x = np.ascontiguousarray(x, _F)
        out = np.empty_like(x)
        norm = C.c_double()
        T, H, W = x.shape
        rc = self.lib.sfref_normalize_l2(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), _vp(x),
                                         _vp(out), C.byref(norm))
        return out, norm.value, rc

    def project_binary(self, x, it, cfg):
        x = np.ascontiguousarray(x, _F)
        out = np.empty_like(x)
        T, H, W = x.shape
        p = params(cfg)
        self._chk(self.lib.sfref_project_binary(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W),
                                                _vp(x), C.c_int32(it), C.byref(p), _vp(out)))
        return out

    def threshold_final(self, x, frac):
        x = np.ascontiguousarray(x, _F)
        out = np.empty(x.shape, np.uint8)
        T, H, W = x.shape
        self._chk(self.lib.sfref_threshold_final(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W),
                                                 _vp(x), C.c_double(frac), _vp(out)))
        return out

    def run(self, S, F, cfg, x0=None, checkpoints=(), threads=1):
        S = np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        T, H, W = S.shape
        soft = np.empty_like(S)
        mask = np.empty(S.shape, np.uint8)
        norms = np.zeros(cfg.iterations)
        ck = np.asarray(checkpoints, np.int32)
        ck_out = np.empty((len(ck),) + S.shape, _F)
        p = params(cfg)
        self._chk(self.lib.sfref_run(
            C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), C.c_int32(len(F)), _vp(S),
            C.cast(_chans(F), C.c_void_p),
            _vp(np.ascontiguousarray(x0, _F)) if x0 is not None else None, C.byref(p),
            C.c_int(threads), _vp(soft), _vp(mask), _vp(norms), _vp(ck) if len(ck) else None,
            C.c_int32(len(ck)), _vp(ck_out) if len(ck) else None))
        return soft, mask, norms, ck_out

    def save_volume(self, path, v):
        """sfseg_ref::save_volume (volume.cpp:117-140)"""
        v = np.ascontiguousarray(v, _F)
        T, H, W = v.shape
        self._chk(self.lib.sfref_save_volume(str(path).encode(), C.c_uint32(T), C.c_uint32(H),
                                             C.c_uint32(W), _vp(v)))

    def load_volume_rc(self, path):
        """sfseg_ref::load_volume (volume.cpp:142-184): (status, (T, H, W) or None)"""
        dims = (C.c_uint32 * 3)()
        rc = self.lib.sfref_load_volume(str(path).encode(), dims, None, C.c_size_t(0))
        return rc, (tuple(int(d) for d in dims) if rc == 0 else None)

    _KINDS = {"exact": 0, "taylor": 1, "taylor_channel_sum": 2}

    def affinity_matvec(self, S, F, cfg, x, kind="taylor"):
        """sfseg_ref::matvec(build_affinity_<kind>(...), x) (oracle.cpp:67-207);
        returns (status, y)"""
        S = np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty_like(x)
        T, H, W = S.shape
        p = params(cfg)
        rc = self.lib.sfref_affinity_matvec(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W),
                                            C.c_int32(len(F)), _vp(S), C.cast(_chans(F), C.c_void_p),
                                            C.byref(p), C.c_int32(self._KINDS[kind]), _vp(x), _vp(y))
        return rc, y

    def power_iteration(self, S, F, cfg, x0, max_iters, tol, kind="taylor"):
        """sfseg_ref::power_iteration (oracle.cpp:219-247): (vec, value, used)"""
        S = np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        x0 = np.ascontiguousarray(x0, np.float64)
        vec = np.empty_like(x0)
        val, used = C.c_double(), C.c_int32()
        T, H, W = S.shape
        p = params(cfg)
        self._chk(self.lib.sfref_power_iteration(
            C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), C.c_int32(len(F)), _vp(S),
            C.cast(_chans(F), C.c_void_p), C.byref(p), C.c_int32(self._KINDS[kind]), _vp(x0),
            C.c_int32(max_iters), C.c_double(tol), _vp(vec), C.byref(val), C.byref(used)))
        return vec, val.value, used.value

    def global_loop(self, S, F, cfg, iterations, threads=1):
        S = np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        T, H, W = S.shape
        out = np.empty_like(S)
        p = params(cfg)
        self._chk(self.lib.sfref_global_loop(C.c_uint32(T), C.c_uint32(H), C.c_uint32(W),
                                             C.c_int32(len(F)), _vp(S),
                                             C.cast(_chans(F), C.c_void_p), C.byref(p),
                                             C.c_int(threads), C.c_int32(iterations), _vp(out)))
        return out

    def global_loop_ck(self, S, F, cfg, iterations, checkpoints, threads=1):
        """global_loop plus the normalised iterate after each checkpoint
        iteration and the pre-normalisation norms: (final, snaps, norms)"""
        S = np.ascontiguousarray(S, _F)
        F = [np.ascontiguousarray(f, _F) for f in F]
        T, H, W = S.shape
        out = np.empty_like(S)
        ck = np.asarray(sorted(checkpoints), np.int32)
        snaps = np.empty((len(ck),) + S.shape, _F)
        norms = np.zeros(iterations)
        p = params(cfg)
        self._chk(self.lib.sfref_global_loop_ck(
            C.c_uint32(T), C.c_uint32(H), C.c_uint32(W), C.c_int32(len(F)), _vp(S),
            C.cast(_chans(F), C.c_void_p), C.byref(p), C.c_int(threads), C.c_int32(iterations),
            _vp(out), _vp(ck), C.c_int32(len(ck)), _vp(snaps), _vp(norms)))
        return out, {int(k): snaps[i] for i, k in enumerate(ck)}, norms

    def xoshiro_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.sfref_xoshiro_u64(C.c_uint64(seed), _vp(out), C.c_size_t(n))
        return out

    def xoshiro_gaussian(self, seed, n):
        out = np.empty(n, np.float64)
        self.lib.sfref_xoshiro_gaussian(C.c_uint64(seed), _vp(out), C.c_size_t(n))
        return out


def reference_available() -> bool:
    return (REF_DIR / "libsfseg_ref.so").exists()


def oracle_available() -> bool:
    return (REF_DIR / "liboracle.so").exists()


def random_volume(shape, seed, lo=0.0, hi=1.0):
    """Seeded float32 volume: float(next_double()) per voxel like the
    reference tests' random_volume (test_engine.cpp:35-40)."""
    u = Oracle().xoshiro_u64(seed, int(np.prod(shape)))
    d = (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (lo + (hi - lo) * d).astype(np.float32).reshape(shape)
