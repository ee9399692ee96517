"""Workload for the compute-sanitizer runs (tests/test_gpu_sanitizer.py).

Small problems that drive every fused kernel family through the C ABI:
fused_step_ws (EXACT, C = 1), fused_step_rs (FAST, C = 1), fused_step_mc HEAD /
TAIL / EXACT (C > 1, tensor-memory ring), the in-epilogue peer push and
k_halo_push (two shards of one process), plus the load / finalize / mask
kernels around them. No torch import: the sanitizer slows every CUDA call, so
the process stays as small as possible. The reference has no sanitizer step
(CMakeLists.txt:26 is -Wall -Wextra only); SURVEY.md §5 asks for one here
because these kernels use mbarrier/TMA pipelines, TMEM and peer stores.

With SFSEG_DEBUG_GUARD=1 (tests/test_gpu_guardbands.py) the library puts a
poisoned guard band around every volume buffer and poisons the buffers
themselves; every case then also checks that no band word changed.

usage: python tests/sanitizer_workload.py [--out results.npz] [case ...]   (default: all)
"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1907_02731_b200 import _native as N  # noqa: E402
from paper_1907_02731_b200 import engine as E  # noqa: E402


GUARD = os.environ.get("SFSEG_DEBUG_GUARD", "0") not in ("", "0")


def check_guards(what):
    """no kernel stored outside its buffers (guard mode only)"""
    if not GUARD:
        return
    lib = N.load_library()
    bad, nbuf = C.c_ulonglong(), C.c_int32()
    lib.sfseg_debug_check_guards.argtypes = [C.POINTER(C.c_ulonglong), C.POINTER(C.c_int32)]
    N.check(lib.sfseg_debug_check_guards(C.byref(bad), C.byref(nbuf)))
    assert nbuf.value > 0, f"{what}: no guarded buffer is live"
    assert bad.value == 0, f"{what}: {bad.value} guard-band words were overwritten"


def _volume(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.random(shape, dtype=np.float32)


def _cfg(radii, arith, iterations=3, binarize_start=None):
    return E.SfsegConfig(alpha=1.0, p=0.1, kernel=E.KernelConfig(tuple(radii), (0.5, 1.5, 1.5)),
                         arith=arith, iterations=iterations,
                         binarize_start=iterations + 1 if binarize_start is None else binarize_start)


def _run(shape, channels, radii, arith, **kw):
    S = _volume(shape, 1)
    F = [_volume(shape, 2 + c) for c in range(channels)]
    res = E.run(E.FeatureSet(S, F), _cfg(radii, arith, **kw))
    assert np.isfinite(res.soft).all()
    check_guards("run")
    return res.soft


def _multi(shape, channels, radii, arith, shards):
    lib = N.load_library()
    S = _volume(shape, 1)
    F = [_volume(shape, 2 + c) for c in range(channels)]
    cfg = _cfg(radii, arith)
    m = C.c_void_p()
    dev = (C.c_int32 * shards)(*([0] * shards))
    N.check(lib.sfseg_multi_create(shards, dev, C.byref(m)))
    try:
        T, H, W = shape
        soft = np.empty_like(S)
        mask = np.empty(shape, np.uint8)
        recs = (N.IterRecord * cfg.iterations)()
        fp = (C.c_void_p * channels)(*[f.ctypes.data for f in F])
        p = cfg.to_params()
        N.check(lib.sfseg_multi_run(m, T, H, W, channels, C.c_void_p(S.ctypes.data),
                                    C.cast(fp, C.c_void_p), None, C.byref(p),
                                    C.c_void_p(soft.ctypes.data), C.c_void_p(mask.ctypes.data),
                                    recs, N.SFSEG_MEM_HOST))
        check_guards("multi")
    finally:
        lib.sfseg_multi_destroy(m)
    one = E.run(E.FeatureSet(S, F), cfg)
    assert np.array_equal(soft, one.soft)
    return soft


CASES = {
    # name: thunk. Shapes are a few tiles (64 x 32) wide so the persistent
    # schedule has full, partial and edge tiles, and T > 2 RT + 1
    "ws_exact_c0": lambda: _run((8, 64, 64), 1, (1, 3, 3), "exact", iterations=3, binarize_start=2),
    "rs_fast_c1": lambda: _run((7, 70, 100), 1, (2, 5, 5), "fast"),
    "ws_exact_c1": lambda: _run((7, 70, 100), 1, (2, 5, 5), "exact"),
    "rs_fast_sigmoid": lambda: _run((6, 40, 70), 1, (1, 2, 2), "fast", iterations=4, binarize_start=2),
    "mc_fast_c2": lambda: _run((9, 70, 70), 3, (3, 7, 7), "fast"),
    "mc_fast_c4": lambda: _run((11, 66, 40), 3, (4, 10, 10), "fast"),
    "mc_exact_c2": lambda: _run((9, 70, 70), 2, (3, 7, 7), "exact"),
    "rs_tmem_large_radius": lambda: _run((9, 70, 40), 1, (3, 7, 7), "fast"),
    "peer_push_fast": lambda: _multi((10, 70, 70), 1, (2, 5, 5), "fast", 2),
    "halo_push_mc": lambda: _multi((12, 66, 40), 2, (3, 7, 7), "fast", 2),
    "step_stateless": lambda: E.sfseg_step(_volume((5, 33, 70), 7),
                                           E.FeatureSet(_volume((5, 33, 70), 8), [_volume((5, 33, 70), 9)]),
                                           _cfg((1, 3, 3), "exact")),
}


def main(argv):
    out = None
    if argv[:1] == ["--out"]:
        out, argv = argv[1], argv[2:]
    names = argv or list(CASES)
    results = {}
    for n in names:
        results[n] = np.asarray(CASES[n]())
        assert np.isfinite(results[n]).all(), n
        print(f"ok {n}", flush=True)
    if out:
        np.savez(out, **results)


if __name__ == "__main__":
    main(sys.argv[1:])
