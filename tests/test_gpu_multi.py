"""In-process multi-GPU solve (sfseg_multi_*, SFSEG_NUM_GPUS in the drop-in):
time shards with peer-memory halos and an event-ordered gather of the
per-frame sums, all device-side. Several shards share the test GPU (the
devices list repeats 0): no kernel waits on another, the ordering is by
stream events, so this is the same data path as N GPUs of one process.
Results must equal one context bit for bit; the
reference's own run() tests also pass through it (test_gpu_dropin.py)."""
import ctypes as C

import numpy as np
import pytest

from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth

pytestmark = pytest.mark.gpu


def multi_run(fs, cfg, devices):
    lib = N.load_library()
    m = C.c_void_p()
    dev = (C.c_int32 * len(devices))(*devices)
    N.check(lib.sfseg_multi_create(len(devices), dev, C.byref(m)))
    try:
        S = np.ascontiguousarray(fs.unary, np.float32)
        F = [np.ascontiguousarray(f, np.float32) for f in fs.pairwise]
        T, H, W = S.shape
        soft = np.empty_like(S)
        mask = np.empty(S.shape, np.uint8)
        recs = (N.IterRecord * cfg.iterations)()
        fp = (C.c_void_p * len(F))(*[f.ctypes.data for f in F])
        p = cfg.to_params()
        N.check(lib.sfseg_multi_run(m, T, H, W, len(F), C.c_void_p(S.ctypes.data),
                                    C.cast(fp, C.c_void_p), None, C.byref(p),
                                    C.c_void_p(soft.ctypes.data), C.c_void_p(mask.ctypes.data),
                                    recs, N.SFSEG_MEM_HOST))
        return soft, mask, [r.l2_norm_pre_normalize for r in recs], [r.wall_time_s for r in recs]
    finally:
        lib.sfseg_multi_destroy(m)


CASES = [
    # (config, frames, crop H x W, arith, binarize, shards)
    (1, 12, None, "fast", False, 2),   # fused_rs: in-kernel peer push, U carried between steps
    (1, 12, None, "exact", True, 3),   # fused_ws + k_halo_push, binarised iterations
    (2, 12, (100, 150), "fast", False, 3),  # C = 8: fused_mc HEAD + TAILs, k_halo_push
    (4, 16, (120, 200), "fast", True, 2),   # C = 3, radii (4, 10, 10)
    (4, 16, (120, 200), "exact", False, 3),
    (3, 30, None, "fast", False, 4),   # a c3 clip (T = 30): shards of at least rt frames
]


@pytest.mark.parametrize("idx,frames,crop,arith,binarize,shards", CASES)
def test_multi_shards_bit_identical_to_one_context(idx, frames, crop, arith, binarize, shards):
    prob = synth.config(idx, frames=frames)[0]
    fs, _ = prob.generate()
    if crop:
        h, w = crop
        fs = E.FeatureSet(np.ascontiguousarray(fs.unary[:, :h, :w]),
                          [np.ascontiguousarray(f[:, :h, :w]) for f in fs.pairwise])
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 6,
                           "binarize_start": 3 if binarize else 7})
    one = E.run(fs, cfg)
    soft, mask, norms, walls = multi_run(fs, cfg, [0] * shards)
    assert np.array_equal(norms, [r.l2_norm_pre_normalize for r in one.trace.iterations])
    assert np.array_equal(soft, one.soft)
    assert np.array_equal(mask, one.mask)
    assert all(w >= 0.0 for w in walls)


def test_multi_applies_the_unit_range_guard_globally():
    # channels outside [0, 1]: every shard rescales with the GLOBAL min/max
    prob = synth.config(1, frames=9)[0]
    fs, _ = prob.generate()
    F = [(2.0 * fs.pairwise[0] - 0.3).astype(np.float32)]
    F[0][0, 0, 0] = -1.0  # the global minimum sits in shard 0's frames only
    fs = E.FeatureSet(fs.unary, F)
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": "exact", "iterations": 4,
                           "binarize_start": 5})
    one = E.run(fs, cfg)
    soft, mask, norms, _ = multi_run(fs, cfg, [0, 0, 0])
    assert np.array_equal(soft, one.soft)
    assert np.array_equal(norms, [r.l2_norm_pre_normalize for r in one.trace.iterations])
