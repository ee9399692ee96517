"""sfseg_run_batch (BASELINE configs[3]: a batch of independent clips). The
reference solves one video per run() call (engine.cpp:247); the batch entry
must return, for every clip, exactly what the one-clip call returns — whatever
the number of contexts, the LPT order or the buffer reuse between clips of
different shapes — and report a failing clip without losing the others."""
import ctypes as C

import numpy as np
import pytest

from paper_1907_02731_b200 import _native as N
from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth
from paper_1907_02731_b200.sharding import assign_clips, run_clips
from tests.oracle_lib import random_volume

pytestmark = pytest.mark.gpu

# ragged batch: both c3 resolutions (cropped), lengths that grow and shrink so
# a context's buffers are reused, re-zeroed (new row layout) and reallocated
SHAPES = [(9, 60, 80), (21, 90, 160), (7, 90, 160), (30, 60, 80), (5, 33, 47), (12, 90, 160),
          (6, 60, 80)]


def _batch(channels=1, aliased=True):
    clips = []
    for i, s in enumerate(SHAPES):
        S = random_volume(s, 300 + i)
        F = [S] if aliased and channels == 1 else [random_volume(s, 400 + 10 * i + c) for c in range(channels)]
        clips.append(E.FeatureSet(S, F))
    return clips


def _cfg(arith, radii=(2, 4, 4), iterations=5, binarize_start=6):
    return E.SfsegConfig(kernel=E.KernelConfig(radii, (0.5, 1.5, 1.5)), iterations=iterations,
                         binarize_start=binarize_start, arith=arith)


@pytest.mark.parametrize("arith", ["fast", "exact"])
@pytest.mark.parametrize("nctx", [1, 2, 3])
def test_batch_equals_one_call_per_clip(arith, nctx):
    clips = _batch()
    cfg = _cfg(arith)
    ctxs = [E.Context(0) for _ in range(nctx)]
    try:
        got = E.run_batch(clips, cfg, ctxs=ctxs)
    finally:
        for c in ctxs:
            c.close()
    assert len(got) == len(clips)
    assert {r.worker for r in got} <= set(range(nctx))
    ref_ctx = E.Context(0)
    try:
        for fs, r in zip(clips, got):
            one = E.run_once(fs, cfg, ctx=ref_ctx)
            assert np.array_equal(r.soft, one.soft)
            assert np.array_equal(r.mask, one.mask)
            assert [x.l2_norm_pre_normalize for x in r.trace.iterations] == \
                   [x.l2_norm_pre_normalize for x in one.trace.iterations]
    finally:
        ref_ctx.close()


def test_batch_multichannel_and_binarised():
    clips = _batch(channels=3, aliased=False)[:4]
    cfg = _cfg("fast", radii=(3, 7, 7), iterations=4, binarize_start=3)
    ctxs = [E.Context(0), E.Context(0)]
    try:
        got = E.run_batch(clips, cfg, ctxs=ctxs)
        for fs, r in zip(clips, got):
            one = E.run_once(fs, cfg, ctx=ctxs[0])
            assert np.array_equal(r.soft, one.soft)
            assert np.array_equal(r.mask, one.mask)
    finally:
        for c in ctxs:
            c.close()


def test_batch_reports_the_failing_clip_and_runs_the_rest():
    clips = _batch()[:4]
    bad = clips[1].unary.copy()
    bad[0, 0, 0] = -1.0  # ValidationError in run() (volume.cpp:76-81 role check)
    clips[1] = E.FeatureSet(bad, [bad])
    cfg = _cfg("fast")
    lib = N.load_library()
    ctxs = [E.Context(0), E.Context(0)]
    try:
        with pytest.raises(E.ValidationError, match="clip 1"):
            E.run_batch(clips, cfg, ctxs=ctxs)
        # the C ABI keeps every clip's own status
        p = cfg.to_params()
        arr = (N.Clip * len(clips))()
        outs = []
        for i, fs in enumerate(clips):
            T, H, W = fs.unary.shape
            soft = np.zeros(fs.unary.shape, np.float32)
            fp = (C.c_void_p * 1)(fs.pairwise[0].ctypes.data)
            outs.append((soft, fp))
            arr[i].frames, arr[i].height, arr[i].width, arr[i].channels = T, H, W, 1
            arr[i].unary = fs.unary.ctypes.data
            arr[i].pairwise = C.cast(fp, C.c_void_p)
            arr[i].soft = soft.ctypes.data
        h = (C.c_void_p * 2)(ctxs[0].handle.value, ctxs[1].handle.value)
        rc = lib.sfseg_run_batch(C.cast(h, C.c_void_p), 2, arr, len(clips), C.byref(p), N.SFSEG_MEM_HOST)
        assert rc == N.SFSEG_ERR_VALIDATION
        assert [arr[i].status for i in range(4)] == [0, N.SFSEG_ERR_VALIDATION, 0, 0]
        for i in (0, 2, 3):
            one = E.run_once(clips[i], cfg, ctx=ctxs[0])
            assert np.array_equal(outs[i][0], one.soft)
    finally:
        for c in ctxs:
            c.close()


def test_batch_argument_errors_and_empty_batch():
    cfg = _cfg("fast")
    ctx = E.Context(0)
    try:
        assert E.run_batch([], cfg, ctxs=[ctx]) == []
        lib = N.load_library()
        p = cfg.to_params()
        h = (C.c_void_p * 2)(ctx.handle.value, ctx.handle.value)
        arr = (N.Clip * 1)()
        assert lib.sfseg_run_batch(C.cast(h, C.c_void_p), 2, arr, 1, C.byref(p), N.SFSEG_MEM_HOST) == \
               N.SFSEG_ERR_PARAMETER  # the same context twice
        assert lib.sfseg_run_batch(None, 1, arr, 1, C.byref(p), N.SFSEG_MEM_HOST) == N.SFSEG_ERR_PARAMETER
    finally:
        ctx.close()


def test_run_clips_shards_a_callers_batch_by_lpt():
    clips = _batch()
    cfg = _cfg("fast")
    vox = [int(np.prod(c.unary.shape)) for c in clips]
    parts = assign_clips(vox, 2)
    got = {}
    for rank in range(2):
        res = run_clips(clips, cfg, rank=rank, world=2)
        assert sorted(res) == sorted(parts[rank])
        got.update(res)
    assert sorted(got) == list(range(len(clips)))
    for i, fs in enumerate(clips):
        assert np.array_equal(got[i].soft, E.run_once(fs, cfg).soft)


def test_context_reuse_across_shapes_is_clean():
    # one context, clips of different row layouts back to back, then the first
    # again: stale pitch padding or partials of a larger clip must not leak
    cfg = _cfg("exact", iterations=3, binarize_start=2)
    ctx, fresh = E.Context(0), None
    try:
        clips = _batch()
        first = E.run_once(clips[1], cfg, ctx=ctx)  # the largest: sets the capacity
        for fs in clips[2:]:
            E.run_once(fs, cfg, ctx=ctx)
        again = E.run_once(clips[1], cfg, ctx=ctx)
        assert np.array_equal(first.soft, again.soft)
        for fs in (clips[4], clips[0]):
            fresh = E.Context(0)
            assert np.array_equal(E.run_once(fs, cfg, ctx=ctx).soft, E.run_once(fs, cfg, ctx=fresh).soft)
            fresh.close()
    finally:
        ctx.close()


def test_full_c3_batch_equals_one_call_per_clip():
    # BASELINE configs[3] at full size: 14 clips, T in [21, 279], two
    # resolutions, 25 iterations, through three contexts of the GPU
    probs = synth.config(3)
    cfg = E.SfsegConfig(**{**probs[0].cfg.__dict__, "arith": "fast"})
    clips = []
    for p in probs:
        fs, _ = p.generate()
        clips.append(E.FeatureSet(fs.unary, [fs.unary]))  # f = S, passed once
    ctxs = [E.Context(0) for _ in range(3)]
    try:
        got = E.run_batch(clips, cfg, ctxs=ctxs)
        assert len({r.worker for r in got}) > 1  # the queue really spread the clips
        for fs, r in zip(clips, got):
            one = E.run_once(fs, cfg, ctx=ctxs[0])
            assert np.array_equal(r.soft, one.soft)
            assert np.array_equal(r.mask, one.mask)
            assert np.isfinite(r.soft).all() and abs(float(np.linalg.norm(r.soft.astype(np.float64))) - 1.0) < 1e-5
    finally:
        for c in ctxs:
            c.close()
