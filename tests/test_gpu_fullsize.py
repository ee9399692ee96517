"""Parity at BASELINE.json's full c1 size (80 x 480 x 854, kernel 5x11x11).

The CPU reference can afford single steps and a short global-step loop at
this size (all host threads), so these are direct comparisons, plus
size-independent properties of the operator:
  * EXACT step == reference sfseg_step, bit for bit (engine.cpp:141-166)
  * scaling: step(2x) == 2 step(x) exactly (every product and sum scales by a
    power of two), EXACT and FAST
  * symmetry: the affinity matrix is symmetric (oracle.cpp:67-175), so
    <x, M y> == <M x, y> up to fp32 rounding, EXACT and FAST
  * the whole c1 and c2 workloads (30 iterations, binarisation off) against
    the reference's normalize_l2(sfseg_step) loop (bench.cpp:154-155), which
    run() equals bit for bit (test_engine.cpp:276-297): north-star gates and
    the scale-aware forms at every checkpoint (1, 5, 10, 20, 30) and on the
    final iterate and mask
"""
import os

import numpy as np
import pytest

from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth
from tests.oracle_lib import Reference, random_volume, reference_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]

THREADS = max(1, os.cpu_count() or 1)


@pytest.fixture(scope="module")
def c1():
    prob = synth.config(1)[0]
    fs, _ = prob.generate()
    return prob, fs


def _cfg(prob, arith, **kw):
    return E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, **kw})


def test_full_c1_step_bit_exact(c1):
    prob, fs = c1
    x = random_volume(prob.shape, 7)
    cfg = _cfg(prob, "exact")
    got = E.sfseg_step(x, fs, cfg)
    want = Reference().step(x, fs.unary, fs.pairwise, cfg, threads=THREADS)
    assert np.array_equal(got, want), f"{int(np.sum(got != want))} values differ"


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_full_c1_step_scales_exactly(c1, arith):
    prob, fs = c1
    x = random_volume(prob.shape, 8)
    cfg = _cfg(prob, arith)
    y1 = E.sfseg_step(x, fs, cfg)
    y2 = E.sfseg_step((2.0 * x).astype(np.float32), fs, cfg)
    assert np.array_equal(y2, 2.0 * y1)


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_full_c1_operator_is_symmetric(c1, arith):
    prob, fs = c1
    x = random_volume(prob.shape, 9)
    y = random_volume(prob.shape, 10)
    cfg = _cfg(prob, arith)
    mx = E.sfseg_step(x, fs, cfg).astype(np.float64)
    my = E.sfseg_step(y, fs, cfg).astype(np.float64)
    a = float(np.dot(x.astype(np.float64).ravel(), my.ravel()))
    b = float(np.dot(y.astype(np.float64).ravel(), mx.ravel()))
    assert abs(a - b) <= 1e-6 * abs(a), (a, b)


@pytest.fixture(scope="module")
def c1_ref(c1):
    prob, fs = c1
    iters = prob.cfg.iterations  # 30
    cfg = _cfg(prob, "exact", iterations=iters, binarize_start=iters + 1)
    return Reference().global_loop_ck(fs.unary, fs.pairwise, cfg, iters, CKS, threads=THREADS)


CKS = (1, 5, 10, 20, 30)


def _run_checkpoints(fs, cfg):
    snaps = {}
    res = E.run(fs, cfg, observer=lambda it, x: snaps.__setitem__(it, x.copy()) if it in CKS else None)
    return res, snaps


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_full_c1_solve_matches_reference_global_loop(c1, c1_ref, arith):
    prob, fs = c1
    want, ref_snaps, norms = c1_ref
    iters = prob.cfg.iterations
    cfg = _cfg(prob, arith, iterations=iters, binarize_start=iters + 1)
    res, snaps = _run_checkpoints(fs, cfg)
    for it in CKS:  # every checkpointed iteration (north star)
        _gates(snaps[it], ref_snaps[it], cfg.final_threshold)
    _gates(res.soft, want, cfg.final_threshold)
    mine = np.array([r.l2_norm_pre_normalize for r in res.trace.iterations])
    assert np.allclose(mine, norms, rtol=1e-9 if arith == "exact" else 1e-5)


def _gates(got, want, frac):
    """North-star gates on the final iterate plus the mask band, and the
    scale-aware forms: error relative to max|x_ref| and a
    mask band of 1e-4 * max."""
    got = got.astype(np.float64)
    want = want.astype(np.float64)
    err = float(np.max(np.abs(got - want)))
    cos = float(np.dot(got.ravel(), want.ravel()) / (np.linalg.norm(got) * np.linalg.norm(want)))
    assert err <= 1e-4, err
    assert cos >= 1 - 1e-6, cos
    mx = float(want.max())
    assert err <= 1e-3 * mx, (err, mx)
    cut_g, cut_w = frac * float(got.max()), frac * mx
    flips = (got > cut_g) != (want > cut_w)
    assert np.all(np.abs(want[flips] - cut_w) <= 1e-4 * mx), int(flips.sum())


@pytest.fixture(scope="module")
def c2_ref():
    # full c2: 80 x 480 x 854, C = 8, kernel 7 x 15 x 15 (sigma_t box), 30 iterations
    prob = synth.config(2)[0]
    fs, _ = prob.generate()
    iters = prob.cfg.iterations
    cfg = _cfg(prob, "exact", iterations=iters, binarize_start=iters + 1)
    want = Reference().global_loop_ck(fs.unary, fs.pairwise, cfg, iters, CKS, threads=THREADS)
    return prob, fs, want


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_full_c2_solve_matches_reference_global_loop(c2_ref, arith):
    prob, fs, (want, ref_snaps, norms) = c2_ref
    iters = prob.cfg.iterations
    cfg = _cfg(prob, arith, iterations=iters, binarize_start=iters + 1)
    res, snaps = _run_checkpoints(fs, cfg)
    for it in CKS:
        _gates(snaps[it], ref_snaps[it], cfg.final_threshold)
    _gates(res.soft, want, cfg.final_threshold)
    mine = np.array([r.l2_norm_pre_normalize for r in res.trace.iterations])
    assert np.allclose(mine, norms, rtol=1e-9 if arith == "exact" else 1e-5)


@pytest.mark.parametrize("clip", [0, 8])  # one clip of each resolution
def test_full_c3_clip_matches_reference_global_loop(clip):
    # whole c3 clips (T, H, W drawn by the config's seed), kernel 5 x 9 x 9, 25 iterations
    prob = synth.config(3)[clip]
    fs, _ = prob.generate()
    iters = prob.cfg.iterations
    want = Reference().global_loop(fs.unary, fs.pairwise,
                                   _cfg(prob, "exact", iterations=iters, binarize_start=iters + 1),
                                   iters, threads=THREADS)
    for arith in ("exact", "fast"):
        cfg = _cfg(prob, arith, iterations=iters, binarize_start=iters + 1)
        _gates(E.run(fs, cfg).soft, want, cfg.final_threshold)
