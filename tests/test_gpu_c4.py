"""Parity on BASELINE.json configs[4] (c4: 1024 x 1080 x 1920, C = 3, kernel
9 x 21 x 21, 20 iterations) — the bench's headline workload — and on the
one-call C-ABI entry point sfseg_run that bench.py's e2e times.

* A 32 x 1080 x 1920 crop (full frame: 60 x 17 = 1020 tiles per frame, so
  the persistent schedule's main path runs, not only its remainder branch)
  against the reference's normalize_l2(sfseg_step) loop (bench.cpp:154-155,
  bit-identical to run() for pure power iteration, test_engine.cpp:276-297),
  EXACT and FAST, with the north-star gates at checkpoints 1/5/10/20 and the
  scale-aware forms.
* The full c4 volume: one context against a 2-shard solve of two contexts on
  the same GPU, bit for bit (soft, mask, every norm): the frame-ordered
  canonical reduction makes the result independent of the GPU count, which
  is the c4 multi-GPU parity claim (the reference's own
  thread-count invariance is test_engine.cpp:453-473, acceptance.cpp:521-557).
* sfseg_run (load with S^p under the DMA + solve + download in one call)
  against the reference, including the aliased f = S call of c0/c1/c3.
"""
import os

import numpy as np
import pytest

from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth
from tests.oracle_lib import Reference, reference_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]

THREADS = max(1, os.cpu_count() or 1)
CKS = (1, 5, 10, 20)


def _cfg(prob, arith, **kw):
    return E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, **kw})


def gates(got, want, frac, what=""):
    """North-star gates (max|x - x_ref| <= 1e-4, cos >= 1 - 1e-6, masks equal
    outside a 1e-4 band) plus the scale-aware forms: error <= 1e-3 max|x_ref|
    and mask flips only within 1e-4 max of the cut."""
    got = got.astype(np.float64)
    want = want.astype(np.float64)
    err = float(np.max(np.abs(got - want)))
    cos = float(np.dot(got.ravel(), want.ravel()) / (np.linalg.norm(got) * np.linalg.norm(want)))
    mx = float(want.max())
    assert err <= 1e-4, (what, err)
    assert cos >= 1 - 1e-6, (what, cos)
    assert err <= 1e-3 * mx, (what, err, mx)
    cut_g, cut_w = frac * float(got.max()), frac * mx
    flips = (got > cut_g) != (want > cut_w)
    assert np.all(np.abs(want[flips] - cut_w) <= 1e-4 * mx), (what, int(flips.sum()))
    assert np.all(np.abs(want[flips] - cut_w) <= 1e-4), (what, int(flips.sum()))


@pytest.fixture(scope="module")
def c4_crop():
    prob = synth.config(4, frames=32)[0]
    assert prob.shape == (32, 1080, 1920) and prob.channels == 3
    fs, _ = prob.generate()
    iters = prob.cfg.iterations
    cfg = _cfg(prob, "exact", iterations=iters, binarize_start=iters + 1)
    want, snaps, norms = Reference().global_loop_ck(fs.unary, fs.pairwise, cfg, iters, CKS,
                                                    threads=THREADS)
    return prob, fs, want, snaps, norms


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_c4_crop_checkpoints_match_reference(c4_crop, arith):
    prob, fs, want, snaps, norms = c4_crop
    iters = prob.cfg.iterations
    cfg = _cfg(prob, arith, iterations=iters, binarize_start=iters + 1)
    got = {}
    res = E.run(fs, cfg, observer=lambda it, x: got.__setitem__(it, x.copy()) if it in CKS else None)
    for it in CKS:
        gates(got[it], snaps[it], cfg.final_threshold, f"c4 crop {arith} iter {it}")
    gates(res.soft, want, cfg.final_threshold, f"c4 crop {arith} final")
    mine = np.array([r.l2_norm_pre_normalize for r in res.trace.iterations])
    assert np.allclose(mine, norms, rtol=1e-9 if arith == "exact" else 1e-5)


def test_c4_crop_tap_trim_matches_reference(c4_crop):
    # opt-in FAST tap trimming (sfseg_ctx_set_tap_trim): c4's taps beyond
    # |d| = 8 (space) and |d| = 2 (time) are below 2^-24 of the centre tap, the
    # step runs as (2, 8, 8); same gates against the reference at every
    # checkpoint, and fp32-rounding-level distance from the untrimmed solve
    prob, fs, want, snaps, norms = c4_crop
    iters = prob.cfg.iterations
    cfg = _cfg(prob, "fast", iterations=iters, binarize_start=iters + 1)
    assert E.effective_radii(cfg) == (2, 8, 8)
    for i in (0, 1, 2, 3):  # the other BASELINE kernels keep every tap
        other = synth.config(i)[0].cfg
        assert E.effective_radii(other) == tuple(other.kernel.radii)
    ctx = E.Context(0)
    try:
        ctx.set_tap_trim(True)
        got = {}
        res = E.run(fs, cfg, ctx=ctx,
                    observer=lambda it, x: got.__setitem__(it, x.copy()) if it in CKS else None)
    finally:
        ctx.close()
    for it in CKS:
        gates(got[it], snaps[it], cfg.final_threshold, f"c4 crop trimmed iter {it}")
    gates(res.soft, want, cfg.final_threshold, "c4 crop trimmed final")
    mine = np.array([r.l2_norm_pre_normalize for r in res.trace.iterations])
    assert np.allclose(mine, norms, rtol=1e-5)
    ctx = E.Context(0)
    try:
        ctx.set_tap_trim(False)  # whatever SFSEG_FAST_TRIM says
        base = E.run(fs, cfg, ctx=ctx)
    finally:
        ctx.close()
    d = float(np.max(np.abs(res.soft.astype(np.float64) - base.soft)))
    assert d <= 1e-5 * float(base.soft.max()), d
    assert not np.array_equal(res.soft, base.soft)  # the trimmed kernel did run
    # EXACT never trims: bit-identical with the switch on
    ctx = E.Context(0)
    try:
        ctx.set_tap_trim(True)
        small = synth.config(4, frames=6)[0]
        sf, _ = small.generate()
        ecfg = _cfg(small, "exact", iterations=2, binarize_start=3)
        a = E.run(sf, ecfg, ctx=ctx)
    finally:
        ctx.close()
    b = E.run(sf, ecfg)
    assert np.array_equal(a.soft, b.soft)


@pytest.mark.parametrize("arith", ["fast", "exact"])
def test_c4_crop_run_once_matches_run(c4_crop, arith):
    # sfseg_run in one call equals the load/solve/download sequence bit for bit
    prob, fs, want, _, _ = c4_crop
    iters = prob.cfg.iterations
    cfg = _cfg(prob, arith, iterations=iters, binarize_start=iters + 1)
    a = E.run_once(fs, cfg)
    b = E.run(fs, cfg)
    assert np.array_equal(a.soft, b.soft)
    assert np.array_equal(a.mask, b.mask)
    gates(a.soft, want, cfg.final_threshold, f"c4 crop sfseg_run {arith}")


@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("binarize", [False, True])
def test_run_once_aliased_unary_matches_reference(arith, binarize):
    # c1 T-cropped, f = S passed as the same pointer (sfseg_run uploads it once)
    prob = synth.config(1, frames=12)[0]
    fs, _ = prob.generate()
    alias = E.FeatureSet(fs.unary, [fs.unary])
    iters = prob.cfg.iterations
    cfg = _cfg(prob, arith, binarize_start=3 if binarize else iters + 1)
    res = E.run_once(alias, cfg)
    soft, mask, norms, _ = Reference().run(fs.unary, [fs.unary], cfg, threads=THREADS)
    gates(res.soft, soft, cfg.final_threshold, f"sfseg_run {arith}")
    mine = np.array([r.l2_norm_pre_normalize for r in res.trace.iterations])
    assert np.allclose(mine, norms, rtol=1e-9 if arith == "exact" else 1e-5)


def _sharded_solve(fs, cfg, world):
    """Two (or more) shard contexts on this GPU, exchanging halos and frame
    sums through the host the way NCCL send/recv + all-gather do
    (sharding.py); no kernel waits on another."""
    import torch

    from paper_1907_02731_b200.sharding import CudaBackend, buffer_range, shard_range

    T, H, W = fs.unary.shape
    halo = cfg.kernel.radii[0]
    ranks = []
    for r in range(world):
        t0, t1 = shard_range(T, world, r)
        b0, b1 = buffer_range(T, t0, t1, halo)
        be = CudaBackend(0)
        be.load(T, H, W, fs.unary[b0:b1], [f[b0:b1] for f in fs.pairwise], None, t0, t1, halo)
        be.cfg = cfg
        ranks.append((be, t0, t1))
    params = cfg.to_params()
    for it in range(1, cfg.iterations + 1):
        ios = [be.step(params, it) for be, _, _ in ranks]
        for be, _, _ in ranks:
            be.before_exchange()
        for r in range(world - 1):
            ios[r + 1].recv_lo.copy_(ios[r].send_hi)
            ios[r].recv_hi.copy_(ios[r + 1].send_lo)
        fsum = torch.cat([io.frame_sum for io in ios]).contiguous()
        fmax = torch.cat([io.frame_max for io in ios]).contiguous()
        for be, _, _ in ranks:
            be.after_exchange()
            be.finalize(params, it, fsum, fmax)
    norms = [be.norms(cfg.iterations) for be, _, _ in ranks]
    soft = np.empty(fs.unary.shape, np.float32)
    mask = np.empty(fs.unary.shape, np.uint8)
    for be, a, b in ranks:
        s, m = be.download(cfg.final_threshold, a, b)
        soft[a:b] = s
        mask[a:b] = m
        be.close()
    return soft, mask, norms


@pytest.mark.slow
def test_full_c4_two_shards_bit_identical_to_one_context():
    prob = synth.config(4)[0]
    assert prob.shape == (1024, 1080, 1920)
    fs, _ = prob.generate()
    cfg = _cfg(prob, "fast", binarize_start=prob.cfg.iterations + 1)
    ctx = E.Context(0)  # released before the shards allocate (76 GB each way)
    one = E.run(fs, cfg, ctx=ctx)
    ctx.close()
    soft, mask, norms = _sharded_solve(fs, cfg, 2)
    assert all(n == norms[0] for n in norms)
    assert np.array_equal(norms[0], [r.l2_norm_pre_normalize for r in one.trace.iterations])
    assert np.array_equal(soft, one.soft)
    assert np.array_equal(mask, one.mask)
