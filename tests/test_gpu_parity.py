"""GPU parity: the sm_100a path against the CPU oracle / reference (gpu marker).

Bar (BASELINE.json north_star): after normalisation max|x - x_ref| <= 1e-4 and
cosine >= 1 - 1e-6 at every checkpoint; masks identical except voxels within
1e-4 of the threshold. In EXACT arithmetic the step itself is bit-identical to
the reference (same products, sums and order), so the step tests demand
equality of every value.
"""
import numpy as np
import pytest

from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth
from tests.oracle_lib import Oracle, Reference, random_volume, reference_available

pytestmark = pytest.mark.gpu

TOL_ABS = 1e-4
TOL_COS = 1e-6


def _cfg(radii=(1, 3, 3), sigmas=(0.5, 1.5, 1.5), alpha=1.0, p=0.1, arith="exact", **kw):
    return E.SfsegConfig(alpha=alpha, p=p, kernel=E.KernelConfig(tuple(radii), tuple(sigmas)),
                         arith=arith, **kw)


def _equal_values(a, b):
    """bit-equal up to the sign of zero"""
    return np.array_equal(a, b) and a.shape == b.shape


def _features(shape, seed, channels=1):
    S = random_volume(shape, seed)
    F = [random_volume(shape, seed + 1 + c) for c in range(channels)]
    return S, F


def _gate(x, ref, what=""):
    x = x.astype(np.float64).ravel()
    ref = ref.astype(np.float64).ravel()
    err = np.max(np.abs(x - ref))
    cos = float(np.dot(x, ref) / (np.linalg.norm(x) * np.linalg.norm(ref)))
    assert err <= TOL_ABS, f"{what}: max abs {err:.3e}"
    assert cos >= 1 - TOL_COS, f"{what}: cosine {cos:.12f}"
    return err, cos


def _mask_gate(m, mref, soft_ref, frac):
    cut = np.float32(frac * float(max(0.0, soft_ref.max())))
    diff = m != mref
    band = np.abs(soft_ref - cut) <= 1e-4
    assert not np.any(diff & ~band), f"{int(np.sum(diff & ~band))} mask flips outside the band"


# the four kernel/alpha/p cases of test_engine.cpp:161-191, plus the configs'
STEP_CASES = [
    ((4, 8, 8), 1.0, 0.1, (1, 3, 3), (0.5, 1.5, 1.5)),
    ((4, 8, 8), 0.7, 0.5, (1, 1, 1), (0.9, 0.9, 0.9)),
    ((3, 6, 6), 1.0, 0.0, (0, 2, 2), (1.0, 2.0, 2.0)),
    ((2, 5, 7), 0.5, 1.0, (1, 2, 2), (0.7, 1.2, 1.2)),
    ((8, 64, 64), 1.0, 0.1, (1, 3, 3), (1e30, 1e30, 1e30)),
    ((9, 70, 130), 1.0, 0.1, (2, 5, 5), (0.5, 1.5, 1.5)),
    ((7, 45, 97), 1.0, 0.3, (2, 4, 4), (0.5, 1.5, 1.5)),
    ((5, 33, 200), 0.9, 0.2, (2, 3, 5), (0.6, 1.2, 1.7)),
]


@pytest.mark.parametrize("shape,alpha,p,radii,sigmas", STEP_CASES)
def test_step_channel_bit_exact(shape, alpha, p, radii, sigmas):
    S, F = _features(shape, 11)
    x = random_volume(shape, 99)
    cfg = _cfg(radii, sigmas, alpha, p)
    got = E.sfseg_step_channel(x, S, F[0], cfg)
    want = Oracle().step(x, S, F, cfg)
    assert _equal_values(got, want), f"max diff {np.max(np.abs(got - want)):.3e}"


def test_step_multichannel_is_channel_sum():
    shape = (3, 7, 7)
    S, F = _features(shape, 5, channels=3)
    x = random_volume(shape, 6)
    cfg = _cfg((1, 2, 2), (0.6, 1.1, 1.1), p=0.3)
    got = E.sfseg_step(x, E.FeatureSet(S, F), cfg)
    assert _equal_values(got, Oracle().step(x, S, F, cfg))
    manual = E.sfseg_step_channel(x, S, F[0], cfg)
    for c in range(1, 3):
        manual = manual + E.sfseg_step_channel(x, S, F[c], cfg)  # float32 add, channel order
    assert _equal_values(got, manual)


def test_normalize_project_threshold_match_oracle():
    o = Oracle()
    x = random_volume((5, 21, 40), 3)
    u, n = E.normalize_l2(x)
    uo, no, _ = o.normalize_l2(x)
    assert abs(n - no) <= 1e-12 * no
    assert np.max(np.abs(u - uo)) <= 1e-7
    cfg = _cfg(binarize_start=2)
    assert _equal_values(E.project_binary(x, 1, cfg), x)
    pb = E.project_binary(x, 3, cfg)
    assert np.max(np.abs(pb - o.project_binary(x, 3, cfg))) <= 1e-7
    assert np.array_equal(E.threshold_final(x, 0.5), o.threshold_final(x, 0.5))


def test_known_answers():
    # 3-4-5 (test_engine.cpp:99-110)
    v = np.array([[[3.0, 4.0]]], np.float32)
    u, n = E.normalize_l2(v)
    assert n == pytest.approx(5.0, rel=1e-12)
    assert u.ravel().tolist() == pytest.approx([0.6, 0.8], rel=1e-7)
    with pytest.raises(E.DegenerateSolutionError):
        E.normalize_l2(np.zeros((1, 1, 2), np.float32))
    # strict threshold (test_engine.cpp:148-159)
    x = np.array([[[0.9, 0.44, 0.46, 0.1]]], np.float32)
    assert E.threshold_final(x, 0.5).ravel().tolist() == [1, 0, 1, 0]
    assert E.threshold_final(np.zeros((1, 1, 4), np.float32), 0.5).sum() == 0
    # sigmoid schedule (test_engine.cpp:112-146)
    cfg = _cfg(binarize_start=3)
    x = np.array([[[0.0, 0.5, 1.0]]], np.float32)
    p3 = E.project_binary(x, 3, cfg).ravel()
    assert p3[0] == pytest.approx(1 / (1 + np.exp(5.0)), rel=1e-6)
    assert p3[1] == pytest.approx(0.5, rel=1e-6)
    p5 = E.project_binary(x, 5, cfg).ravel()
    assert p5[2] == pytest.approx(1 / (1 + np.exp(-20.0)), rel=1e-6)


def _problem(idx, frames=None, k=0):
    prob = synth.config(idx, frames=frames)[k]
    fs, gt = prob.generate(mask=True)
    return prob, fs, gt


@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("binarize", [False, True])
def test_run_c0_matches_reference(binarize, arith):
    prob, fs, _ = _problem(0)
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith})
    if binarize:
        cfg = E.SfsegConfig(**{**cfg.__dict__, "binarize_start": 3})
    cks = [1, 5, 10, 15, 20]
    snaps = {}
    res = E.run(fs, cfg, observer=lambda it, x: snaps.__setitem__(it, x.copy()))
    soft, mask, norms, ck = Oracle().run(fs.unary, fs.pairwise, cfg, checkpoints=cks)
    for i, it in enumerate(cks):
        _gate(snaps[it], ck[i], f"iter {it}")
    _gate(res.soft, soft, "final")
    _mask_gate(res.mask, mask, soft, cfg.final_threshold)
    got_norms = np.array([r.l2_norm_pre_normalize for r in res.trace.iterations])
    assert np.allclose(got_norms, norms, rtol=1e-10 if arith == "exact" else 1e-5)


@pytest.mark.parametrize("shape,alpha,p,radii,sigmas", STEP_CASES)
def test_step_fast_within_tolerance(shape, alpha, p, radii, sigmas):
    S, F = _features(shape, 11)
    x = random_volume(shape, 99)
    cfg = _cfg(radii, sigmas, alpha, p, arith="fast")
    got = E.sfseg_step_channel(x, S, F[0], cfg).astype(np.float64)
    want = Oracle().step(x, S, F, cfg).astype(np.float64)
    # FMA vs separately rounded products: a few ulps of the step's scale
    assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


# FAST with C > 1 runs the (C + 2)-field kernels (fused_mc.cuh): a HEAD launch
# (u, Q u) and TAIL launches of one or two channels. Same operator, regrouped,
# so the step matches the reference within the FAST tolerance.
MC_CASES = [
    ((9, 70, 130), (2, 5, 5), (0.5, 1.5, 1.5), 2),
    ((7, 45, 97), (2, 4, 4), (0.5, 1.5, 1.5), 3),
    ((8, 96, 160), (3, 7, 7), (1e30, 5.0, 5.0), 8),
    ((10, 90, 150), (4, 10, 10), (0.5, 1.5, 1.5), 3),
    ((6, 67, 70), (4, 10, 10), (0.5, 1.5, 1.5), 5),
]


@pytest.mark.parametrize("shape,radii,sigmas,C", MC_CASES)
def test_step_multichannel_fast_within_tolerance(shape, radii, sigmas, C):
    # twice with the same shape and new channel data: the per-solve derived
    # fields (Q, 2 S^p f_c) must not survive a change of the channels
    for seed in (21, 121):
        S, F = _features(shape, seed, channels=C)
        x = random_volume(shape, 77)
        cfg = _cfg(radii, sigmas, 1.0, 0.1 if seed == 21 else 0.3, arith="fast")
        fs = E.FeatureSet(S, F)
        got = E.sfseg_step(x, fs, cfg).astype(np.float64)
        want = Oracle().step(x, S, F, cfg).astype(np.float64)
        assert np.max(np.abs(got - want)) <= 1e-5 * np.max(np.abs(want))


def test_run_c1_cropped_fast_matches_reference():
    prob, fs, _ = _problem(1, frames=12)
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": "fast"})
    res = E.run(fs, cfg)
    soft, mask, norms, _ = Oracle().run(fs.unary, fs.pairwise, cfg)
    _gate(res.soft, soft, "c1[T=12] fast")
    _mask_gate(res.mask, mask, soft, cfg.final_threshold)


def test_run_c1_cropped_matches_reference():
    prob, fs, _ = _problem(1, frames=10)
    cfg = prob.cfg
    snaps = {}
    res = E.run(fs, cfg, observer=lambda it, x: snaps.__setitem__(it, x.copy()) if it == 1 else None)
    soft, mask, norms, ck = Oracle().run(fs.unary, fs.pairwise, cfg, checkpoints=[1])
    _gate(res.soft, soft, "c1[T=10]")
    _mask_gate(res.mask, mask, soft, cfg.final_threshold)
    # exact arithmetic: after one iteration the iterate is bit-identical except
    # where float(y * inv) rounds differently because the fp64 norm was summed
    # in another order (a few voxels); later iterations spread those ulps.
    assert np.mean(snaps[1] == ck[0]) > 0.9999
    assert np.allclose([r.l2_norm_pre_normalize for r in res.trace.iterations], norms, rtol=1e-9)


def test_run_is_normalize_of_step():
    # test_engine.cpp:359-387 / 276-297: run(1 iteration) == normalize_l2(step)
    prob, fs, _ = _problem(0)
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "iterations": 1, "binarize_start": 2})
    res = E.run(fs, cfg)
    stepped = E.sfseg_step(fs.unary, fs, cfg)
    want, _ = E.normalize_l2(stepped)
    assert _equal_values(res.soft, want)


# --- the remaining BASELINE configs (c2, c3, c4), cropped so the reference
# CPU run finishes in seconds; same channels, kernel and iteration count ---

def _crop(fs, T, H, W):
    sl = (slice(0, T), slice(0, H), slice(0, W))
    return E.FeatureSet(np.ascontiguousarray(fs.unary[sl]),
                        [np.ascontiguousarray(f[sl]) for f in fs.pairwise])


def _ref_threads():
    import os
    return max(1, os.cpu_count() or 1)


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("arith", ["exact", "fast"])
@pytest.mark.parametrize("idx,crop", [(2, (8, 96, 160)), (4, (10, 90, 150))])
def test_run_multichannel_configs_cropped_match_reference(idx, crop, arith):
    # c2: C=8, radii (3,7,7), box in t; c4: C=3, radii (4,10,10)
    prob = synth.config(idx, frames=crop[0])[0]
    fs, _ = prob.generate()
    fs = _crop(fs, *crop)
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith})
    cks = [1, 5, cfg.iterations]
    snaps = {}
    res = E.run(fs, cfg, observer=lambda it, x: snaps.__setitem__(it, x.copy()) if it in cks else None)
    soft, mask, norms, ck = Reference().run(fs.unary, fs.pairwise, cfg, checkpoints=cks,
                                            threads=_ref_threads())
    for i, it in enumerate(cks):
        _gate(snaps[it], ck[i], f"c{idx}{list(crop)} iter {it}")
    _gate(res.soft, soft, f"c{idx} final")
    _mask_gate(res.mask, mask, soft, cfg.final_threshold)
    got = np.array([r.l2_norm_pre_normalize for r in res.trace.iterations])
    assert np.allclose(got, norms, rtol=1e-9 if arith == "exact" else 1e-5)


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_run_c3_clips_match_reference():
    # c3: independent clips (each its own problem, own norm); every clip of
    # the batch T-cropped to 12 frames, full resolution
    from paper_1907_02731_b200.sharding import run_problems

    clips = synth.config(3, frames=12)[:4]
    results = run_problems(clips, rank=0, world=1)  # the clip-sharded driver, one rank
    assert sorted(results) == list(range(len(clips)))
    for i, prob in enumerate(clips):
        fs, _ = prob.generate()
        res = results[i]
        soft, mask, _, _ = Reference().run(fs.unary, fs.pairwise, prob.cfg, threads=_ref_threads())
        _gate(res.soft, soft, prob.name)
        _mask_gate(res.mask, mask, soft, prob.cfg.final_threshold)


# radii beyond the fused instantiations run the generic multi-pass path; in
# EXACT arithmetic it is bit-identical to the reference step as well
GENERIC_CASES = [
    ((5, 40, 70), 1.0, 0.1, (3, 7, 7), (1e30, 5.0, 5.0), 3),
    ((9, 50, 60), 1.0, 0.1, (4, 10, 10), (0.5, 1.5, 1.5), 2),
]


@pytest.mark.parametrize("shape,alpha,p,radii,sigmas,C", GENERIC_CASES)
def test_step_generic_path_bit_exact(shape, alpha, p, radii, sigmas, C):
    S, F = _features(shape, 21, channels=C)
    x = random_volume(shape, 98)
    cfg = _cfg(radii, sigmas, alpha, p)
    fs = E.FeatureSet(S, F)
    got = E.sfseg_step(x, fs, cfg)
    want = Oracle().step(x, S, F, cfg)
    assert _equal_values(got, want)


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_observer_may_call_the_engine_on_the_same_context(arith):
    # the stateless operators run on the context's scratch buffers: calling
    # them from an IterationObserver (same default context, same thread)
    # neither deadlocks nor disturbs the resident solve
    prob, fs, _ = _problem(2, frames=6)
    fs = _crop(fs, 6, 60, 90)
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 5})
    base = E.run(fs, cfg)
    seen = []

    def obs(it, x):
        y = E.sfseg_step(x, fs, cfg)
        u, n = E.normalize_l2(y)
        E.threshold_final(u, 0.5)
        seen.append(n)

    res = E.run(fs, cfg, observer=obs)
    assert len(seen) == cfg.iterations
    assert np.array_equal(res.soft, base.soft)
    assert np.array_equal(res.mask, base.mask)
    # the observer's step of iterate k is the solve's step k+1: same norm
    norms = [r.l2_norm_pre_normalize for r in res.trace.iterations]
    assert np.allclose(seen[:-1], norms[1:], rtol=1e-5)


@pytest.mark.parametrize("shape,radii,sigmas", [
    ((5, 9, 11), (1, 2, 3), (0.5, 1.5, 1.5)),
    ((3, 17, 40), (2, 4, 4), (0.7, 1.1, 2.0)),
    ((6, 6, 6), (0, 1, 0), (1.0, 1e30, 1.0)),
])
def test_convolve_direct_matches_reference_and_separable(shape, radii, sigmas):
    # conv3d.hpp:62-68 / conv3d.cpp:187-243: the dense fp64 triple sum. Bit
    # for bit against the reference's own convolve_direct; and the relation
    # test_conv3d.cpp:159-176 pins: separable == direct within 1e-5
    v = random_volume(shape, 77)
    k = E.KernelConfig(radii, sigmas)
    got = E.convolve_direct(v, k)
    sep = E.convolve_separable(v, k)
    assert np.max(np.abs(got - sep)) <= 1e-5
    if reference_available():
        want = Reference().convolve_direct(v, radii, sigmas)
        assert _equal_values(got, want), f"max diff {np.max(np.abs(got - want)):.3e}"
    # impulse response = outer product of the taps (test_conv3d.cpp:110-139)
    imp = np.zeros(shape, np.float32)
    c = tuple(s // 2 for s in shape)
    imp[c] = 1.0
    kk = E.make_gaussian_kernel(sigmas, radii)
    out = E.convolve_direct(imp, kk)
    for dt in range(-radii[0], radii[0] + 1):
        for dy in range(-radii[1], radii[1] + 1):
            for dx in range(-radii[2], radii[2] + 1):
                p = (c[0] + dt, c[1] + dy, c[2] + dx)
                if all(0 <= p[a] < shape[a] for a in range(3)):
                    w = kk.taps_t[dt + radii[0]] * kk.taps_y[dy + radii[1]] * kk.taps_x[dx + radii[2]]
                    assert abs(float(out[p]) - w) <= 1e-6 * max(1.0, abs(w))
