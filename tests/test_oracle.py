"""CPU checker tests (no GPU): the oracle (oracle/sfseg_oracle.c) is pinned
bit-for-bit against the golden vectors generated from the reference
(tests/golden/make_golden.py) and, where the reference library is built, against
the reference itself on fresh seeded inputs; plus the known-answer tests of
proj/tests/test_engine.cpp and test_conv3d.cpp."""
from pathlib import Path

import math

import numpy as np
import pytest

from paper_1907_02731_b200.engine import KernelConfig, SfsegConfig
from tests.oracle_lib import Oracle, Reference, random_volume, reference_available

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "reference_vectors.npz")
needs_ref = pytest.mark.skipif(not reference_available(), reason="reference library not built")


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.asarray(a).view(np.uint32),
                                                 np.asarray(b).view(np.uint32))


def cfg_from(prefix):
    g = lambda k: GOLD[f"{prefix}_cfg_{k}"]
    return SfsegConfig(alpha=float(g("alpha")), p=float(g("p")),
                       kernel=KernelConfig(tuple(int(v) for v in g("radii")),
                                           tuple(float(v) for v in g("sigmas"))),
                       iterations=int(g("iterations")), binarize_start=int(g("binarize_start")),
                       sigmoid_slope0=float(g("slope0")), slope_growth=float(g("growth")),
                       threshold_frac=float(g("threshold_frac")),
                       final_threshold=float(g("final_threshold")),
                       allow_negative_affinity=bool(int(g("allow_negative"))))


@pytest.mark.parametrize("i", range(4))
def test_oracle_step_matches_golden(i):
    cfg = cfg_from(f"step{i}")
    got = Oracle().step(GOLD[f"step{i}_x"], GOLD[f"step{i}_S"], [GOLD[f"step{i}_F"]], cfg)
    assert bits_equal(got, GOLD[f"step{i}_out"])


def test_oracle_multichannel_matches_golden():
    cfg = SfsegConfig(p=0.3, kernel=KernelConfig((1, 2, 2), (0.6, 1.1, 1.1)))
    got = Oracle().step(GOLD["mc_x"], GOLD["mc_S"], list(GOLD["mc_F"]), cfg)
    assert bits_equal(got, GOLD["mc_out"])


@pytest.mark.parametrize("tag", ["pi", "bin"])
def test_oracle_run_matches_golden(tag):
    cfg = cfg_from(f"c0_{tag}")
    soft, mask, norms, ck = Oracle().run(GOLD["c0_S"], [GOLD["c0_F"]], cfg,
                                         checkpoints=[1, 5, 10, 20])
    assert bits_equal(soft, GOLD[f"c0_{tag}_soft"])
    assert np.array_equal(mask, GOLD[f"c0_{tag}_mask"])
    assert np.array_equal(norms, GOLD[f"c0_{tag}_norms"])
    assert bits_equal(ck, GOLD[f"c0_{tag}_ck"])


def test_oracle_conv_taps_rng_match_golden():
    o = Oracle()
    assert bits_equal(o.convolve_separable(GOLD["conv_v"], (2, 3, 4), (0.8, 1.3, 2.1)),
                      GOLD["conv_out"])
    tt, ty, tx = o.make_kernel((2, 5, 5), (0.5, 1.5, 1.5))
    assert np.array_equal(tt, GOLD["taps_t"]) and np.array_equal(ty, GOLD["taps_y"])
    assert np.array_equal(tx, GOLD["taps_x"])
    assert np.array_equal(o.xoshiro_u64(20190708, 64), GOLD["rng_u64"])


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_matches_reference_on_fresh_inputs(seed):
    """Random shapes/kernels/alpha/p, incl. radii larger than the volume."""
    rng = np.random.default_rng(seed)
    o, r = Oracle(), Reference()
    for _ in range(4):
        shape = tuple(int(v) for v in rng.integers(1, 9, 3))
        radii = tuple(int(v) for v in rng.integers(0, 4, 3))
        sigmas = tuple(float(v) for v in rng.uniform(0.4, 2.5, 3))
        C = int(rng.integers(1, 4))
        cfg = SfsegConfig(alpha=float(rng.uniform(0.3, 1.0)), p=float(rng.choice([0, 0.1, 0.5, 1])),
                          kernel=KernelConfig(radii, sigmas), iterations=4,
                          binarize_start=int(rng.integers(1, 6)))
        S = random_volume(shape, seed * 100 + 1)
        F = [random_volume(shape, seed * 100 + 2 + c) for c in range(C)]
        x = random_volume(shape, seed * 100 + 9)
        assert bits_equal(o.step(x, S, F, cfg), r.step(x, S, F, cfg))
        a, b = o.run(S, F, cfg), r.run(S, F, cfg)
        assert bits_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.array_equal(a[2], b[2])
        assert bits_equal(o.convolve_separable(x, radii, sigmas),
                          r.convolve_separable(x, radii, sigmas))


@needs_ref
def test_oracle_guard_and_projection_match_reference():
    o, r = Oracle(), Reference()
    S = random_volume((3, 10, 10), 5)
    F = [random_volume((3, 10, 10), 6) * 3.0 - 1.0]  # out of [0,1]: guard rescales
    cfg = SfsegConfig(iterations=3)
    a, b = o.run(S, F, cfg), r.run(S, F, cfg)
    assert bits_equal(a[0], b[0])
    x = random_volume((2, 9, 9), 7)
    for it in (1, 3, 5):
        assert bits_equal(o.project_binary(x, it, cfg), r.project_binary(x, it, cfg))
    assert np.array_equal(o.threshold_final(x, 0.3), r.threshold_final(x, 0.3))
    un, nn, _ = o.normalize_l2(x)
    ur, nr, _ = r.normalize_l2(x)
    assert bits_equal(un, ur) and nn == nr


# ---- known answers (proj/tests/test_engine.cpp, test_conv3d.cpp) -------------

def test_known_answers_normalize_threshold_sigmoid():
    o = Oracle()
    u, n, rc = o.normalize_l2(np.array([[[3.0, 4.0]]], np.float32))  # :99-110
    assert rc == 0 and n == pytest.approx(5.0, rel=1e-12)
    assert u.ravel().tolist() == pytest.approx([0.6, 0.8], rel=1e-7)
    assert o.normalize_l2(np.zeros((1, 1, 2), np.float32))[2] == 4  # DegenerateSolution
    x = np.array([[[0.9, 0.44, 0.46, 0.1]]], np.float32)  # :148-159
    assert o.threshold_final(x, 0.5).ravel().tolist() == [1, 0, 1, 0]
    cfg = SfsegConfig(binarize_start=3)  # :112-146
    x = np.array([[[0.0, 0.5, 1.0]]], np.float32)
    assert bits_equal(o.project_binary(x, 2, cfg), x)
    p3 = o.project_binary(x, 3, cfg).ravel()
    assert p3[0] == pytest.approx(1 / (1 + math.exp(5.0)), rel=1e-6)
    assert o.project_binary(x, 5, cfg).ravel()[2] == pytest.approx(1 / (1 + math.exp(-20)), rel=1e-6)


def test_known_answers_kernel_and_convolution():
    o = Oracle()
    tt, ty, tx = o.make_kernel((1, 3, 3), (0.5, 1.5, 1.5))  # test_conv3d.cpp:60-84
    raw = lambda s, d: math.exp(-d * d / (2 * s * s))
    total = (sum(raw(0.5, d) for d in range(-1, 2)) * sum(raw(1.5, d) for d in range(-3, 4)) ** 2)
    assert ty[3] == 1.0 and tx[3] == 1.0
    assert tt[1] == pytest.approx(1 / total, rel=1e-14)
    mass = np.einsum("i,j,k->", tt, ty, tx)
    assert mass == pytest.approx(1.0, rel=1e-12)
    v = random_volume((3, 5, 4), 99)  # radius-0 identity (:100-108)
    assert bits_equal(o.convolve_separable(v, (0, 0, 0), (1.0, 1.0, 1.0)), v)
    imp = np.zeros((3, 9, 9), np.float32)  # impulse response (:110-139)
    imp[1, 4, 4] = 1.0
    out = o.convolve_separable(imp, (1, 3, 3), (0.5, 1.5, 1.5))
    w = np.einsum("i,j,k->ijk", tt, ty, tx)
    assert np.allclose(out[0:3, 1:8, 1:8], w, rtol=1e-5, atol=0)
    assert out[1, 4, 8] == 0.0 and out[1, 0, 4] == 0.0
