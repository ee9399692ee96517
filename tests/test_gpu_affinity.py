"""The reference's explicit-matrix oracle on the GPU (SURVEY §8(f) row 3,
oracle.cpp:67-258): sfseg_affinity_matvec / sfseg_affinity_power_iteration
against the reference's own build_affinity_* + matvec + power_iteration
(compiled from its sources, oracle/_ref), and beyond the reference's
1e6-node cap against the engine's Taylor step (test_engine.cpp:161-215's
relation step(x) = M x / alpha)."""
import numpy as np
import pytest

from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200._native import SFSEG_ERR_CAPACITY
from tests.oracle_lib import Reference, random_volume, reference_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]

# test_engine.cpp:170-175 cases, the multi-channel case (:194-199), configs' radii
CASES = [
    ((4, 8, 8), 1.0, 0.1, (1, 3, 3), (0.5, 1.5, 1.5), 1),
    ((4, 8, 8), 0.7, 0.5, (1, 1, 1), (0.9, 0.9, 0.9), 1),
    ((3, 6, 6), 1.0, 0.0, (0, 2, 2), (1.0, 2.0, 2.0), 1),
    ((2, 5, 7), 0.5, 1.0, (1, 2, 2), (0.7, 1.2, 1.2), 1),
    ((3, 7, 7), 1.0, 0.3, (1, 2, 2), (0.6, 1.1, 1.1), 3),
    ((6, 40, 52), 1.0, 0.1, (2, 5, 5), (0.5, 1.5, 1.5), 2),
    ((5, 30, 33), 0.8, 0.2, (3, 7, 7), (1e30, 5.0, 5.0), 8),
]


def _problem(shape, C, seed):
    S = random_volume(shape, seed)
    F = [random_volume(shape, seed + 1 + c) for c in range(C)]
    return S, F


@pytest.mark.parametrize("kind", ["taylor", "taylor_channel_sum", "exact"])
@pytest.mark.parametrize("shape,alpha,p,radii,sigmas,C", CASES)
def test_matvec_matches_reference(shape, alpha, p, radii, sigmas, C, kind):
    S, F = _problem(shape, C, 31)
    cfg = E.SfsegConfig(alpha=alpha, p=p, kernel=E.KernelConfig(radii, sigmas))
    x = random_volume(shape, 7).astype(np.float64)
    got = E.affinity_matvec(E.FeatureSet(S, F), cfg, x, kind)
    rc, want = Reference().affinity_matvec(S, F, cfg, x, kind)
    assert rc == 0
    if kind == "exact":  # device exp vs libm exp: within a few ulps per entry
        assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))
    else:  # same entries, same order, same rounding
        assert np.array_equal(got, want), f"max diff {np.max(np.abs(got - want)):.3e}"


@pytest.mark.parametrize("kind", ["taylor_channel_sum", "exact"])
def test_power_iteration_matches_reference(kind):
    shape, C = (5, 24, 30), 2
    S, F = _problem(shape, C, 41)
    cfg = E.SfsegConfig(kernel=E.KernelConfig((1, 3, 3), (0.5, 1.5, 1.5)))
    x0 = S.astype(np.float64)
    vec, val, used = E.power_iteration(E.FeatureSet(S, F), cfg, x0, 300, 1e-9, kind)
    rvec, rval, rused = Reference().power_iteration(S, F, cfg, x0, 300, 1e-9, kind)
    assert abs(used - rused) <= 1  # the stopping test compares ~1e-9 with fp64 tree vs serial sums
    assert np.max(np.abs(vec - rvec)) <= 1e-9
    assert abs(val - rval) <= 1e-12 * abs(rval)
    assert abs(np.linalg.norm(vec) - 1.0) <= 1e-12


def test_beyond_reference_node_cap_matches_engine_step():
    # 16 x 256 x 256 = 1.05e6 voxels: the reference refuses (CapacityError);
    # the GPU oracle and the fused EXACT step agree as in test_engine.cpp:161-215
    shape, C = (16, 256, 256), 2
    S, F = _problem(shape, C, 51)
    cfg = E.SfsegConfig(p=0.3, kernel=E.KernelConfig((1, 2, 2), (0.6, 1.1, 1.1)))
    x = random_volume(shape, 9)
    rc, _ = Reference().affinity_matvec(S, F, cfg, x.astype(np.float64), "taylor_channel_sum")
    assert rc == SFSEG_ERR_CAPACITY
    mx = E.affinity_matvec(E.FeatureSet(S, F), cfg, x.astype(np.float64), "taylor_channel_sum")
    step = E.sfseg_step(x, E.FeatureSet(S, F), cfg).astype(np.float64)
    assert np.max(np.abs(step - mx / cfg.alpha)) <= 1e-4


def test_errors_follow_the_reference():
    S, F = _problem((2, 8, 8), 1, 61)
    fs = E.FeatureSet(S, F)
    cfg = E.SfsegConfig()
    with pytest.raises(E.ParameterError):
        E.power_iteration(fs, cfg, S.astype(np.float64), 0, 1e-6)
    with pytest.raises(E.ParameterError):
        E.power_iteration(fs, cfg, np.zeros(S.shape), 5, 1e-6)
    with pytest.raises(E.ValidationError):  # guard on: a channel outside [0, 1]
        E.affinity_matvec(E.FeatureSet(S, [F[0] + 1.0]), cfg, np.ones(S.shape))
    ok = E.affinity_matvec(E.FeatureSet(S, [F[0] + 1.0]), E.SfsegConfig(allow_negative_affinity=True),
                           np.ones(S.shape))
    assert np.all(np.isfinite(ok))
