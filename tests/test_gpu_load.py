"""Host-memory loads through the pipelined path (row chunks on a copy stream,
re-pitch and validation on the library stream, one flag read-back): the
validation errors of FeatureSet::validate (volume.cpp:72-93) and of a bad x0
(engine.cpp:266) in load order, and a clean load after a failed one.
Widths that are not a multiple of 32 floats take the pipelined path; the
volume spans several 32 MB chunks so the staging ring wraps."""
import numpy as np
import pytest

from paper_1907_02731_b200 import engine as E
from tests.oracle_lib import random_volume

pytestmark = pytest.mark.gpu

SHAPE = (24, 480, 854)  # 39 MB per volume: two chunks, P != W


def _problem(channels=2):
    S = random_volume(SHAPE, 1)
    F = [random_volume(SHAPE, 2 + c) for c in range(channels)]
    cfg = E.SfsegConfig(kernel=E.KernelConfig((1, 3, 3), (0.5, 1.5, 1.5)), iterations=3,
                        binarize_start=4, arith="fast")
    return S, F, cfg


def test_pipelined_load_matches_sequential_semantics():
    S, F, cfg = _problem()
    ctx = E.Context(0)
    a = E.run(E.FeatureSet(S, F), cfg, ctx=ctx).soft
    b = E.run(E.FeatureSet(S, F), cfg, ctx=ctx).soft  # reloading the same context
    assert np.array_equal(a, b)
    # device-resident inputs take the direct path: same result
    import torch
    dS = torch.from_numpy(S).cuda()
    dF = [torch.from_numpy(f).cuda() for f in F]
    c = E.run(E.FeatureSet(dS, dF), cfg, ctx=ctx).soft
    assert np.array_equal(a, np.asarray(c.cpu() if hasattr(c, "cpu") else c))


@pytest.mark.parametrize("where,value,msg", [
    ("unary", -1.0, "negative"),
    ("unary", np.nan, "non-finite"),
    ("pairwise1", np.inf, "pairwise"),
    ("x0", -0.5, "x0"),
])
def test_pipelined_load_validation_errors(where, value, msg):
    S, F, cfg = _problem()
    x0 = None
    t, y, x = 17, 401, 853  # in the second chunk, last column
    if where == "unary":
        S = S.copy()
        S[t, y, x] = value
    elif where == "pairwise1":
        F = [F[0], F[1].copy()]
        F[1][t, y, x] = value
    else:
        x0 = random_volume(SHAPE, 9)
        x0[t, y, x] = value
    ctx = E.Context(0)
    with pytest.raises(E.ValidationError, match=msg):
        E.run(E.FeatureSet(S, F), cfg, x0=x0, ctx=ctx)
    # the context recovers: a clean problem loads and solves as on a fresh one
    S2, F2, _ = _problem()
    got = E.run(E.FeatureSet(S2, F2), cfg, ctx=ctx).soft
    want = E.run(E.FeatureSet(S2, F2), cfg, ctx=E.Context(0)).soft
    assert np.array_equal(got, want)


def test_pipelined_load_reports_the_first_bad_volume():
    S, F, cfg = _problem()
    S = S.copy()
    S[0, 0, 0] = -1.0
    F = [F[0].copy(), F[1]]
    F[0][0, 0, 0] = np.nan
    with pytest.raises(E.ValidationError, match="unary"):
        E.run(E.FeatureSet(S, F), cfg, ctx=E.Context(0))


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_feature_aliasing_unary_is_uploaded_once_same_result(arith):
    # f = S passed as one host buffer (sfseg_load uploads it once and copies it
    # on the device) == f passed as its own copy, bit for bit
    S, F, cfg = _problem()
    cfg.arith = arith
    ctx = E.Context(0)
    a = E.run(E.FeatureSet(S, [S, F[1]]), cfg, ctx=ctx).soft
    b = E.run(E.FeatureSet(S, [S.copy(), F[1]]), cfg, ctx=ctx).soft
    assert np.array_equal(a, b)
    c = E.run(E.FeatureSet(S, [S]), cfg, ctx=ctx).soft
    d = E.run(E.FeatureSet(S, [S.copy()]), cfg, ctx=E.Context(0)).soft
    assert np.array_equal(c, d)
