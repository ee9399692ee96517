"""Early-exit power iteration (sfseg_solve_until).

The reference's run() always performs cfg.iterations. Its two stopping rules
are restated on the CPU reference (oracle/_ref, the reference compiled from
its sources) and compared with the GPU solve:
  * angle(x_k, x_{k-1}) < tol degrees  — bench.cpp:75-80 converged_conv, which
    iterates normalize_l2(sfseg_step(x)) from x = unary;
  * ||x_k - x_{k-1}||_2 < tol           — oracle.cpp:234-242 power_iteration.
The EXACT step is bit-identical to the reference's; the norm differs in the
fp64 summation order only, so the stopping iteration may differ by one where
the criterion crosses the tolerance within rounding.
"""
import numpy as np
import pytest

from paper_1907_02731_b200 import engine as E
from paper_1907_02731_b200 import synth
from tests.oracle_lib import Reference, reference_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]


def _angle_deg(a, b):
    a = a.astype(np.float64).ravel()
    b = b.astype(np.float64).ravel()
    c = np.clip(a.dot(b) / (np.linalg.norm(a) * np.linalg.norm(b)), -1.0, 1.0)
    return float(np.degrees(np.arccos(c)))


def _reference_loop(fs, cfg, criterion, tol, max_iter):
    ref = Reference()
    x = fs.unary.copy()
    for k in range(1, max_iter + 1):
        xn, _, _ = ref.normalize_l2(ref.step(x, fs.unary, fs.pairwise, cfg))
        if criterion == "angle":
            d = _angle_deg(xn, x)
        else:
            d = float(np.linalg.norm(xn.astype(np.float64) - x.astype(np.float64)))
        x = xn
        if d < tol:
            return x, k
    return x, max_iter


@pytest.mark.parametrize("criterion,tol", [("angle", 1e-5), ("step", 1e-6)])
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_converged_solve_matches_reference_loop(criterion, tol, arith):
    prob = synth.config(0)[0]
    fs, _ = prob.generate()
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 400,
                           "binarize_start": 401})
    res, done = E.run_until_converged(fs, cfg, tol, criterion=criterion)
    want, k = _reference_loop(fs, cfg, criterion, tol, 400)
    assert k < 400, "reference loop did not converge"
    assert abs(done - k) <= (1 if arith == "exact" else 3), (done, k)
    assert len(res.trace.iterations) == done
    err = float(np.max(np.abs(res.soft.astype(np.float64) - want)))
    assert err <= 1e-4
    assert _angle_deg(res.soft, want) < 1e-3


def test_zero_tolerance_runs_every_iteration_like_run():
    prob = synth.config(0)[0]
    fs, _ = prob.generate()
    cfg = prob.cfg
    res, done = E.run_until_converged(fs, cfg, 0.0, criterion="step")
    assert done == cfg.iterations
    full = E.run(fs, cfg)
    assert np.array_equal(res.soft, full.soft)
    assert np.array_equal(res.mask, full.mask)


@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_stop_is_decided_on_the_device_and_the_solve_resumes(arith):
    # the stopping rule is evaluated by k_conv_final on the device: iterations
    # already enqueued behind the stopping one must leave the iterate alone,
    # and a later sfseg_solve continues from it exactly as a straight
    # fixed-count solve would
    import ctypes as C

    from paper_1907_02731_b200 import _native as N

    prob = synth.config(0)[0]
    fs, _ = prob.generate()
    cfg = E.SfsegConfig(**{**prob.cfg.__dict__, "arith": arith, "iterations": 400,
                           "binarize_start": 401})
    p = cfg.to_params()
    ctx = E.Context(0)
    lib = ctx._lib
    try:
        T, H, W = fs.unary.shape
        fp = (C.c_void_p * 1)(fs.pairwise[0].ctypes.data)
        load = lambda: N.check(lib.sfseg_load(ctx.handle, T, H, W, 1, C.c_void_p(fs.unary.ctypes.data),
                                              C.cast(fp, C.c_void_p), None, N.SFSEG_MEM_HOST))
        soft = lambda: (lambda a: (N.check(lib.sfseg_download(ctx.handle, 0.5, C.c_void_p(a.ctypes.data),
                                                              None, N.SFSEG_MEM_HOST)), a)[1])(
            np.empty(fs.unary.shape, np.float32))
        load()
        done = C.c_int32()
        recs = (N.IterRecord * 400)()
        N.check(lib.sfseg_solve_until(ctx.handle, C.byref(p), 1, 400, N.SFSEG_CONV_STEP, 1e-5,
                                      C.byref(done), recs))
        k = done.value
        assert 3 < k < 392  # iterations k+1.. of its chunk were already enqueued when it stopped
        x_stop = soft()
        # a straight k-iteration solve gives the same iterate bit for bit: the
        # iterations enqueued after the stopping one did nothing
        load()
        N.check(lib.sfseg_solve(ctx.handle, C.byref(p), 1, k, None))
        assert np.array_equal(soft(), x_stop)
        # and the stopped solve resumes (the flag was cleared)
        N.check(lib.sfseg_solve(ctx.handle, C.byref(p), k + 1, k + 2, None))
        x_more = soft()
        load()
        N.check(lib.sfseg_solve_until(ctx.handle, C.byref(p), 1, 400, N.SFSEG_CONV_STEP, 1e-5,
                                      C.byref(done), recs))
        assert done.value == k
        N.check(lib.sfseg_solve(ctx.handle, C.byref(p), k + 1, k + 2, None))
        assert np.array_equal(soft(), x_more)
        assert not np.array_equal(x_more, x_stop)
        assert [recs[i].iter for i in range(k)] == list(range(1, k + 1))
        assert all(recs[i].l2_norm_pre_normalize > 0 for i in range(k))
    finally:
        ctx.close()
